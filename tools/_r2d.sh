set -u
O=gpurun_out/r2d; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_fused.py tests/test_gpu_twopath.py tests/test_gpu_golden.py tests/test_gpu_apps.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "EXIT $?" >> $O/tests.log
for v in 1 0; do MMJ_EMIT_RR=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench_rr$v.json 2>>$O/bench.err; done
MMJ_EMIT_RR=1 timeout 600 python bench.py --config cfg3 --no-e2e --no-cpu-baseline > $O/cfg3_rr1.json 2>>$O/bench.err
for f in lists records; do timeout 600 python bench.py --config cfg5 --bsi-form $f --no-e2e --no-cpu-baseline > $O/cfg5_$f.json 2>>$O/bench.err; done
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_cases.py > $O/memcheck.log 2>&1; echo "EXIT $?" >> $O/memcheck.log
FC="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify --no-light-work --x-limit 65536"
$FC > $O/full_plain.json 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_merge_emit" -s 8 -c 1 \
      -o $O/merge_emit_rr $FC > $O/full_ncu.log 2>&1
ls -la $O
