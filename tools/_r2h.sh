set -u
O=gpurun_out/r2h; mkdir -p $O
for v in 2 1 2 1; do MMJ_EMIT_RR=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench_rr$v.$RANDOM.json 2>>$O/bench.err; done
for i in 1 2; do timeout 600 python bench.py --config cfg5 --no-e2e --no-cpu-baseline > $O/cfg5_lists.$i.json 2>>$O/bench.err; done
MMJ_EMIT_RR=2 timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_twopath.py tests/test_gpu_apps.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "EXIT $?" >> $O/tests.log
ls -la $O
