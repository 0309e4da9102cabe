set -u
O=gpurun_out/r2b; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > $O/gpu_tests.log 2>&1; echo "EXIT $?" >> $O/gpu_tests.log
cp gpurun_out/reference_suite.log $O/ 2>/dev/null
for c in cfg1 cfg3 cfg4 cfg5; do timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err; echo "EXIT $?" >> $O/bench_$c.err; done
FC="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify --no-light-work --x-limit 65536"
$FC > $O/full_plain.json 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_merge_emit" -s 8 -c 1 \
      -o $O/merge_emit_or $FC > $O/full_ncu.log 2>&1
ls -la $O
