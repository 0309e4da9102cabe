set -u
O=gpurun_out/r2k; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/gpu_tests.log 2>&1; echo "EXIT $?" >> $O/gpu_tests.log
python bench.py --no-e2e --no-cpu-baseline > $O/bench_default.json 2> $O/bench_default.err
for c in cfg1 cfg5 cfg4; do python bench.py --config $c --no-e2e --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
ls -la $O
