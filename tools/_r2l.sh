set -u
O=gpurun_out/r2l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_apps.py -q -p no:cacheprovider -k bsi > $O/tests.log 2>&1; echo "EXIT $?" >> $O/tests.log
for i in 1 2; do python bench.py --config cfg5 --no-e2e --no-cpu-baseline > $O/cfg5.$i.json 2>>$O/bench.err; done
for v in 0 1 2 0 1 2; do MMJ_FUSE_SHAPE=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench_shape$v.$RANDOM.json 2>>$O/bench.err; done
ls -la $O
