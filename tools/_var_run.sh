set -u
O=gpurun_out/var2; mkdir -p $O
MMJ_FUSE_VARIANT=3 timeout 600 python -m pytest tests/test_gpu_fused.py -x -q > $O/tests_3.log 2>&1; echo EXIT $? >> $O/tests_3.log
for v in 3 0 3 0 3 0; do MMJ_FUSE_VARIANT=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench_${v}_$RANDOM.json 2>>$O/bench.err; done
