set -u
O=gpurun_out/var3; mkdir -p $O
MMJ_FUSE_VARIANT=4 timeout 600 python -m pytest tests/test_gpu_fused.py -x -q > $O/tests_4.log 2>&1; echo EXIT $? >> $O/tests_4.log
for v in 4 0 4 0 4 0; do MMJ_FUSE_VARIANT=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench_${v}_$RANDOM.json 2>>$O/bench.err; done
