set -u
O=gpurun_out/var; mkdir -p $O
for v in 3 4; do MMJ_FUSE_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_golden.py -x -q > $O/tests_$v.log 2>&1; echo EXIT $? >> $O/tests_$v.log; done
for v in 3 0 4 3 0 4; do MMJ_FUSE_VARIANT=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench_${v}_$RANDOM.json 2>>$O/bench.err; done
