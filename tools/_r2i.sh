set -u
O=gpurun_out/r2i; mkdir -p $O
MMJ_EMIT_RR=3 timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_twopath.py tests/test_gpu_golden.py -q -x -p no:cacheprovider > $O/tests_rr3.log 2>&1; echo "EXIT $?" >> $O/tests_rr3.log
for v in 3 1 3 1; do MMJ_EMIT_RR=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench_rr$v.$RANDOM.json 2>>$O/bench.err; done
timeout 1200 python -m pytest tests/test_gpu_checked.py -q -p no:cacheprovider > $O/checked.log 2>&1; echo "EXIT $?" >> $O/checked.log
cp gpurun_out/checked_cases.log $O/ 2>/dev/null
ls -la $O
