set -u
O=gpurun_out/cta3; mkdir -p $O
MMJ_CTA_EMIT=1 timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_golden.py -x -q > $O/tests.log 2>&1; echo EXIT $? >> $O/tests.log
for v in 1 0 1; do MMJ_CTA_EMIT=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench_${v}_$RANDOM.json 2>>$O/bench.err; done
