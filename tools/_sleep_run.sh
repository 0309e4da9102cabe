set -u
O=gpurun_out/sleep; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_golden.py -x -q > $O/tests.log 2>&1; echo EXIT $? >> $O/tests.log
B="python bench.py --no-e2e --no-cpu-baseline --no-light-work"
timeout 600 $B > $O/b128_a.json 2>>$O/err.txt
for ns in 0 512 128; do
  MMJ_NVCC_EXTRA="-DMMJ_LOOKBACK_SLEEP_NS=$ns" python -m paper_2002_12459_b200.build --force >> $O/build.txt 2>&1
  timeout 600 $B > $O/b${ns}_b.json 2>>$O/err.txt
done
