set -u
O=gpurun_out/r3i; mkdir -p $O
for lr in 1e10 3e10 1e11 3e11 1e12; do
  MMJ_STAR_MMA_RATE=3.8e15 MMJ_STAR_LIGHT_RATE=$lr timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg3_lr$lr.json 2>$O/bench_lr$lr.err
done
timeout 600 python -m pytest tests/test_gpu_apps.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "ssj or cfg4 or scj" > $O/tests_ssj.log 2>&1; echo "EXIT $?" >> $O/tests_ssj.log
for i in 1 2; do timeout 600 python bench.py --config cfg4 --no-e2e --no-cpu-baseline --steps 5 > $O/bench_cfg4.$i.json 2>>$O/bench4.err; done
ls -la $O
