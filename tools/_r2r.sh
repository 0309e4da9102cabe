set -u
O=gpurun_out/r2r; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_apps.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "ssj or cfg4 or scj" > $O/tests.log 2>&1; echo "EXIT $?" >> $O/tests.log
for i in 1 2; do timeout 600 python bench.py --config cfg4 --no-e2e --no-cpu-baseline --steps 5 > $O/bench_cfg4.$i.json 2>>$O/bench.err; done
ls -la $O
