set -u
O=gpurun_out/r2q; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_twopath.py tests/test_gpu_fused.py tests/test_gpu_golden.py tests/test_gpu_apps.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "not cfg5_bsi_eighth" > $O/tests.log 2>&1; echo "EXIT $?" >> $O/tests.log
for i in 1 2; do MMJ_BENCH_DIAG=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work --steps 5 > $O/bench.$i.json 2>>$O/bench.err; done
for c in cfg1 cfg4 cfg3; do MMJ_BENCH_DIAG=1 timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > $O/bench_$c.json 2>>$O/bench.err; done
ls -la $O
