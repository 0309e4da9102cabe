set -u
O=gpurun_out/r2e; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/store_lab tools/store_lab.cu && ./tools/store_lab > $O/store_lab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_apps.py -q -x -p no:cacheprovider -k bsi > $O/tests.log 2>&1; echo "EXIT $?" >> $O/tests.log
for f in lists records lists; do timeout 600 python bench.py --config cfg5 --bsi-form $f --no-e2e --no-cpu-baseline > $O/cfg5_$f.$RANDOM.json 2>>$O/bench.err; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k cfg5_bsi_full > $O/tests_full.log 2>&1; echo "EXIT $?" >> $O/tests_full.log
ls -la $O
