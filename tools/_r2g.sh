set -u
O=gpurun_out/r2g; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/store_lab tools/store_lab.cu && ./tools/store_lab sweep > $O/store_lab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_formats.py tests/test_gpu_apps.py -q -p no:cacheprovider > $O/tests.log 2>&1; echo "EXIT $?" >> $O/tests.log
for i in 1 2; do timeout 600 python bench.py --config cfg5 --no-e2e --no-cpu-baseline > $O/cfg5_lists.$i.json 2>>$O/bench.err; done
C5="python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
$C5 > $O/cfg5_plain.json 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_bsi_answer" -s 3 -c 1 -o $O/bsi_lists2 $C5 > $O/bsi_ncu.log 2>&1
ls -la $O
