set -u
O=gpurun_out/r2f; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/store_lab tools/store_lab.cu && ./tools/store_lab > $O/store_lab.txt 2>&1
for tw in 8192 4096 2048 8192 4096; do MMJ_FUSE_TW=$tw timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench_tw$tw.$RANDOM.json 2>>$O/bench.err; done
C5="python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
$C5 > $O/cfg5_plain.json 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_bsi_answer" -s 3 -c 1 -o $O/bsi_lists $C5 > $O/bsi_ncu.log 2>&1
ls -la $O
