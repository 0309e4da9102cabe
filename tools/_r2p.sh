set -u
O=gpurun_out/r2p; mkdir -p $O
for i in 1 2; do MMJ_BENCH_DIAG=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work --no-verify --steps 5 > $O/bench.$i.json 2>>$O/bench.err; done
ls -la $O
