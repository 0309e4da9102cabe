set -u
O=gpurun_out/r2n; mkdir -p $O
for i in 1 2 3 4; do timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work --steps 5 > $O/bench.$i.json 2>>$O/bench.err; done
timeout 600 python bench.py --config cfg5 --no-e2e --no-cpu-baseline > $O/cfg5.json 2>>$O/bench.err
ls -la $O
