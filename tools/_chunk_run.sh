set -u
O=gpurun_out/chunk; mkdir -p $O
for c in 20480 16384 24576 16384 20480; do timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work --chunk-rows $c > $O/bench_${c}_$RANDOM.json 2>>$O/bench.err; done
