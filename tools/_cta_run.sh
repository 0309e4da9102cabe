set -u
O=gpurun_out/cta2; mkdir -p $O
for v in 1 0 1; do MMJ_CTA_EMIT=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench_${v}_$RANDOM.json 2>>$O/bench.err; done
