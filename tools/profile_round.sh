#!/bin/bash
# Round profile capture (run under gpurun from the repo root):
#   bench (full contract) + reference arm + per-config lines, then the ncu
#   launch list of the default bench and one --set full capture of the hot
#   kernels at 4096-row chunks.  Each ncu pass runs only after the same
#   command exited 0 without ncu.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err || exit 1
python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
python tools/bench_configs.py > $OUT/configs.jsonl 2> $OUT/configs.err
LL="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-light-work"
$LL > $OUT/ll_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $LL > $OUT/ll_ncu.log 2>&1
FC="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --chunk-rows 4096 --x-limit 16384"
$FC > $OUT/full_plain.json 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"k_merge_emit|heavy_mma_kernel" -s 4 -c 2 \
      -o $OUT/full_mma_merge_emit $FC > $OUT/full_ncu.log 2>&1
ls -la $OUT
