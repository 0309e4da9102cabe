#!/bin/bash
# Round profile capture (run under gpurun from the repo root):
#   tools/profile_round.sh TAG
# GPU tests + smoke, the default bench (full contract) + reference arm, one
# bench line per BASELINE config, then the ncu launch list of the default
# bench and --set full captures of the hot kernels (k_merge_emit at cfg2,
# k_bsi_answer_lists at cfg5, heavy_mma_kernel at cfg3).  Each ncu pass runs
# only after the same command exited 0 without ncu.
set -u
TAG=${1:-rX}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $OUT/gpu_tests.log 2>&1; echo "EXIT $?" >> $OUT/gpu_tests.log
cp gpurun_out/reference_suite.log gpurun_out/checked_cases.log $OUT/ 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "EXIT $?" >> $OUT/smoke.log
python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for c in cfg1 cfg3 cfg4 cfg5; do python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
LL="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-light-work --no-verify"
$LL > $OUT/ll_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_cfg2.csv $LL > $OUT/ll_ncu.log 2>&1
FC="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify --no-light-work --x-limit 65536"
$FC > $OUT/full_plain.json 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"k_merge_emit" -s 8 -c 1 \
      -o $OUT/full_merge_emit $FC > $OUT/full_ncu.log 2>&1
C5="python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
$C5 > $OUT/cfg5_plain.json 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"k_bsi_answer" -s 3 -c 1 -o $OUT/full_bsi_answer $C5 > $OUT/bsi_ncu.log 2>&1
C3="python bench.py --config cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
$C3 > $OUT/cfg3_plain.json 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"heavy_mma_kernel" -s 3 -c 1 -o $OUT/full_heavy_mma $C3 > $OUT/mma_ncu.log 2>&1
ls -la $OUT
