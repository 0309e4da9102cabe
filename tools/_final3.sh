set -u
O=gpurun_out/fin3; mkdir -p $O
(timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1; echo EXIT $? >> $O/smoke.log)
(timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo EXIT $? >> $O/gpu_tests.log)
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
LL="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-light-work"
$LL > $O/ll_plain.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $LL > $O/ll_ncu.log 2>&1
FC="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --chunk-rows 4096 --x-limit 16384"
$FC > $O/full_plain.json 2>&1 && ncu --set full --import-source on --clock-control none -k regex:"k_merge_emit" -s 2 -c 1 -o $O/full_merge_emit $FC > $O/full_ncu.log 2>&1
