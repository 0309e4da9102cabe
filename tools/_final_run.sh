set -u
O=gpurun_out/r1f; mkdir -p $O
(timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo EXIT $? >> $O/gpu_tests.log)
timeout 900 python tools/bench_configs.py > $O/configs.jsonl 2> $O/configs.err
timeout 300 python -c "
import cProfile, pstats, sys
sys.argv=['x']
exec(open('tools/_c4prof.py').read().replace('for i in range(5):', 'pr = cProfile.Profile()\nfor i in range(5):\n    if i == 2: pr.enable()').replace('print(tot)', 'pr.disable(); pstats.Stats(pr).sort_stats(\"cumtime\").print_stats(25)'))
" > $O/c4_cprofile.txt 2>&1
timeout 900 python tools/bench_configs.py cfg5 > $O/cfg5_plain.jsonl 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/cfg5_launches.csv python tools/bench_configs.py cfg5 > $O/cfg5_ncu.log 2>&1
ls -la $O
