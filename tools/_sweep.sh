python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in "MMJ_COUNT16=1" "MMJ_COUNT16=0"; do env $v MMJ_CFG4_PLANS="194,1" python tools/bench_configs.py cfg4 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('$v', d['plan'], round(d['seconds']*1e3,2), d['phase_ms'])"; done
