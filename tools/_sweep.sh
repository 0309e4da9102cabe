python -m pytest tests/test_gpu_apps.py tests/test_gpu_twopath.py tests/test_gpu_golden.py -x -q 2>&1 | tail -1
MMJ_CFG4_PLANS="194,1" python tools/bench_configs.py cfg4 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(d['plan'], round(d['seconds']*1e3,2), d['phase_ms'])"
