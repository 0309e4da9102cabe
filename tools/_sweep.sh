python -m pytest tests/test_gpu_twopath.py tests/test_gpu_golden.py tests/test_gpu_apps.py -x -q 2>&1 | tail -1
for v in "MMJ_EMIT_V=2" "MMJ_EMIT_V=3"; do env $v python tools/bench_configs.py cfg3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v cfg3', d['seconds'])"; done
for v in "MMJ_EMIT_V=3" "MMJ_EMIT_V=2" "MMJ_EMIT_V=3"; do env $v python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],1), {k:round(v['ms'],1) for k,v in d['phases'].items()})"; done
