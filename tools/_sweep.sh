python -m pytest tests/test_gpu_twopath.py tests/test_gpu_golden.py -x -q 2>&1 | tail -1
for v in 1 2; do python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tile8192', round(d['ms_per_step'],1), {k:round(v['ms'],1) for k,v in d['phases'].items()})"; done
