python -m pytest tests/test_gpu_apps.py tests/test_gpu_fullsize.py -x -q -k "star or cfg3" 2>&1 | tail -1
for v in "MMJ_PAIR=1" "MMJ_STAR_CHUNK_BYTES=1073741824"; do env $v python tools/bench_configs.py cfg3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['seconds'], d['light_witnesses'])"; done
