set -u
O=gpurun_out/c4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_apps.py tests/test_gpu_fullsize.py -k "ssj or compact or cfg4 or scj" -x -q > $O/tests3.log 2>&1; echo EXIT $? >> $O/tests3.log
timeout 600 python tools/bench_configs.py cfg4 > $O/cfg4c.jsonl 2> $O/cfg4c.err
timeout 300 python tools/_c4prof2.py > $O/c4prof2b.txt 2>&1
