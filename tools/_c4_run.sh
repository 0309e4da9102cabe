set -u
O=gpurun_out/c4; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_apps.py tests/test_gpu_fullsize.py tests/test_gpu_twopath.py -k "ssj or compact or cfg4 or scj or count" -x -q > $O/tests2.log 2>&1; echo EXIT $? >> $O/tests2.log
timeout 600 python tools/bench_configs.py cfg4 > $O/cfg4b.jsonl 2> $O/cfg4b.err
timeout 300 python tools/_c4prof.py > $O/c4prof.txt 2>&1
