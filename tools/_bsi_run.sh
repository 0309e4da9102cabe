set -u
O=gpurun_out/bsi; mkdir -p $O
(timeout 900 python -m pytest tests/test_gpu_apps.py tests/test_gpu_fullsize.py tests/test_gpu_ingest.py -k "bsi or cfg5 or ingest or compact or ssj" -x -q > $O/tests.log 2>&1; echo EXIT $? >> $O/tests.log)
timeout 600 python tools/bench_configs.py cfg5 > $O/cfg5.jsonl 2> $O/cfg5.err
