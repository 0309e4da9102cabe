set -u
O=gpurun_out/eng; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_twopath.py tests/test_gpu_fused.py -x -q > $O/tests.log 2>&1; echo EXIT $? >> $O/tests.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench.json 2> $O/bench.err
timeout 900 python tools/shard_balance.py > $O/shard_balance.jsonl 2> $O/shard.err
