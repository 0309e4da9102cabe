python -m pytest tests/test_gpu_twopath.py tests/test_gpu_golden.py -x -q 2>&1 | tail -1 > gpurun_out/pt.txt
for v in 1 2; do for sch in serial mma_ahead pipelined; do
  MMJ_EMIT_V=$v python bench.py --no-e2e --no-cpu-baseline --steps 3 --schedule $sch 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v$v $sch', round(d['ms_per_step'],1), {k:round(v['ms'],1) for k,v in d['phases'].items()})"
done; done
cat gpurun_out/pt.txt
