for pl in 3190,1 1500,1 800,1 400,1; do
  python bench.py --no-e2e --no-cpu-baseline --steps 3 --plan $pl --schedule serial 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$pl serial', d['ms_per_step'], d['config']['k_heavy'], d['config']['light_intermediate'], {k:round(v['ms'],1) for k,v in d['phases'].items()})"
done
