set -u
O=gpurun_out/r3h; mkdir -p $O
for mt in 1 0; do
MMJ_BSI_MATCH=$mt timeout 900 python -m pytest tests/test_gpu_apps.py tests/test_gpu_golden.py -q -p no:cacheprovider -k "bsi" -rf > $O/tests_bsi_m$mt.log 2>&1; echo "EXIT $?" >> $O/tests_bsi_m$mt.log
done
for mt in 1 0 1 0; do
  MMJ_BSI_MATCH=$mt timeout 600 python bench.py --config cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> $O/bench_cfg5_m$mt.json 2>>$O/bench_m$mt.err
done
C5="python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-verify"
MMJ_BSI_MATCH=1 ncu --set full --import-source on --clock-control none -k regex:"k_bsi_answer" -s 3 -c 1 -o $O/full_bsi_answer_match $C5 > $O/bsi_ncu.log 2>&1
MMJ_BSI_MATCH=1 timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "cfg5" -rf > $O/tests_cfg5_m1.log 2>&1; echo "EXIT $?" >> $O/tests_cfg5_m1.log
ls -la $O
