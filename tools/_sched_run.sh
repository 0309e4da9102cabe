set -u
O=gpurun_out/sched; mkdir -p $O
timeout 300 python tools/_c4prof.py > $O/c4prof.txt 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --no-light-work --schedule mma_ahead"
for n in 16 24 32 48; do MMJ_COLOC=0 MMJ_MMA_CTAS=$n timeout 600 $B > $O/ahead_ctas$n.json 2>> $O/err.txt; done
timeout 600 $B > $O/ahead_coloc.json 2>> $O/err.txt
