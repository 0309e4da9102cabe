#!/bin/bash
# Heavy-y count (K) sweep on cfg2: the heavy product alone at K = 128..1024
# (tools/mma_lab.py) and the whole step at plans that put K = 128..768 y on
# the tensor-core side; plus the HBM store-shape ceilings (tools/emit_lab.cu).
set -u
OUT=gpurun_out/ksweep
mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/emit_lab tools/emit_lab.cu && timeout 300 /tmp/emit_lab > $OUT/emit_lab.txt 2>&1
for k in 128 256 384 512 640 768 1024; do
  timeout 300 python tools/mma_lab.py 16384 500736 $k >> $OUT/mma_lab.txt 2>&1
done
for p in gpu 1599,1 1082,1 817,1 657,1 544,1; do
  timeout 600 python bench.py --plan $p --no-e2e --no-cpu-baseline > $OUT/bench_$p.json 2> $OUT/bench_$p.err
done
