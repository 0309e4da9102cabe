set -u
O=gpurun_out/r2c; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/emit_lab tools/emit_lab.cu && (./tools/emit_lab 0.49 > $O/emit_lab_049.txt 2>&1; ./tools/emit_lab 1.0 > $O/emit_lab_100.txt 2>&1)
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_twopath.py tests/test_gpu_golden.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "EXIT $?" >> $O/tests.log
for v in 1 0 1 0; do MMJ_EMIT_RR=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-light-work > $O/bench_rr$v.$RANDOM.json 2>>$O/bench.err; done
for v in 1 0; do MMJ_EMIT_RR=$v timeout 600 python bench.py --config cfg3 --no-e2e --no-cpu-baseline > $O/cfg3_rr$v.json 2>>$O/bench.err; done
ls -la $O
