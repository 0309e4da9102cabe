set -u
mkdir -p gpurun_out/r2a
nvidia-smi -L > gpurun_out/r2a/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1; echo "SMOKE EXIT $?" >> gpurun_out/r2a/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r2a/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/r2a/gpu_tests.log
timeout 600 python bench.py > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err; echo "EXIT $?" >> gpurun_out/r2a/bench.err
