set -u
O=gpurun_out/prof
rm -rf $O; mkdir -p $O
(timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1; echo EXIT $? >> $O/smoke.log)
(timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo EXIT $? >> $O/gpu_tests.log)
timeout 1800 bash tools/profile_round.sh
