cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
timeout 900 python -m pytest tests/test_gpu_mttkrp.py -q -x > gpurun_out/mttkrp_tests.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/mttkrp_tests.log
for c in 5 2 4 3; do timeout 600 python tools/ab_cold.py $c 0 16 32 64 96 > gpurun_out/ab_cold_$c.log 2>&1; echo "cfg$c rc=$?"; cat gpurun_out/ab_cold_$c.log | tail -6; done
