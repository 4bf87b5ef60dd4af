cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
timeout 900 python -m pytest tests/test_gpu_pull.py -x -q > gpurun_out/pull_tests.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pull_tests.log
timeout 600 python tools/ab_pull.py 2 4 5 > gpurun_out/ab_pull.log 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_pull.log | tail -20
