# A/B session (run under gpurun from the repo root).
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_mttkrp.py -m gpu -x -q > gpurun_out/pytest_mttkrp.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_mttkrp.log
AB_FLAGS=4096 timeout 900 python tools/ab_mstream.py 2 0 1024 > gpurun_out/ab2.log 2>&1; echo "ab2 rc=$?"; cat gpurun_out/ab2.log
timeout 600 python bench.py --skip-cpu > gpurun_out/bench2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench2.log | cut -c1-400
AB_FLAGS=4096 timeout 1500 python tools/ab_mstream.py 5 0 1024 > gpurun_out/ab5.log 2>&1; echo "ab5 rc=$?"; cat gpurun_out/ab5.log
