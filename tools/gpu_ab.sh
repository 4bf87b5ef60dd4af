cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_container.py tests/test_gpu_mttkrp.py -x -q 2>&1 | tail -2
timeout 600 python tools/bench_container.py 2 2>&1 | tail -1
timeout 600 python tools/ab_mstream.py 2 0 1024 2>&1 | tail -3
