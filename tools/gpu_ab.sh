cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_mttkrp.py -q -x 2>&1 | tail -1
timeout 600 python tools/ab_mstream.py 2 0 1024 2>&1 | tail -3
timeout 900 python tools/ab_mstream.py 5 0 1024 2>&1 | tail -3
