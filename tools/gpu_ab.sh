cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_mttkrp.py -q -x -k pinned 2>&1 | grep -E "Error|error|assert|^E " | head -20
