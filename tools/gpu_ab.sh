cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_cpd.py tests/test_gpu_dist.py -x -q 2>&1 | tail -3
timeout 600 python tools/prof_cpals.py 3 2>&1 | tail -1
