cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_cpd.py tests/test_cli.py -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python tools/prof_cpals.py 2 2>&1 | tail -1
timeout 900 python tools/prof_cpals.py 4 2>&1 | tail -1
