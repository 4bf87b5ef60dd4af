cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
ALTO_MS_RANKS=16,32 timeout 900 python tools/ab_mstream.py 3 0 1024 2>&1 | tail -4
