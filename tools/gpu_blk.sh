cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
for c in 2 5 3 4; do timeout 900 python tools/ab_secondary.py $c > gpurun_out/ab_sec_$c.log 2>&1; echo "sec$c rc=$?"; tail -4 gpurun_out/ab_sec_$c.log | cut -c1-400; done
