cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
for c in 2 5; do timeout 900 python tools/ab_rawx.py $c > gpurun_out/ab_rawx_$c.log 2>&1; echo "rawx$c rc=$?"; tail -5 gpurun_out/ab_rawx_$c.log; done
