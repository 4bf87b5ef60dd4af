cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 1200 ncu --set full --clock-control none -k regex:"mstream_kernel" -o gpurun_out/r02e_cfg5_l2pol -f python tools/ncu_l2.py 5 > gpurun_out/ncu_l2.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_l2.log
