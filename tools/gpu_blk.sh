cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:onesweep_pass --launch-skip 2 -c 2 -o gpurun_out/r02e_cfg5_sort -f python bench.py --skip-paths --skip-cpals --skip-cpu --steps 1 --e2e-steps 1 > gpurun_out/ncu_s.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_s.log
