cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r02e_launches_cfg5_cpals.csv python bench.py --steps 1 --warmup 3 --skip-cpu --skip-paths --e2e-steps 1 > gpurun_out/ncu_lc.log 2>&1; echo "launches rc=$?"
