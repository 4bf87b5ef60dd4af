cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
timeout 900 python -m pytest tests/test_gpu_mttkrp.py -q -x > gpurun_out/t_d.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_d.log
timeout 600 python tools/ab_delta.py 5 > gpurun_out/ab_delta_5.log 2>&1; echo "d5 rc=$?"; cat gpurun_out/ab_delta_5.log | tail -4
timeout 600 python tools/ab_delta.py 3 32 16 > gpurun_out/ab_delta_3.log 2>&1; echo "d3 rc=$?"; cat gpurun_out/ab_delta_3.log | tail -6
timeout 900 python tools/rank_sweep.py 2 > gpurun_out/rank_sweep_2.log 2>&1; echo "sweep rc=$?"; tail -4 gpurun_out/rank_sweep_2.log | cut -c1-700
