cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
timeout 900 python -m pytest tests/test_gpu_pull.py tests/test_gpu_format.py tests/test_gpu_cpals_cfg5.py -q -x > gpurun_out/t_f.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_f.log
rm -f gpurun_out/fullsize_parity.jsonl
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/t_full.log 2>&1; echo "full rc=$?"; tail -3 gpurun_out/t_full.log; cut -c1-200 gpurun_out/fullsize_parity.jsonl | tail -8
timeout 600 python tools/ab_pull.py 5 3 > gpurun_out/ab_pull.log 2>&1; echo "ab rc=$?"; cut -c1-400 gpurun_out/ab_pull.log
