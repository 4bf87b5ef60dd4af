cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
timeout 1200 python -m pytest tests/test_gpu_mttkrp.py tests/test_gpu_pull.py tests/test_gpu_cpd.py -q > gpurun_out/t_blk.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/t_blk.log
rm -f gpurun_out/fullsize_parity.jsonl
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -s --durations=0 > gpurun_out/fullsize.log 2>&1; echo "fullsize rc=$?"
tail -8 gpurun_out/fullsize.log
cat gpurun_out/fullsize_parity.jsonl | cut -c1-600
