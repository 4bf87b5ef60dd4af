cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
rm -f gpurun_out/fullsize_parity.jsonl
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -s --durations=0 > gpurun_out/fullsize.log 2>&1; echo "rc=$?"
tail -30 gpurun_out/fullsize.log
cat gpurun_out/fullsize_parity.jsonl
