cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
rm -f gpurun_out/fullsize_parity.jsonl gpurun_out/cfg5_cpals_parity.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py --deselect tests/test_gpu_cpals_cfg5.py --deselect tests/test_gpu_reference_suite.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_cpals_cfg5.py -q --durations=0 > gpurun_out/fullsize.log 2>&1; echo "full rc=$?"; tail -25 gpurun_out/fullsize.log
cat gpurun_out/fullsize_parity.jsonl | cut -c1-330; cat gpurun_out/cfg5_cpals_parity.jsonl | cut -c1-200
timeout 900 python -m pytest tests/test_gpu_reference_suite.py -q > gpurun_out/refsuite.log 2>&1; echo "ref rc=$?"; tail -30 gpurun_out/refsuite.log; tail -40 gpurun_out/reference_suite.log
