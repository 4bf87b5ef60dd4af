cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
timeout 900 python -m pytest tests/test_gpu_mttkrp.py tests/test_gpu_pull.py tests/test_gpu_sort.py tests/test_gpu_cpd.py -q -x > gpurun_out/t_e.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_e.log
rm -f gpurun_out/fullsize_parity.jsonl
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/t_full.log 2>&1; echo "full rc=$?"; tail -3 gpurun_out/t_full.log; cut -c1-250 gpurun_out/fullsize_parity.jsonl
timeout 600 python tools/ab_delta.py 3 32 16 > gpurun_out/ab_delta_3.log 2>&1; echo "d3 rc=$?"; cat gpurun_out/ab_delta_3.log | tail -6
timeout 600 python tools/ab_delta.py 5 > gpurun_out/ab_delta_5.log 2>&1; echo "d5 rc=$?"; cat gpurun_out/ab_delta_5.log | tail -4
timeout 600 python bench.py --skip-paths --skip-cpals --skip-cpu --steps 5 --e2e-steps 1 > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?"; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_quick.log') if l.startswith('{')][-1]); print('build_ms', d['build_ms'], 'plans', d['plans'], 'value', d['value'], d['roofline']['frac'])"
