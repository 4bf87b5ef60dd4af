cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
timeout 900 python -m pytest tests/test_gpu_mttkrp.py tests/test_gpu_sort.py tests/test_gpu_format.py tests/test_coo.py -q -x > gpurun_out/t_c.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_c.log
timeout 600 python bench.py --skip-paths --skip-cpals --skip-cpu --steps 3 --e2e-steps 1 > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?"; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_quick.log') if l.startswith('{')][-1]); print('build_ms', d['build_ms'], 'plans', d['plans'], 'value', d['value'])"
timeout 900 ncu --set full --clock-control none -k regex:radix_scatter --launch-skip 0 -c 2 -o gpurun_out/r02b_cfg5_sort -f python bench.py --skip-paths --skip-cpals --skip-cpu --steps 1 --e2e-steps 1 > gpurun_out/ncu_s.log 2>&1; echo "ncu rc=$?"
timeout 900 python tools/rank_sweep.py 2 > gpurun_out/rank_sweep_2.log 2>&1; echo "sweep rc=$?"; tail -4 gpurun_out/rank_sweep_2.log | cut -c1-600
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_workload.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/sanitize_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_workload.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -5 gpurun_out/sanitize_racecheck.log
