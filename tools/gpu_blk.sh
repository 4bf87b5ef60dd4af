cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
timeout 1200 python -m pytest tests/test_gpu_sort.py tests/test_gpu_layout.py tests/test_gpu_format.py tests/test_coo.py tests/test_gpu_mttkrp.py tests/test_gpu_pull.py tests/test_container.py -q -x > gpurun_out/t_s.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_s.log
for c in 5 2 3 4; do timeout 600 python bench.py --config $c --skip-paths --skip-cpals --skip-cpu --steps 3 --e2e-steps 1 > gpurun_out/bq$c.log 2>&1; echo "bench$c rc=$?"; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bq$c.log') if l.startswith('{')][-1]); print('cfg$c build_ms', d['build_ms'], 'plans', d['plans'], 'value', d['value'], d['roofline']['frac'])"; done
