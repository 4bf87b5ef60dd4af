cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_sort.py tests/test_gpu_format.py -q -x 2>&1 | tail -1
for c in 5 2; do timeout 600 python bench.py --config $c --skip-paths --skip-cpals --skip-cpu --steps 2 --e2e-steps 1 > gpurun_out/bq$c.log 2>&1; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bq$c.log') if l.startswith('{')][-1]); print('cfg$c build_ms', d['build_ms'], 'plan', d['plans'])"; done
