cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_smoke.py tests/test_gpu_sort.py tests/test_gpu_layout.py tests/test_gpu_format.py tests/test_coo.py tests/test_gpu_mttkrp.py -q > gpurun_out/t_s.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_s.log
for ot in 512 256; do
for c in 5 2; do ALTO_SORT_OT=$ot timeout 600 python bench.py --config $c --skip-paths --skip-cpals --skip-cpu --steps 3 --e2e-steps 1 > gpurun_out/bq$c.log 2>&1; echo "ot=$ot bench$c rc=$?"; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bq$c.log') if l.startswith('{')][-1]); print('cfg$c build_ms', d['build_ms'], 'plans', d['plans'], 'value', d['value'], d['roofline']['frac'])"; done
done
