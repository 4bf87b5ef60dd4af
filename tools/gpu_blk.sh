cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
timeout 1500 python -m pytest tests/test_gpu_mttkrp.py tests/test_gpu_cpd.py tests/test_gpu_smoke.py tests/test_cli.py -q > gpurun_out/t_blk.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/t_blk.log
rm -f gpurun_out/fullsize_parity.jsonl
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s > gpurun_out/fullsize.log 2>&1; echo "fullsize rc=$?"
tail -4 gpurun_out/fullsize.log
python - <<'P'
import json
for l in open('gpurun_out/fullsize_parity.jsonl'):
    d=json.loads(l); print(d['cfg'], d['mode'], {k: float('%.2e'%v) for k,v in d['rel_err'].items()})
P
timeout 900 python bench.py --config 5 --skip-cpals --skip-cpu --steps 3 --e2e-steps 1 > gpurun_out/bq5.log 2>&1; echo "bench5 rc=$?"; python -c "
import json; d=json.loads([l for l in open('gpurun_out/bq5.log') if l.startswith('{')][-1]); print({k:(v['per_mode_ms'],v.get('roofline_frac')) for k,v in d['paths'].items()})"
