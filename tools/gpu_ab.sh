cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --skip-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], [p['kernel_ms'] for p in d['roofline']['per_mode']], d['cpals_ms_per_iter'])"
