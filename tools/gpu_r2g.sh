# Round-2 (session 4) evidence run: full GPU suite, smoke, bench lines per config, ncu for the blocked kernel.
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo "build rc=$?"
( time timeout 3000 python -m pytest tests -m gpu -q --durations=10 ) > gpurun_out/pytest_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -18 gpurun_out/pytest_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench_cfg5.jsonl 2> gpurun_out/bench_cfg5.err; echo "bench5 rc=$?"; cut -c1-300 gpurun_out/bench_cfg5.jsonl
for c in 1 2 3 4; do
timeout 900 python bench.py --config $c --skip-cpu > gpurun_out/bench_cfg$c.jsonl 2> gpurun_out/bench_cfg$c.err; echo "bench$c rc=$?"; cut -c1-300 gpurun_out/bench_cfg$c.jsonl
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.jsonl 2> gpurun_out/bench_reference.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/bench_reference.jsonl
