cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref2.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/bench2.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_ref2.log | cut -c1-400
