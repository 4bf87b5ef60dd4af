cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
make -C oracle >/dev/null
timeout 600 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/dist.log 2>&1; echo "dist rc=$?"; tail -5 gpurun_out/dist.log
timeout 900 python bench.py > gpurun_out/bench_cfg5.log 2>&1; echo "bench rc=$?"; tail -c 6000 gpurun_out/bench_cfg5.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 1500 gpurun_out/bench_ref.log
timeout 900 python tools/sim_shards.py 5 > gpurun_out/sim_shards.log 2>&1; echo "sim rc=$?"; tail -c 4000 gpurun_out/sim_shards.log
