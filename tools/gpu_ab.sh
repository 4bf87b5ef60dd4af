# A/B session (run under gpurun from the repo root).
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_mttkrp.py -m gpu -x -q > gpurun_out/pytest_mttkrp.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_mttkrp.log
for pb in 0 1000000 67108864; do
ALTO_MS_PAIR_BYTES=$pb timeout 900 python tools/ab_mstream.py 4 0 1024 > gpurun_out/ab4_$pb.log 2>&1; echo "ab4 pairbytes=$pb rc=$?"; grep mode gpurun_out/ab4_$pb.log | cut -c1-120
done
timeout 600 python bench.py --config 4 --steps 10 > gpurun_out/bench4.log 2>&1; echo "bench4 rc=$?"; tail -1 gpurun_out/bench4.log | cut -c1-300
ALTO_MS_PAIR_BYTES=0 timeout 600 python bench.py --config 4 --steps 10 --skip-cpu > gpurun_out/bench4_nopair.log 2>&1; echo "bench4 nopair rc=$?"; tail -1 gpurun_out/bench4_nopair.log | cut -c1-300
