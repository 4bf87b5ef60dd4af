# One GPU session of round measurements (run under gpurun from the repo root):
#   gpurun --timeout 3600 -- 'bash tools/gpu_round.sh'
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -C oracle >/dev/null
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 2000 gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --skip-cpu --skip-cpals --skip-paths --e2e-steps 1 > gpurun_out/ncu_l.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstream_kernel --launch-skip 12 -c 3 \
  -o gpurun_out/cfg5_mstream -f python bench.py --steps 1 --warmup 3 --skip-cpu --skip-cpals --skip-paths --e2e-steps 1 \
  > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
