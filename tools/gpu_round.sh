# One GPU session of measurements (run under gpurun from the repo root).
set -x
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstream_kernel --launch-skip 6 -c 3 -o gpurun_out/mstream_full -f python bench.py --steps 3 --warmup 3 --skip-cpu --skip-cpals > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
for c in 1 3 4; do timeout 900 python bench.py --config $c --steps 10 > gpurun_out/bench_cfg$c.log 2>&1; echo "cfg$c rc=$?"; tail -1 gpurun_out/bench_cfg$c.log | cut -c1-300; done
timeout 1800 python bench.py --config 5 --steps 5 --cpu-sample 1000000 > gpurun_out/bench_cfg5.log 2>&1; echo "cfg5 rc=$?"; tail -1 gpurun_out/bench_cfg5.log | cut -c1-300
