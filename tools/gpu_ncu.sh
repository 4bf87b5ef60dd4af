# ncu evidence (run under gpurun; one GPU; each command only after the bench exits 0 without ncu)
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
B="python bench.py --steps 1 --warmup 3 --skip-cpu --skip-cpals --e2e-steps 1"
timeout 900 python bench.py --steps 2 --warmup 3 --skip-cpu --skip-cpals --skip-paths --e2e-steps 1 > gpurun_out/bench_pre_ncu.log 2>&1; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02e_launches_cfg5.csv python bench.py --steps 2 --warmup 3 --skip-cpu --skip-cpals --skip-paths --e2e-steps 1 > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstream_kernel --launch-skip 12 -c 3 -o gpurun_out/r02e_cfg5_mstream -f $B --skip-paths > gpurun_out/ncu_1.log 2>&1; echo "ms rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_stage_kernel --launch-skip 7 -c 3 -o gpurun_out/r02e_cfg5_pull -f $B > gpurun_out/ncu_2.log 2>&1; echo "pull rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:planned_kernel --launch-skip 0 -c 3 -o gpurun_out/r02e_cfg5_alto_order -f $B > gpurun_out/ncu_3.log 2>&1; echo "alto-order rc=$?"
ls -la gpurun_out/*.ncu-rep
