# ncu evidence for round 2 (run under gpurun; one GPU; each command only after the bench exits 0 without ncu)
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
B="python bench.py --steps 1 --warmup 3 --skip-cpu --skip-cpals --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_cfg5.csv python bench.py --steps 2 --warmup 3 --skip-cpu --skip-cpals --skip-paths --e2e-steps 1 > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstream_kernel --launch-skip 12 -c 3 -o gpurun_out/r02_cfg5_mstream -f $B --skip-paths > gpurun_out/ncu_1.log 2>&1; echo "ms rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pull_stage_kernel --launch-skip 7 -c 3 -o gpurun_out/r02_cfg5_pull -f $B > gpurun_out/ncu_2.log 2>&1; echo "pull rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:radix --launch-skip 0 -c 6 -o gpurun_out/r02_cfg5_sort -f $B --skip-paths > gpurun_out/ncu_3.log 2>&1; echo "sort rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstream_kernel --launch-skip 15 -c 5 -o gpurun_out/r02_cfg4_mstream -f $B --skip-paths --config 4 > gpurun_out/ncu_4.log 2>&1; echo "cfg4 rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:cpd_update --launch-skip 6 -c 3 -o gpurun_out/r02_cfg5_cpd_update -f python bench.py --steps 1 --warmup 3 --skip-cpu --skip-paths --e2e-steps 1 > gpurun_out/ncu_5.log 2>&1; echo "cpd rc=$?"
ls -la gpurun_out/*.ncu-rep
