cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 600 python tools/reuse_stats.py 5 > gpurun_out/reuse_stats_cfg5.jsonl 2> gpurun_out/reuse.err; echo "reuse rc=$?"; cat gpurun_out/reuse_stats_cfg5.jsonl
B="python bench.py --steps 1 --warmup 3 --skip-cpu --skip-cpals --e2e-steps 1 --skip-paths"
for c in 3 4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mstream_blk_kernel --launch-skip 8 -c 5 -o gpurun_out/r02e_cfg${c}_mstream_blk -f $B --config $c > gpurun_out/ncu_b$c.log 2>&1; echo "ncu cfg$c rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02e_launches_cfg$c.csv python bench.py --steps 2 --warmup 3 --skip-cpu --skip-cpals --skip-paths --e2e-steps 1 --config $c > gpurun_out/ncu_l$c.log 2>&1; echo "launches cfg$c rc=$?"
done
ls -la gpurun_out/*.ncu-rep
