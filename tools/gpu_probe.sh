# Gather-path probe session (run under gpurun from the repo root).
cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/gather_probe tools/gather_probe.cu -L/usr/local/cuda/lib64/stubs -lcuda
for sk in 0 1; do
  timeout 120 ./gpurun_out/gather_probe ldg $sk; echo "rc=$?"
  timeout 120 ./gpurun_out/gather_probe tma $sk 1; echo "rc=$?"
done
timeout 120 ./gpurun_out/gather_probe tma 0 4; echo "rc=$?"
rm -f gpurun_out/gather_probe
