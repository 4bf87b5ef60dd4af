# Gather-path probe session (run under gpurun from the repo root).
cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/gather_probe tools/gather_probe.cu -L/usr/local/cuda/lib64/stubs -lcuda
for sk in 0 1; do
  for v in ldg tex4 tex2 tex1; do
  timeout 120 ./gpurun_out/gather_probe $v $sk; echo "rc=$?"
  done
done
for rows in 200000 1000000 20000000 40000000; do timeout 300 ./gpurun_out/gather_probe ldg 0 1 $rows; done
rm -f gpurun_out/gather_probe
