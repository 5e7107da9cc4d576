cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/dmma_probe tools/dmma_probe.cu && timeout 120 gpurun_out/dmma_probe > gpurun_out/r33_dmma.log 2>&1
rm -f gpurun_out/dmma_probe
