cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tail2d_block_kernel" -c 1 -o gpurun_out/r39_tb python tools/assemble_once.py c5 --reps 1 > gpurun_out/r39_ncu.log 2>&1
