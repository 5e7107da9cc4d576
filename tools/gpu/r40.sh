cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"near_block_kernel" -c 1 -o gpurun_out/r40_near python tools/assemble_once.py c5 --reps 1 > gpurun_out/r40_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cross2d_kernel" -c 1 -o gpurun_out/r40_xgen python tools/assemble_once.py c5 --reps 1 > gpurun_out/r40_ncu2.log 2>&1
