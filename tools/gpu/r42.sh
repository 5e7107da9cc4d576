cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/assemble_once.py c2 --reps 5 > gpurun_out/r42_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"cross1d_tile_kernel|tail1d_kernel" --launch-skip 4 -c 2 -o gpurun_out/r42_c2 python tools/assemble_once.py c2 --reps 3 > gpurun_out/r42_ncu.log 2>&1
