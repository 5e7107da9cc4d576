cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tail_kernel|near_block_kernel" -c 2 -o gpurun_out/r38_tw_near python tools/assemble_once.py c5 --reps 1 > gpurun_out/r38_ncu.log 2>&1
