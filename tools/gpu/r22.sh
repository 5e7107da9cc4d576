cd $GRAFT_REPO_ROOT
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:'^tail_kernel$' -c 1 -o gpurun_out/r22_c5tk python tools/assemble_once.py c5 > gpurun_out/r22_ncu_tk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^near_block_kernel$' -c 1 -o gpurun_out/r22_c5near python tools/assemble_once.py c5 > gpurun_out/r22_ncu_near.log 2>&1
