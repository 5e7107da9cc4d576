cd $GRAFT_REPO_ROOT
timeout 300 python tools/assemble_once.py c5 --hist > gpurun_out/r5_c5_hist.log 2>&1
echo "hist rc=$?" >> gpurun_out/r5_c5_hist.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -c 1 -o gpurun_out/r5_c5tail python tools/assemble_once.py c5 > gpurun_out/r5_ncu_tail.log 2>&1
echo "full rc=$?" >> gpurun_out/r5_ncu_tail.log
