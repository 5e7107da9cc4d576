cd $GRAFT_REPO_ROOT
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r28_c5.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r28_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r28_t_all.log
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:tail2d_block -c 1 -o gpurun_out/r28_c5tb python tools/assemble_once.py c5 > gpurun_out/r28_ncu_tb.log 2>&1
