cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_solve.py tests/test_gpu_parity.py -x -q -k "lockstep or tie or ties or nccl or x0 or split" > gpurun_out/r3_t.log 2>&1
echo "t rc=$?" >> gpurun_out/r3_t.log
timeout 300 python tools/assemble_once.py c5 --hist > gpurun_out/r3_c5_hist.log 2>&1
echo "hist rc=$?" >> gpurun_out/r3_c5_hist.log
timeout 300 python tools/assemble_once.py c5 > gpurun_out/r3_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_c5_launches.csv python tools/assemble_once.py c5 > gpurun_out/r3_ncu_l.log 2>&1
echo "launch rc=$?" >> gpurun_out/r3_ncu_l.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cross2d_kernel -s 1 -c 1 -o gpurun_out/r3_c5cross python tools/assemble_once.py c5 > gpurun_out/r3_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/r3_ncu_full.log
