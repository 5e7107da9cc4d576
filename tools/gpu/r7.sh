cd $GRAFT_REPO_ROOT
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r7_c5.log 2>&1
echo "rc=$?" >> gpurun_out/r7_c5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r7_c5_launches.csv python tools/assemble_once.py c5 > gpurun_out/r7_ncu_l.log 2>&1
echo "launch rc=$?" >> gpurun_out/r7_ncu_l.log
