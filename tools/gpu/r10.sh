cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r10_c5_launches.csv python tools/assemble_once.py c5 > gpurun_out/r10_ncu_l.log 2>&1
echo "launch rc=$?" >> gpurun_out/r10_ncu_l.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:cross2d_uni -c 1 -o gpurun_out/r10_c5uni python tools/assemble_once.py c5 > gpurun_out/r10_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/r10_ncu_full.log
