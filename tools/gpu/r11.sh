cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r11_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r11_t_all.log
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r11_c5.log 2>&1
FRACLAP_B200_LIB=paper_1708_03912_b200/lib/var/xu3.so timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r11_c5_xu3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r11_c5_launches.csv python tools/assemble_once.py c5 > gpurun_out/r11_ncu_l.log 2>&1
