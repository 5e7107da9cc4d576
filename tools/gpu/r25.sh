cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r25_c2_launches.csv python tools/assemble_once.py c2 > gpurun_out/r25_ncu_l.log 2>&1
