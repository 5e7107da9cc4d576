cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r47_launches.csv python tools/assemble_once.py c5 --reps 1 > gpurun_out/r47_ncu_l.log 2>&1
