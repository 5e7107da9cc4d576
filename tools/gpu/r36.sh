cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r36_c5_base.log 2>&1
FRACLAP_B200_LIB=paper_1708_03912_b200/lib/var/xu3.so timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r36_c5_xu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel -c 1 -o gpurun_out/r36_tailwarp python tools/assemble_once.py c5 --reps 1 > gpurun_out/r36_ncu.log 2>&1
