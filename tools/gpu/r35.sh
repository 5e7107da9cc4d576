cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FRACLAP_TAIL_FOLD_WARP=0 timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r35_c5_warp0.log 2>&1
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r35_c5_warp1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cross2d_uni_kernel -c 1 -o gpurun_out/r35_crossuni python tools/assemble_once.py c5 --reps 1 > gpurun_out/r35_ncu.log 2>&1
