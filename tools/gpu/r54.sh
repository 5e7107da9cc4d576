cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FRACLAP_CROSS2D_UNI=0 timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r54_c5_uni0.log 2>&1
