cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/assemble_once.py c5 --reps 3 > gpurun_out/r46_c5.log 2>&1
FRACLAP_TRACE=1 timeout 300 python tools/assemble_once.py c5 --reps 1 > gpurun_out/r46_c5_trace.log 2>&1
