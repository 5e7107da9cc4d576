cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FRACLAP_TRACE=1 timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r48_c5_trace.log 2>&1
