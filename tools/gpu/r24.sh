cd $GRAFT_REPO_ROOT
timeout 300 python tools/assemble_once.py c2 --reps 5 > gpurun_out/r24_c2.log 2>&1
FRACLAP_TAIL1D=warp timeout 300 python tools/assemble_once.py c2 --reps 5 > gpurun_out/r24_c2_warp.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r24_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r24_t_all.log
