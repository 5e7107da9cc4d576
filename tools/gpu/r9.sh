cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r9_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r9_t_all.log
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r9_c5.log 2>&1
echo "rc=$?" >> gpurun_out/r9_c5.log
FRACLAP_CROSS2D_UNI=0 timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r9_c5_nouni.log 2>&1
echo "rc=$?" >> gpurun_out/r9_c5_nouni.log
