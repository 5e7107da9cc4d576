cd $GRAFT_REPO_ROOT
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r18_c5.log 2>&1
FRACLAP_CROSS2D_UNI_ORDER=heavy timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r18_c5_heavy.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r18_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r18_t_all.log
