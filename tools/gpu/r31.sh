cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FRACLAP_EXACT_RANGE=0 timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r31_c5_off.log 2>&1
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r31_c5_on.log 2>&1
timeout 300 python tools/assemble_once.py c4a --reps 2 > gpurun_out/r31_c4a_on.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r31_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r31_t_all.log
