cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/assemble_once.py c5 --reps 3 > gpurun_out/r53_c5.log 2>&1
timeout 300 python tools/assemble_once.py c4a --reps 2 > gpurun_out/r53_c4a.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r53_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r53_t_all.log
