cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/diag/jitter_rows.py 32 0.5 > gpurun_out/r49_diag.log 2>&1
timeout 300 python tools/assemble_once.py c5 --reps 3 > gpurun_out/r49_c5.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r49_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r49_t_all.log
