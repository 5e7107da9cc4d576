cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/diag/jitter_rows.py 32 0.5 > gpurun_out/r45_diag.log 2>&1
timeout 900 python tools/diag/jitter_rows.py 40 0.75 >> gpurun_out/r45_diag.log 2>&1
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r45_c5.log 2>&1
timeout 300 python tools/assemble_once.py c3 --reps 1 > gpurun_out/r45_c3.log 2>&1
