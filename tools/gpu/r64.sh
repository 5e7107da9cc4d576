cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/diag/irregular_rows.py graded2d:64:0.3 jitter2d:64:0.5 graded2d:72:0.5 jitter2d:56:0.3 square2d:64:0.3 > gpurun_out/r64_diag.log 2>&1
