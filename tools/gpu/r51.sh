cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/diag/irregular_rows.py > gpurun_out/r51_diag.log 2>&1
