cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r37_c5.log 2>&1
FRACLAP_TAIL_FOLD_WARP=0 timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r37_c5_w0.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "2d or block or large or row_block or c3 or sampled or c5" > gpurun_out/r37_t.log 2>&1
echo "rc=$?" >> gpurun_out/r37_t.log
