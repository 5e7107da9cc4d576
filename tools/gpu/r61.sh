cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r61_base.log 2>&1
export FRACLAP_B200_LIB=paper_1708_03912_b200/lib/var/coldof.so
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r61_coldof.log 2>&1
timeout 300 python tools/assemble_once.py c4a --reps 2 > gpurun_out/r61_coldof_c4a.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "2d or block or large or row_block or c3 or sampled or c5 or jitter or irregular" > gpurun_out/r61_t.log 2>&1
echo "rc=$?" >> gpurun_out/r61_t.log
