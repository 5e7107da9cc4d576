cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "jitter or block_paths or kernel_power" > gpurun_out/r44_t.log 2>&1
echo "rc=$?" >> gpurun_out/r44_t.log
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r44_c5.log 2>&1
