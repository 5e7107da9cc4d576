cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "block_paths" > gpurun_out/r57_t.log 2>&1
echo "rc=$?" >> gpurun_out/r57_t.log
