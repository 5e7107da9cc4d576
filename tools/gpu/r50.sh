cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "jitter or row_block or shard_rows or order_ties" > gpurun_out/r50_t.log 2>&1
echo "rc=$?" >> gpurun_out/r50_t.log
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r50_c5.log 2>&1
