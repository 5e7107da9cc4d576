cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "row_block or small_full or c1_ or c3 or shard_rows_bitwise or sampled" > gpurun_out/r2_t_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/r2_t_parity.log
timeout 600 python -m pytest tests/test_gpu_solve.py -x -q > gpurun_out/r2_t_solve.log 2>&1
echo "solve rc=$?" >> gpurun_out/r2_t_solve.log
timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu > gpurun_out/r2_bench_c5.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench_c5.log
