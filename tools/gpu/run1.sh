cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_solve.py -x -q > gpurun_out/r1_t_solve.log 2>&1
echo "solve rc=$?" >> gpurun_out/r1_t_solve.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r1_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r1_t_all.log
timeout 900 python bench.py --steps 2 --warmup 1 --e2e-steps 1 > gpurun_out/r1_bench_c5.log 2>&1
echo "bench rc=$?" >> gpurun_out/r1_bench_c5.log
