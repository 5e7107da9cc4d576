cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r8_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r8_t_all.log
timeout 900 python bench.py --steps 3 --warmup 2 --e2e-steps 1 --no-cpu --no-ref-own > gpurun_out/r8_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r8_bench.log
