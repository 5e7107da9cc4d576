cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r62_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r62_t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r62_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r62_smoke.log
timeout 1500 python bench.py > gpurun_out/r62_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r62_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r62_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/r62_ref.log
