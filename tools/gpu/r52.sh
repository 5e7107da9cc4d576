cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r52_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r52_t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r52_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r52_smoke.log
timeout 1500 python bench.py > gpurun_out/r52_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r52_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r52_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/r52_ref.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r52_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-extra --no-e2e --no-cg --matvecs 3 > gpurun_out/r52_ncu_l.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tail2d_block_kernel" -c 1 -o gpurun_out/r52_tb python tools/assemble_once.py c5 --reps 1 > gpurun_out/r52_ncu2.log 2>&1
