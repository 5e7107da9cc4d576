cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r4_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r4_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r4_t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r4_smoke.log
timeout 1200 python bench.py > gpurun_out/r4_bench_c5.log 2>&1
echo "bench rc=$?" >> gpurun_out/r4_bench_c5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4_c5_launches.csv python tools/assemble_once.py c5 > gpurun_out/r4_ncu_l.log 2>&1
echo "launch rc=$?" >> gpurun_out/r4_ncu_l.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cross2d -s 1 -c 1 -o gpurun_out/r4_c5cross python tools/assemble_once.py c5 > gpurun_out/r4_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/r4_ncu_full.log
