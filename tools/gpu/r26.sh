cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r26_t_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r26_t_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r26_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r26_smoke.log
timeout 1200 python bench.py > gpurun_out/r26_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r26_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r26_c5_launches.csv python tools/assemble_once.py c5 > gpurun_out/r26_ncu_l.log 2>&1
