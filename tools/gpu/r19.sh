cd $GRAFT_REPO_ROOT
timeout 1200 python bench.py > gpurun_out/r19_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r19_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r19_c5_launches.csv python tools/assemble_once.py c5 > gpurun_out/r19_ncu_l.log 2>&1
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:tail2d_block -c 1 -o gpurun_out/r19_c5tb python tools/assemble_once.py c5 > gpurun_out/r19_ncu_tb.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cross2d_uni -c 1 -o gpurun_out/r19_c5xu python tools/assemble_once.py c5 > gpurun_out/r19_ncu_xu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"tail_kernel<2" -c 1 -o gpurun_out/r19_c5tk python tools/assemble_once.py c5 > gpurun_out/r19_ncu_tk.log 2>&1
