cd $GRAFT_REPO_ROOT
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:tail2d_block -c 1 -o gpurun_out/r17_sq128tb python tools/assemble_once.py --square 128 --s 0.5 > gpurun_out/r17_ncu.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:cross2d_uni -c 1 -o gpurun_out/r17_sq128xu python tools/assemble_once.py --square 128 --s 0.5 > gpurun_out/r17_ncu2.log 2>&1
