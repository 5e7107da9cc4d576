cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cross2d_uni_kernel" -c 1 -o gpurun_out/r60_xuni python tools/assemble_once.py c5 --reps 1 > gpurun_out/r60_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"mv_rows_kernel|matvec" --launch-skip 2 -c 1 -o gpurun_out/r60_mv python bench.py --steps 1 --warmup 0 --no-cpu --no-extra --no-e2e --no-cg --matvecs 3 > gpurun_out/r60_ncu2.log 2>&1
