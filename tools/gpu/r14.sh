cd $GRAFT_REPO_ROOT
timeout 300 python tools/assemble_once.py c5 --reps 2 > gpurun_out/r14_c5.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "small or row_block or c3 or sampled or full_c5 or block_paths or irregular or tiny or deterministic" > gpurun_out/r14_t.log 2>&1
echo "t rc=$?" >> gpurun_out/r14_t.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:near_block -c 1 -o gpurun_out/r14_c5near python tools/assemble_once.py c5 > gpurun_out/r14_ncu_near.log 2>&1
