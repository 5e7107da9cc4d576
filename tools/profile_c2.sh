#!/bin/bash
# c2 (headline) profile set on the GPU box: default bench line, launch list, ncu --set full of the
# tail, cross and matvec kernels (each ncu command after the same command exited 0 without ncu).
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.log 2>&1 || echo "bench failed"
CMD="python bench.py --config c2 --steps 1 --warmup 1 --no-cg --no-cpu --no-near --matvecs 3"
$CMD > gpurun_out/plain_c2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
      $CMD > gpurun_out/ncu_l_c2.log 2>&1
CMD0="python bench.py --config c2 --steps 1 --warmup 0 --no-cg --no-cpu --no-near --matvecs 3"
$CMD0 > gpurun_out/plain_f_c2.log 2>&1 && {
  ncu --set full --clock-control none --import-source on -k regex:"tail1d_kernel" -c 1 \
      -o gpurun_out/prof_c2tail $CMD0 > gpurun_out/ncu_full_c2tail.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"cross1d_tile" -c 1 \
      -o gpurun_out/prof_c2cross $CMD0 > gpurun_out/ncu_full_c2cross.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"matvec" --launch-skip 1 -c 1 \
      -o gpurun_out/prof_c2mv $CMD0 > gpurun_out/ncu_full_c2mv.log 2>&1
}
ls gpurun_out/*.ncu-rep
