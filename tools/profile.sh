#!/bin/bash
# Usage (on the GPU box, via gpurun):  bash tools/profile.sh <config> [tag] [kernel-regex]
# 1) plain run (must exit 0), 2) ncu launch list, 3) plain run again, 4) ncu --set full on the
# top kernels.  Outputs land in gpurun_out/.
CFG=${1:-c3}; TAG=${2:-$CFG}; KRE=${3:-"cross_tile_kernel|tail_kernel"}
CMD="python bench.py --config $CFG --steps 1 --warmup 0 --no-cg --no-cpu --no-near --matvecs 2"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_l_$TAG.log 2>&1
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
tail -n 2 gpurun_out/ncu_l_$TAG.log gpurun_out/ncu_full_$TAG.log
