#!/bin/bash
# Round profile set (GPU box): launch lists + ncu --set full of the top kernels per config.
# Every ncu command follows a plain run of the same command that exited 0.
set -u
mkdir -p gpurun_out
run() {   # run <tag> <config> [extra bench args]
  local TAG=$1 CFG=$2; shift 2
  local CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cg --no-cpu --no-near --matvecs 3 $*"
  $CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run $TAG failed"; return 1; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
      $CMD > gpurun_out/ncu_l_$TAG.log 2>&1
}
full() {  # full <tag> <config> <kernel-regex> <skip> <count>
  local TAG=$1 CFG=$2 KRE=$3 SKIP=$4 CNT=$5
  local CMD="python bench.py --config $CFG --steps 1 --warmup 0 --no-cg --no-cpu --no-near --matvecs 3"
  $CMD > gpurun_out/plain_f_$TAG.log 2>&1 || { echo "plain run $TAG failed"; return 1; }
  ncu --set full --clock-control none --import-source on -k regex:"$KRE" --launch-skip $SKIP -c $CNT \
      -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
}
run c2 c2
full c2tail c2 "tail1d_kernel" 0 1
full c2cross c2 "cross1d_tile" 0 1
full c2mv c2 "matvec_kernel" 1 1
run c3 c3
full c3tail c3 "tail_kernel" 0 1
full c3cross c3 "cross_tile" 1 1
full c3near c3 "near_block" 0 1
run c5 c5
full c5mv c5 "matvec_kernel" 1 1
ls gpurun_out/*.ncu-rep
