#!/bin/bash
# Usage (GPU box): bash tools/profile_k.sh <config> <tag> <kernel-regex> [launch-skip] [count]
# Plain run first (must exit 0), then one ncu --set full capture of the selected launches.
CFG=$1; TAG=$2; KRE=$3; SKIP=${4:-0}; CNT=${5:-1}
CMD="python bench.py --config $CFG --steps 1 --warmup 0 --no-cg --no-cpu --no-near --matvecs 2"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KRE" --launch-skip $SKIP -c $CNT \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
tail -n 2 gpurun_out/ncu_full_$TAG.log
