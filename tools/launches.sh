#!/bin/bash
# Per-launch device times of one bench configuration (cold-cache, serialised).
# usage: tools/launches.sh <tag> <k> [extra bench args]
TAG=$1; K=$2; shift 2
CMD="python bench.py --ks $K --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $@"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
