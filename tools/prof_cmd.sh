#!/bin/bash
# Profile the predict kernel: plain run first (must exit 0), then ncu on the same command.
# usage: tools/prof_cmd.sh <tag> <k> [nq]
TAG=$1; K=$2; NQ=${3:-1000000}
CMD="python bench.py --nq $NQ --ks $K --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --configs none"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-query_kernel} -s 2 -c 1 \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
tail -2 gpurun_out/ncu_$TAG.log
