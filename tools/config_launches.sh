#!/bin/bash
# Per-config launch lists (cfg0-3): duration and DRAM bytes of every launch of one bench run
# (fit + untimed counters + 1 warm-up + 1 timed step), cold-cache and serialised.
for c in ${CFGS:-0 1 2 3}; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --configs none --parity-sample 20"
  timeout 1500 $CMD > gpurun_out/cfg${c}_plain.log 2>&1 && \
  timeout 2700 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_cfg$c.csv $CMD > /dev/null 2>&1
  echo "cfg$c rc=$?"
done
