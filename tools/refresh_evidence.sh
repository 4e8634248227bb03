#!/bin/bash
# Round evidence on one B200: bench line, reference arm, launch list, per-k DRAM traffic.
# Every ncu command below is the same bench command that already exited 0 without ncu.
set -u
O=gpurun_out
python bench.py > $O/bench.json 2> $O/bench.err || { echo "bench failed"; tail -20 $O/bench.err; exit 1; }
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
echo "bench rc=0"
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --configs none"
$CMD > $O/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"
for K in 1 4 16 64; do
  CMD="python bench.py --ks $K --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --configs none"
  $CMD > $O/plain_tr$K.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__sass_average_branch_targets_threads_uniform.pct \
      --clock-control none -k regex:'tile2d|query_kernel' --csv --log-file $O/traffic_k$K.csv $CMD > $O/ncu_tr$K.log 2>&1
  echo "traffic k=$K rc=$?"
done
# fit launch list (cold-cache, serialised): build the cfg4 index twice, the second is the one to read
timeout 120 python tools/fit_launches.py > $O/fl_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/fit_launches.csv python tools/fit_launches.py > $O/fl_ncu.log 2>&1
echo "fit launch list rc=$?"
# issue-slot captures of the timed kernels (k = 64 bucket select, k = 16 list rounds): --set full, source on
KREGEX=tile2d_sel bash tools/prof_cmd.sh sel64 64 10000000 | tail -1
KREGEX=tile2d_thr_kernel bash tools/prof_cmd.sh thr16 16 10000000 | tail -1
