set -u
O=gpurun_out
python -m pytest tests/test_gpu_neighbors.py -x -q -m gpu 2>&1 | tail -5
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --configs none"
$CMD > $O/plain_launch.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"
for K in 1 4 16 64; do
  CMD="python bench.py --ks $K --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --configs none"
  $CMD > $O/plain_tr$K.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__sass_average_branch_targets_threads_uniform.pct --clock-control none -k regex:'tile2d|query_kernel' --csv --log-file $O/traffic_k$K.csv $CMD > $O/ncu_tr$K.log 2>&1
  echo "traffic k=$K rc=$?"
done
KREGEX=tile2d_sel bash tools/prof_cmd.sh sel64 64 10000000 | tail -1
KREGEX=tile2d_thr_kernel bash tools/prof_cmd.sh thr16 16 10000000 | tail -1
