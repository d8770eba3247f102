#!/bin/bash
# On the GPU box.  usage: tools/profile.sh <bench workload> <full-capture workload>
#  1. launch list of the bench command (per-launch device time, serialised, cold-ish caches)
#  2. DRAM bytes per launch of the hot kernels on the bench workload (traffic for bench.py)
#  3. one `--set full` capture of the hot kernels on a smaller workload with the same code path
wl=${1:-rmat24}; fwl=${2:-rmat20}
B="python bench.py --workload $wl --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${wl}.csv $B > gpurun_out/ncu_launch_${wl}.log 2>&1
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_clique|k_tail|k_expand|k_count_walk|k_filter" --csv --log-file gpurun_out/traffic_${wl}.csv $B > gpurun_out/ncu_traffic_${wl}.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_clique|k_tail|k_count_walk|k_expand" -c 8 \
    -o gpurun_out/full_${fwl} python bench.py --workload $fwl --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full_${fwl}.log 2>&1
echo profile-done
