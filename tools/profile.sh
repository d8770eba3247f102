#!/bin/bash
# On the GPU box: launch list (per-launch device time) + one `--set full` capture of the hot kernels.
# usage: tools/profile.sh <workload> [skip] [count]
wl=${1:-rmat16}; skip=${2:-0}; count=${3:-4}
export GSM_CACHE_DIR=${GSM_CACHE_DIR:-/tmp/gsm_inputs_cache}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${wl}.csv \
    python bench.py --workload $wl --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_${wl}.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_expand|k_tail|k_filter" -s $skip -c $count \
    -o gpurun_out/full_${wl} python bench.py --workload $wl --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full_${wl}.log 2>&1
echo profile-done
