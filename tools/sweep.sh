#!/bin/bash
# usage: tools/sweep.sh <workload> <steps> "<ILP list>" "<TD list>"
wl=$1; steps=$2
for u in $3; do for td in $4; do
  GSM_EXPAND_ILP=$u GSM_EXPAND_TD=$td timeout 900 python bench.py --workload $wl --steps $steps --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sw_${wl}_u${u}_td${td}.log 2>&1
done; done
