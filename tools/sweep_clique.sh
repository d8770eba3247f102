# clique-path timing experiments on the GPU box (R-MAT-24 K3+K4)
B="python bench.py --workload rmat24 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0"
for cfg in "GSM_CLIQUE_DBG=0" "GSM_CLIQUE_DBG=1" "GSM_CLIQUE_DBG=3" "GSM_CLIQUE_DSMEM=1024" "GSM_CLIQUE_WARP=0"; do
  echo "== $cfg" >> gpurun_out/sweep2.txt
  env $cfg timeout 300 $B 2>/dev/null | python tools/show_bench.py /dev/stdin >> gpurun_out/sweep2.txt 2>&1
done
