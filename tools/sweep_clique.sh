# clique-path timing experiments on the GPU box (R-MAT-24 K3+K4)
timeout 600 python -m pytest tests/test_gpu_parity.py -k "clique or chunking" -x -q > gpurun_out/t_clique7.log 2>&1; echo rc=$? >> gpurun_out/t_clique7.log
B="python bench.py --workload rmat24 --steps 3 --warmup 1 --no-cpu-baseline --e2e-steps 0"
for cfg in "GSM_CLIQUE_OCC=1" "GSM_CLIQUE_DBG=1"; do
  echo "== $cfg" >> gpurun_out/sweep6.txt
  env $cfg timeout 300 $B 2>/dev/null | python tools/show_bench.py /dev/stdin >> gpurun_out/sweep6.txt 2>&1
done
