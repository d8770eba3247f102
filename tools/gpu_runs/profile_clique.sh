# source-level ncu captures of the clique kernels on R-MAT-24 (K3 and K4, the (512,1024] bucket)
B="python bench.py --workload rmat24 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_clique_cta --launch-skip 1 -c 1 -o gpurun_out/k3b4 $B > gpurun_out/ncu_k3b4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_clique_cta --launch-skip 7 -c 1 -o gpurun_out/k4b4 $B > gpurun_out/ncu_k4b4.log 2>&1
echo done
