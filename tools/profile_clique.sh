timeout 600 python -m pytest tests/test_gpu_parity.py -k "clique" -x -q > gpurun_out/t_clique4.log 2>&1; echo rc=$? >> gpurun_out/t_clique4.log
B="python bench.py --workload rmat24 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2_rmat24.csv $B > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_clique_cta|k_clique_warp" -c 14 -o gpurun_out/full2_rmat24 $B > gpurun_out/ncu_full2.log 2>&1
echo done
