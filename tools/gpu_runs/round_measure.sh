# Full measurement pass on the GPU box: GPU test suite, bench lines of every config (+ the
# reference arm), ncu launch list / DRAM traffic / --set full capture on the default workload,
# and a capture of the pair-tail kernel on configs[3].
python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for wl in er1000 rmat16 grid1m rmat22; do python bench.py --workload $wl > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; done
B="python bench.py --workload rmat24 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat24.csv $B > gpurun_out/ncu_launch_rmat24.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_clique|k_filter" --csv --log-file gpurun_out/traffic_rmat24.csv $B > gpurun_out/ncu_traffic_rmat24.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_clique_cta --launch-skip 7 -c 1 -o gpurun_out/full_rmat24_k4 $B > gpurun_out/ncu_full_k4.log 2>&1
B22="python bench.py --workload rmat22 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat22.csv $B22 > gpurun_out/ncu_launch_rmat22.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_pair|k_plan_rows|k_expand|k_count_walk" --csv --log-file gpurun_out/traffic_rmat22.csv $B22 > gpurun_out/ncu_traffic_rmat22.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pair -c 1 -o gpurun_out/full_rmat22_pair $B22 > gpurun_out/ncu_full_pair.log 2>&1
echo measure-done
