# Final pass: GPU suite, smoke, bench lines of every config + the reference arm.
python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for wl in er1000 rmat16 grid1m rmat22; do python bench.py --workload $wl > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; done
B22="python bench.py --workload rmat22 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_pair|k_plan_rows|k_expand|k_count_walk" --csv --log-file gpurun_out/traffic_rmat22.csv $B22 > gpurun_out/ncu_traffic_rmat22.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat22.csv $B22 > gpurun_out/ncu_launch_rmat22.log 2>&1
echo final-done
