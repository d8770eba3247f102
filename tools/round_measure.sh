# Full measurement pass on the GPU box: GPU test suite, default bench line (+ other configs),
# ncu launch list, per-kernel DRAM traffic, one --set full capture of the dominant kernel.
python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --workload rmat24 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rmat24.csv $B > gpurun_out/ncu_launch_rmat24.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_clique|k_filter" --csv --log-file gpurun_out/traffic_rmat24.csv $B > gpurun_out/ncu_traffic_rmat24.log 2>&1
python tools/ncu_summary.py metrics gpurun_out/traffic_rmat24.csv rmat24 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_clique_cta --launch-skip 7 -c 1 -o gpurun_out/full_rmat24_k4 $B > gpurun_out/ncu_full_k4.log 2>&1
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for wl in er1000 rmat16 grid1m rmat22; do python bench.py --workload $wl --no-cpu-baseline > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; done
echo measure-done
