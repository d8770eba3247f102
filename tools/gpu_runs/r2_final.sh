# Round-2 final measurement on one B200: full GPU suite + smoke, the bench line of every config,
# the reference arm, and the ncu launch list + traffic of the default bench command.
python -c "from paper_2003_01527_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 2700 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2_gpu_tests_final.log 2>&1; echo rc=$? >> gpurun_out/r2_gpu_tests_final.log; tail -4 gpurun_out/r2_gpu_tests_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_final.log 2>&1; echo rc=$? >> gpurun_out/r2_smoke_final.log; tail -2 gpurun_out/r2_smoke_final.log
b() { tag=$1; shift; timeout 900 "$@" > gpurun_out/r2_bench_final_$tag.json 2> gpurun_out/r2_bench_final_$tag.err; echo "== $tag"; python tools/show_bench.py gpurun_out/r2_bench_final_$tag.json 2>&1 | head -1 | cut -c1-300; }
b rmat24 python bench.py
b reference python bench.py --impl reference --steps 3 --warmup 3
b er1000 python bench.py --workload er1000 --steps 20 --warmup 5 --e2e-steps 5
b rmat16 python bench.py --workload rmat16 --steps 5 --warmup 3
b grid1m python bench.py --workload grid1m --steps 5 --warmup 3
b rmat22 python bench.py --workload rmat22 --steps 5 --warmup 3
b enum16 python bench.py --workload rmat16 --mode enumerate --steps 3 --warmup 3 --no-cpu-baseline
b bfs24 python bench.py --clique 0 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0
B="python bench.py --workload rmat24 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_elapsed.avg
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_final_launches_rmat24.csv $B > gpurun_out/ncu_fl.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_final_traffic_rmat24.csv $B > gpurun_out/ncu_ft.log 2>&1
echo final-done
