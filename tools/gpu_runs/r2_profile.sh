# Round-2 profiling pass (one GPU): launch list + DRAM traffic / sector efficiency of the bench
# command, one `ncu --set full` capture per hot kernel, the random-gather ceiling, and
# compute-sanitizer memcheck / racecheck / synccheck.  Everything -> gpurun_out/.
python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
B() { echo "python bench.py --workload $1 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 $2"; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_elapsed.avg
# 1. launch list of the default bench command (per-launch times: the kernel's share of the step)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_rmat24.csv $(B rmat24) > gpurun_out/ncu_l24.log 2>&1
# 2. traffic + sector efficiency + instructions per launch of every kernel of the bench command
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_traffic_rmat24.csv $(B rmat24) > gpurun_out/ncu_t24.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_traffic_rmat22.csv $(B rmat22) > gpurun_out/ncu_t22.log 2>&1
echo traffic-done
# 3. full captures (source-level) of each hot kernel
# F tag kernel-regex count workload [bench args]
F() { tag=$1; rx=$2; c=$3; wl=$4; shift 4; timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -c $c -o gpurun_out/r2_full_$tag $(B $wl "$*") > gpurun_out/ncu_full_$tag.log 2>&1; echo "full $tag rc=$?"; }
F clique_rmat24 "k_clique_cta|k_clique_warp" 14 rmat24
F filter_rmat24 "k_filter" 1 rmat24
F pair_rmat22 "k_pair|k_plan_rows" 8 rmat22
F refine_rmat22 "k_refine" 2 rmat22 --refine-rounds 1
F expand_rmat16 "k_expand|k_count_walk|k_plan_rows" 8 rmat16
F bfs_rmat24 "k_expand|k_tail|k_plan_rows" 6 rmat24 --clique 0
echo full-done
echo profile-done
