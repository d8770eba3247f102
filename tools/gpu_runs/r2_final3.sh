# Round-2 final measurement 3: every config's bench line (oracle baseline after the timed work),
# reference arm, K1 grid variants, ncu traffic + launch list of the final kernels.
python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
b() { tag=$1; shift; timeout 900 "$@" > gpurun_out/r2_bench_final3_$tag.json 2> gpurun_out/r2_bench_final3_$tag.err; echo "== $tag"; python tools/show_bench.py gpurun_out/r2_bench_final3_$tag.json 2>/dev/null | head -1 | cut -c1-260; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_final3_$tag.json').read().strip().splitlines()[-1]); c=d.get('cpu_baseline') or {}; print('cpu', c.get('value'), c.get('cores'), (c.get('sample') or '')[-100:])"; }
b rmat24 python bench.py
b reference python bench.py --impl reference --steps 3 --warmup 3
b er1000 python bench.py --workload er1000 --steps 20 --warmup 5 --e2e-steps 5
b rmat16 python bench.py --workload rmat16 --steps 5 --warmup 3
b grid1m python bench.py --workload grid1m --steps 5 --warmup 3
b rmat22 python bench.py --workload rmat22 --steps 5 --warmup 3
for bps in 8 32 128; do GSM_FILTER_BPS=$bps timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fbps_$bps.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/fbps_$bps.json').read().strip().splitlines()[-1]); print('filter bps $bps', {q: v['kernel_ms']['filter'] for q, v in d['per_query_rank0'].items()})"; done
B="python bench.py --workload rmat24 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_elapsed.avg
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_final3_launches_rmat24.csv $B > gpurun_out/ncu_fl3.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_final3_traffic_rmat24.csv $B > gpurun_out/ncu_ft3.log 2>&1
timeout 600 python tools/load_phases.py rmat24 > gpurun_out/load_final3.log 2>&1; grep "load 2\|hashed\|relabelled\|upload" gpurun_out/load_final3.log | tail -4
echo final3-done
timeout 2400 python tools/sweep_fig3.py --axis labels --reps 10 --oracle-s 10 --queries 4 --out gpurun_out/r2_fig3_labels.jsonl > gpurun_out/r2_fig3_labels.log 2>&1
echo rc=$? >> gpurun_out/r2_fig3_labels.log; tail -3 gpurun_out/r2_fig3_labels.log
echo labels-done
