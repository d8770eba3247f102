bash tools/gpu_runs/r2_ab6.sh
timeout 300 python tools/r2_trace_small.py > gpurun_out/trace_small.log 2>&1; tail -20 gpurun_out/trace_small.log
timeout 2700 python tools/sweep_fig3.py --reps 10 --oracle-s 20 --out gpurun_out/r2_fig3_sweep.jsonl > gpurun_out/r2_fig3.log 2>&1
echo rc=$? >> gpurun_out/r2_fig3.log
tail -3 gpurun_out/r2_fig3.log
echo sweep2-done
