python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 2400 python tools/sweep_fig3.py --reps 10 --oracle-s 20 --out gpurun_out/r2_fig3_sweep.jsonl > gpurun_out/r2_fig3.log 2>&1
echo rc=$? >> gpurun_out/r2_fig3.log
tail -3 gpurun_out/r2_fig3.log
