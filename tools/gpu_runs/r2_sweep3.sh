python -c "from paper_2003_01527_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest -x -q tests/test_gpu_checked.py tests/test_gpu_parity.py -k "checked or clique_bitmap" > gpurun_out/t_s3.log 2>&1; tail -2 gpurun_out/t_s3.log
timeout 900 python tools/ab.py --workload rmat24 --reps 4 '' 'GSM_CLIQUE_LAZYCK=0' 'GSM_CLIQUE_HASH=0' 'GSM_CLIQUE_HUB_RATIO=128' > gpurun_out/ab7.jsonl 2> gpurun_out/ab7.err; cat gpurun_out/ab7.jsonl; tail -2 gpurun_out/ab7.err
timeout 2400 python tools/sweep_fig3.py --reps 10 --oracle-s 20 --queries 4 --out gpurun_out/r2_fig3_sweep3.jsonl > gpurun_out/r2_fig3_3.log 2>&1
echo rc=$? >> gpurun_out/r2_fig3_3.log; tail -3 gpurun_out/r2_fig3_3.log
echo sweep3-done
