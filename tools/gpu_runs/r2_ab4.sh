python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 1500 python tools/ab.py --workload rmat24 --reps 5 'GSM_CLIQUE_OCC=2' 'GSM_CLIQUE_OCC=3' 'GSM_CLIQUE_OCC=0' 'GSM_CLIQUE_HUB_RATIO=32' > gpurun_out/ab4.jsonl 2> gpurun_out/ab4.err; cat gpurun_out/ab4.jsonl; tail -3 gpurun_out/ab4.err
echo ab4-done
