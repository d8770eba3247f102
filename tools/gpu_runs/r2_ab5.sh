python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 1500 python tools/ab.py --workload rmat24 --reps 5 'GSM_CLIQUE_OCC=3,GSM_CLIQUE_NTSEL=1' 'GSM_CLIQUE_OCC=3,GSM_CLIQUE_NTSEL=0' 'GSM_CLIQUE_OCC=2,GSM_CLIQUE_NTSEL=1' 'GSM_CLIQUE_OCC=4,GSM_CLIQUE_NTSEL=1' 'GSM_CLIQUE_OCC=4,GSM_CLIQUE_NTSEL=0' 'GSM_CLIQUE_OCC=0,GSM_CLIQUE_NTSEL=1' > gpurun_out/ab5.jsonl 2> gpurun_out/ab5.err; cat gpurun_out/ab5.jsonl; tail -3 gpurun_out/ab5.err
echo ab5-done
