python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest -x -q tests/test_gpu_parity.py -k "clique_bitmap" > gpurun_out/t_ab6.log 2>&1; tail -2 gpurun_out/t_ab6.log
timeout 1500 python tools/ab.py --workload rmat24 --reps 4 '' 'GSM_CLIQUE_HUB_RATIO=32' 'GSM_CLIQUE_HUB_RATIO=128' 'GSM_CLIQUE_NH_STREAM=32' 'GSM_CLIQUE_NH_STREAM=128' 'GSM_CLIQUE_STREAM=64' 'GSM_CLIQUE_STREAM=256' 'GSM_CLIQUE_WARP=0' 'GSM_CLIQUE_HASH=0' 'GSM_CLIQUE_NE=0' > gpurun_out/ab6.jsonl 2> gpurun_out/ab6.err; cat gpurun_out/ab6.jsonl; tail -3 gpurun_out/ab6.err
echo ab6-done
