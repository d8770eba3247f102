python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 1200 python tools/ab.py --workload rmat24 --reps 5 'GSM_CLIQUE_RANGES=1' 'GSM_CLIQUE_RANGES=0' 'GSM_CLIQUE_NH_STREAM=48' 'GSM_CLIQUE_NH_STREAM=96' 'GSM_CLIQUE_HUB_RATIO=32' 'GSM_CLIQUE_HUB_RATIO=128' 'GSM_CLIQUE_STREAM=96' 'GSM_CLIQUE_STREAM=192' > gpurun_out/ab1.jsonl 2> gpurun_out/ab1.err; cat gpurun_out/ab1.jsonl; tail -3 gpurun_out/ab1.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab_bench.json 2>/dev/null; python tools/show_bench.py gpurun_out/ab_bench.json | head -1 | cut -c1-200
echo ab-done
