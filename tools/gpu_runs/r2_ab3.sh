python -c "from paper_2003_01527_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest -x -q tests/test_gpu_checked.py tests/test_gpu_parity.py -k "checked or clique_bitmap" > gpurun_out/t_ab3.log 2>&1; echo rc=$? >> gpurun_out/t_ab3.log; tail -3 gpurun_out/t_ab3.log
timeout 1500 python tools/ab.py --workload rmat24 --reps 5 'GSM_CLIQUE_OCC=0' 'GSM_CLIQUE_OCC=2' 'GSM_CLIQUE_OCC=1' 'GSM_CLIQUE_HUB_RATIO=32' 'GSM_CLIQUE_NH_STREAM=48' 'GSM_CLIQUE_NH_STREAM=96' 'GSM_CLIQUE_STREAM=96' 'GSM_CLIQUE_STREAM=192' 'GSM_CLIQUE_RANGES=1' > gpurun_out/ab3.jsonl 2> gpurun_out/ab3.err; cat gpurun_out/ab3.jsonl; tail -3 gpurun_out/ab3.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab3_bench.json 2>/dev/null; python tools/show_bench.py gpurun_out/ab3_bench.json 2>/dev/null | head -1 | cut -c1-200
echo ab3-done
