python -c "from paper_2003_01527_b200 import _build; _build.build(); _build.build(checked=True)" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest -x -q tests/test_gpu_checked.py tests/test_gpu_parity.py -k "checked or clique_bitmap" > gpurun_out/t_ab2.log 2>&1; echo rc=$? >> gpurun_out/t_ab2.log; tail -3 gpurun_out/t_ab2.log
timeout 1200 python tools/ab.py --workload rmat24 --reps 5 'GSM_CLIQUE_RANGES=0' 'GSM_CLIQUE_HUB_RATIO=32' 'GSM_CLIQUE_HUB_RATIO=16' 'GSM_CLIQUE_OCC=0' > gpurun_out/ab2.jsonl 2> gpurun_out/ab2.err; cat gpurun_out/ab2.jsonl; tail -3 gpurun_out/ab2.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ab2_bench.json 2>/dev/null; python tools/show_bench.py gpurun_out/ab2_bench.json 2>/dev/null | head -1 | cut -c1-200
echo ab2-done
