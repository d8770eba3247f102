python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --durations=8 > gpurun_out/gpu_parity.log 2>&1; echo rc=$? >> gpurun_out/gpu_parity.log
bash tools/r2_perf.sh > gpurun_out/perf_summary.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo run2-done
