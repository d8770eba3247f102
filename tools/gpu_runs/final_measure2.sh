timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q > gpurun_out/t_par2.log 2>&1; echo rc=$? >> gpurun_out/t_par2.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for wl in er1000 rmat16 grid1m rmat22; do python bench.py --workload $wl > gpurun_out/bench_$wl.json 2> gpurun_out/bench_$wl.err; done
echo done
