timeout 600 python -m pytest tests/test_gpu_parity.py -k "clique" -x -q > gpurun_out/t_clique12.log 2>&1; echo rc=$? >> gpurun_out/t_clique12.log
GSM_TRACE=2 python tools/probe_overhead.py rmat24 0 2>&1 | tail -3
python tools/probe_overhead.py rmat24 0 2>&1 | tail -2
