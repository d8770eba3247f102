python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1; cat gpurun_out/e2e_probe.log | tail -8
GSM_TRACE=1 timeout 600 python tools/e2e_probe.py 2>&1 | grep "gsm load\]" | tail -14
echo e2e-done
