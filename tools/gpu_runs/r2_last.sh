python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r2_gpu_tests_last.log 2>&1; echo rc=$? >> gpurun_out/r2_gpu_tests_last.log; tail -3 gpurun_out/r2_gpu_tests_last.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_last.log 2>&1; echo rc=$? >> gpurun_out/r2_smoke_last.log; tail -2 gpurun_out/r2_smoke_last.log
for sc in 11 13; do
  timeout 700 python tools/sweep_fig3.py --axis labels --label-scale $sc --reps 10 --oracle-s 10 --queries 2 --out gpurun_out/r2_fig3_labels_s$sc.jsonl > gpurun_out/r2_fig3_labels_s$sc.log 2>&1
  echo "scale $sc rc=$?"; tail -1 gpurun_out/r2_fig3_labels_s$sc.log
done
echo last-done
