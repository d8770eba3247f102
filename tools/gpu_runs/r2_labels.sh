python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
for sc in 11 13; do
  timeout 600 python tools/sweep_fig3.py --axis labels --label-scale $sc --reps 3 --oracle-s 10 --queries 2 --out gpurun_out/r2_fig3_labels_s$sc.jsonl > gpurun_out/r2_fig3_labels_s$sc.log 2>&1
  echo "scale $sc rc=$?"; cat gpurun_out/r2_fig3_labels_s$sc.jsonl | cut -c1-300
done
echo labels-done
