python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
for v in "GSM_BIGSORT=0" "GSM_BIGSORT=1 GSM_BIGSORT_MIN=8192" "GSM_BIGSORT=1 GSM_BIGSORT_MIN=32768" "GSM_BIGSORT=1 GSM_BIGSORT_MIN=131072"; do
  env $v timeout 300 python tools/load_phases.py rmat24 > gpurun_out/bs.log 2>&1; echo "$v: $(grep 'relabelled' gpurun_out/bs.log | tail -1) $(grep 'load 2' gpurun_out/bs.log)"
done
echo bigsort-done
