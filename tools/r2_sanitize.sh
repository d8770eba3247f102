# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_driver.py (SPEC S:396 determinism;
# VERDICT r1 item 8).  Logs -> gpurun_out/sanitize_*.log
python -c "from paper_2003_01527_b200 import _build; _build.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 99 python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
echo sanitize-done
