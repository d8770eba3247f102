python -c "from paper_2003_01527_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
for hb in 65536 49152 98304 131072; do
  GSM_HUB_BITS=$hb timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/hub_$hb.json 2>/dev/null
  python tools/show_bench.py gpurun_out/hub_$hb.json 2>/dev/null | head -1 | cut -c1-200 | sed "s/^/hb=$hb /"
done
echo hub-done
