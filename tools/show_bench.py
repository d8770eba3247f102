"""Summarise bench.py JSON lines: python tools/show_bench.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        try:
            print(f, open(f).read()[-1500:])
        except OSError as e:
            print(f, e)
        continue
    r = d["roofline"]
    e = d.get("e2e") or {}
    print(f, "ms/step %.2f (median %.2f)" % (d["ms_per_step"], d.get("ms_median", 0)), "value %.4g" % d["value"],
          "e2e %.4g" % (e.get("value") or 0), "achieved %.0f GB/s frac %.3f" % (r["achieved"] or 0, r["frac"] or 0),
          "launches", d.get("gpu_launches"), {k: round(v, 2) for k, v in r["per_kernel_ms_per_step"].items()})
    for q, v in d.get("per_query_rank0", {}).items():
        print("  ", q, "unique", v["unique"], "work", v["level_work"], "rows", v["level_rows"],
              "fbytes", v.get("level_frontier_bytes"), "kms", v["kernel_ms"], "ms", v["ms"], "chunks", v["chunks"])
