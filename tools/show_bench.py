import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        print(f, open(f).read()[-1500:]); continue
    r = d["roofline"]
    print(f, "ms/step %.1f" % d["ms_per_step"], "value %.3g" % d["value"], "achieved %.0f GB/s frac %.3f" % (r["achieved"] or 0, r["frac"] or 0),
          {k: round(v, 1) for k, v in r["per_kernel_ms_per_step"].items()})
    for q, v in d.get("per_query_rank0", {}).items():
        print("  ", q, "unique", v["unique"], "work", v["level_work"], "rows", v["level_rows"], "kms", v["kernel_ms"], "chunks", v["chunks"])
