"""Print the BASELINE.md §4 result rows from the committed bench lines (profiles/r1_bench_*.json)."""
import json, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = [("er1000", "[0] G(1000,4000) seed 1", "K3"), ("rmat16", "[1] R-MAT-16, 8 labels", "P4 ×2, S3 ×2"),
        ("grid1m", "[2] grid 1000² + diagonals", "C4, K4"), ("rmat22", "[3] R-MAT-22, 16 labels", "house ×2"),
        ("rmat24_default", "**[4] R-MAT-24 (bench default)**", "K3 + K4")]
for f, name, q in rows:
    p = os.path.join(ROOT, "profiles", f"r1_bench_{f}.json")
    d = json.loads(open(p).read().strip().splitlines()[-1])
    r = d["roofline"]
    e2e = d.get("e2e") or {}
    print(f"| {name} | {q} | {d['counts_per_step']['unique']:.3g} / {d['counts_per_step']['all']:.3g} | "
          f"{d['ms_per_step']:.4g} | {d['value']:.3g} | {e2e.get('value', 0):.3g} | "
          f"`{r['kernel']}` ({(r['frac'] or 0):.2f}; share {(r.get('share_of_step') or 0):.0%}) |")
