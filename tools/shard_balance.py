"""Multi-GPU readiness on one GPU: run the P root
shards of a workload SEQUENTIALLY on one B200 and report per-shard device time and
the max/mean imbalance — the N-GPU step time is the slowest shard, so max/mean is the
scaling efficiency loss due to skew.  Counts of the shards must add up to the
unsharded count.

    python tools/shard_balance.py [--workload rmat24] [--shards 8] [--reps 3]

Prints one JSON line per workload (kept under profiles/)."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="rmat24")
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--level1", action="store_true", help="GSM_FLAG_SHARD_LEVEL1: shard by level-1 pairs")
    args = ap.parse_args()
    import torch

    from gsm_inputs import workloads
    from paper_2003_01527_b200 import gsm

    w = workloads.get(args.workload)
    g = w.graph()
    G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0)
    stream = torch.cuda.current_stream()
    out = {"workload": args.workload, "shards": args.shards, "level1": bool(args.level1), "queries": {}}
    sflags = gsm.GSM_FLAG_SHARD_LEVEL1 if args.level1 else 0

    def timed(q, **kw):
        ms = []
        r = None
        for _ in range(args.reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, mode=gsm.GSM_MODE_COUNT,
                              mem_budget_bytes=w.mem_budget_bytes, stream=stream.cuda_stream, **kw)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        return r, statistics.median(ms[1:])

    step_full = 0.0
    per_shard_step = [0.0] * args.shards
    for q in w.queries:
        r_all, ms_all = timed(q)
        rows = []
        tot = 0
        for s in range(args.shards):
            r, ms = timed(q, shard_index=s, num_shards=args.shards, flags=sflags)
            tot += r.count
            rows.append({"shard": s, "ms": round(ms, 3), "count": r.count, "roots": r.level_rows[0],
                         "level1_rows": r.level_rows[1] if len(r.level_rows) > 1 else None,
                         "level1_sharded": r.level1_sharded})
            per_shard_step[s] += ms
        assert tot == r_all.count, (q.name, tot, r_all.count)
        mss = [x["ms"] for x in rows]
        out["queries"][q.name] = {"unsharded_ms": round(ms_all, 3), "count": r_all.count, "shards": rows,
                                  "max_over_mean": max(mss) / (sum(mss) / len(mss)),
                                  "sum_shards_over_unsharded": sum(mss) / ms_all}
        step_full += ms_all
    out["step"] = {"unsharded_ms": round(step_full, 3), "per_shard_ms": [round(x, 3) for x in per_shard_step],
                   "max_over_mean": max(per_shard_step) / (sum(per_shard_step) / len(per_shard_step)),
                   "ideal_speedup": step_full / max(per_shard_step)}
    G.free()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
