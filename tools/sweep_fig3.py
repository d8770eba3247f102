"""Fig.-3-shaped sweeps on synthetic graphs (PAPER P:218-220:
random-walk queries of a given size, power-law labels; Fig. 3 varies query size and
label count).  Not a bench line: each point prints one JSON line with the CUDA path's
device time (CUDA events on the match stream, median of --reps after one warm-up) and
its count, checked against the oracle's count (test infrastructure, P:70 definition).

    python tools/sweep_fig3.py --scale 13 --out gpurun_out/fig3_sweep.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gsm_inputs as gi  # noqa: E402
import oracle  # noqa: E402
from paper_2003_01527_b200 import gsm  # noqa: E402


def time_match(G, q, reps):
    s = torch.cuda.Stream()
    ts, cnt = [], None
    for i in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(s)
        r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, mode=gsm.GSM_MODE_COUNT, stream=s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        cnt = r.count
        r.free()
        if i:
            ts.append(a.elapsed_time(b))
    return cnt, float(np.median(ts))


def point(out, g, G, q, sweep, x, reps):
    c, ms = time_match(G, q, reps)
    t0 = time.perf_counter()
    ref, _ = oracle.match(g, q, count_only=True)
    ot = time.perf_counter() - t0
    rec = {"sweep": sweep, "x": x, "query": q.name, "k": q.num_nodes, "edges": len(q.edges),
           "count": c, "oracle_count": ref, "match": c == ref, "gpu_ms": ms,
           "oracle_s": ot, "oracle_threads": oracle.num_threads()}
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")
    out.flush()
    return c == ref


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--scale", type=int, default=13)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--out", default="gpurun_out/fig3_sweep.jsonl")
    a = p.parse_args()
    ok = True
    base = gi.rmat(a.scale, 16, 1)
    with open(a.out, "w") as out:
        # (a) query size 3..7 with 20 Zipf labels; 2k-3 edges.  Larger or sparser
        # queries make the plain-DFS oracle's counts (and time) explode on Zipf labels.
        g = base.with_labels(gi.zipf_labels(base.num_nodes, 20, 1), tag="-Z20")
        G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0)
        for k in range(3, 8):
            q = gi.random_walk_query(g, k, max(3, 2 * k - 3), seed=1000 + k)
            ok &= point(out, g, G, q, "query_size", k, a.reps)
        G.free()
        # (b) label count 20..200 at query size 6 (Fig. 3 label axis)
        for L in (20, 50, 100, 200):
            g = base.with_labels(gi.zipf_labels(base.num_nodes, L, 1), tag=f"-Z{L}")
            G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0)
            q = gi.random_walk_query(g, 6, 9, seed=2000 + L)
            ok &= point(out, g, G, q, "labels", L, a.reps)
            G.free()
    print("ALL MATCH" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
