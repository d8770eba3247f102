#!/usr/bin/env python
"""Fig.-3-shaped sweeps on synthetic graphs.

  label sweep : R-MAT-16 (ef 8) with power-law (Zipf, alpha = 1) node labels,
                L in {20, 50, 100, 150, 200}; 10 random-walk queries of 12 nodes /
                22 edges per L ("10 different queries with 12 nodes and
                22 edges ... each query 10 times ... mean runtime").
  size sweep  : R-MAT-14 (ef 8), 8 uniform labels (the paper's Enron/Gowalla are
                unlabeled; unlabeled 13-node random-walk queries have astronomically
                many non-induced embeddings on R-MAT, so labels keep counts finite),
                random-walk queries of 3..13 nodes with ceil(1.5 k) edges.

Every point: mean device ms over `reps` runs (COUNT, all embeddings) and the count;
the first query of each point is checked against the CPU oracle on a root sample
(count and sorted rows of the embeddings with f(query vertex 0) in the sample).
Writes one JSON document (stdout and --out)."""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_point(G, g, queries, reps, stream, check_oracle=True, sample=256):
    import torch
    from paper_2003_01527_b200 import gsm
    out = []
    for qi, q in enumerate(queries):
        ms = []
        cnt = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, stream=stream)
            e1.record()
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
            cnt = r.count
        rec = {"query": q.name, "k": q.num_nodes, "edges": len(q.edges), "count": cnt,
               "ms_mean": sum(ms) / len(ms), "ms_min": min(ms)}
        if check_oracle and qi == 0:
            # parity on a root sample (all embeddings with f(query vertex 0) in the sample):
            # bounded oracle time whatever the query's total count
            import numpy as np
            import oracle
            roots = np.arange(0, g.num_nodes, max(1, g.num_nodes // sample), dtype=np.int32)
            t0 = time.perf_counter()
            oc, ref = oracle.match(g, q, roots=roots)
            rec["oracle_s"] = time.perf_counter() - t0
            rs = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, mode=gsm.GSM_MODE_ENUMERATE, root_subset=roots,
                               stream=stream)
            rows = rs.rows_numpy()
            rs.free()
            rec["sample_roots"] = len(roots)
            rec["oracle_sample_count"] = oc
            rec["parity"] = bool(rs.count == oc and np.array_equal(rows, ref))
        out.append(rec)
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--queries", type=int, default=10)
    p.add_argument("--out", default="")
    p.add_argument("--label-scale", type=int, default=16)
    a = p.parse_args()
    import torch
    import gsm_inputs as gi
    from paper_2003_01527_b200 import gsm
    stream = torch.cuda.current_stream().cuda_stream
    doc = {"label_sweep": [], "size_sweep": []}
    base = gi.rmat(a.label_scale, 8, 1)
    for L in (20, 50, 100, 150, 200):
        g = base.with_labels(gi.zipf_labels(base.num_nodes, L, seed=L))
        G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels)
        qs = [gi.random_walk_query(g, 12, 22, seed=100 * L + s) for s in range(a.queries)]
        pts = run_point(G, g, qs, a.reps, stream)
        G.free()
        doc["label_sweep"].append({"labels": L, "graph": g.name, "mean_ms": sum(x["ms_mean"] for x in pts) / len(pts),
                                   "points": pts})
        print(f"labels {L}: mean {doc['label_sweep'][-1]['mean_ms']:.3f} ms", file=sys.stderr)
    g16 = gi.rmat(14, 8, 1)
    g = g16.with_labels(gi.uniform_labels(g16.num_nodes, 8, 1))
    G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels)
    for k in range(3, 14):
        qs = [gi.random_walk_query(g, k, math.ceil(1.5 * k), seed=1000 * k + s) for s in range(min(a.queries, 5))]
        pts = run_point(G, g, qs, max(1, a.reps // 2), stream)
        doc["size_sweep"].append({"k": k, "mean_ms": sum(x["ms_mean"] for x in pts) / len(pts), "points": pts})
        print(f"k {k}: mean {doc['size_sweep'][-1]['mean_ms']:.3f} ms", file=sys.stderr)
    G.free()
    js = json.dumps(doc)
    print(js)
    if a.out:
        open(a.out, "w").write(js)


if __name__ == "__main__":
    main()
