"""Fig.-3-shaped sweeps on synthetic graphs (PAPER P:213-220:
"size from 3 vertices to 13 vertices" (Fig. 3 left) and "10 different queries with
12 nodes and 22 edges" on "power-law-distributed node ... labels" from 20 to 200,
each query run 10 times, mean runtime (Fig. 3 right)).  Not a bench line: each point
prints one JSON line with the CUDA path's device time (CUDA events on the match stream,
one warm-up, then mean and median of --reps runs) and its count, checked against the
oracle (test infrastructure, the P:70 definition):

  * full count when the plain DFS finishes within --oracle-s (forked, killed after);
  * otherwise root-sampled parity: all embeddings with f(query vertex 0) in a fixed
    strided sample of --sample-roots vertices, on both sides (GSM root_subset).

Graphs: Enron-shaped R-MAT (scale 15, edge factor 8: 32k vertices, ~5 avg degree like
Enron's 36.7k / 183.8k) for the query-size axis, Gowalla-shaped R-MAT (scale 17,
edge factor 8: 131k vertices, Gowalla 196.6k / 950.3k) for the label axis.

    python tools/sweep_fig3.py --out gpurun_out/fig3_sweep.jsonl
"""
import argparse
import json
import multiprocessing as mp
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gsm_inputs as gi  # noqa: E402
import oracle  # noqa: E402
from paper_2003_01527_b200 import gsm  # noqa: E402


def time_match(G, q, reps, root_subset=None):
    """One warm-up run, then `reps` timed runs (1 when the warm-up took over a second: the
    12/13-node points count 1e13+ embeddings and take tens of seconds per match)."""
    s = torch.cuda.Stream()
    ts, cnt = [], None
    i = 0
    while i <= reps:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(s)
        r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, mode=gsm.GSM_MODE_COUNT, stream=s.cuda_stream,
                          root_subset=root_subset)
        b.record(s)
        torch.cuda.synchronize()
        cnt = r.count
        r.free()
        if i:
            ts.append(a.elapsed_time(b))
        elif a.elapsed_time(b) > 1000.0:
            reps = min(reps, 1)
        i += 1
    if not ts:  # reps == 0: the one (warm-up) run is the only sample
        return cnt, None, None
    return cnt, statistics.mean(ts), statistics.median(ts)


def _child(conn, d, n, q, roots):
    lab = os.path.join(d, "labels.npy")
    g = gi.Graph(n, np.load(os.path.join(d, "offsets.npy"), mmap_mode="r"),
                 np.load(os.path.join(d, "cols.npy"), mmap_mode="r"),
                 np.load(lab, mmap_mode="r") if os.path.exists(lab) else None)
    t0 = time.perf_counter()
    c = oracle.match(g, q, roots=roots, count_only=True)[0]
    conn.send((c, time.perf_counter() - t0))
    conn.close()


def oracle_bounded(g, q, roots, limit_s):
    """The oracle's count in a SPAWNED child (graph mmapped from .npy files; a forked child of
    this CUDA process hangs), killed after limit_s.  None on timeout."""
    import bench
    ctx = mp.get_context("spawn")
    a, b = ctx.Pipe(duplex=False)
    p = ctx.Process(target=_child, args=(b, bench._graph_files(g), g.num_nodes, q, roots), daemon=True)
    p.start()
    b.close()
    res = a.recv() if a.poll(limit_s + 10.0) else None
    if p.is_alive():
        p.kill()
    p.join()
    return res


def point(out, g, G, q, sweep, x, args):
    c, ms_mean, ms_med = time_match(G, q, args.reps)
    rec = {"sweep": sweep, "x": x, "graph": g.name, "query": q.name, "k": q.num_nodes, "edges": len(q.edges),
           "count": c, "gpu_ms_mean": ms_mean, "gpu_ms_median": ms_med, "oracle_threads": oracle.num_threads()}
    if ms_med < 5000:  # second GPU search path: the direct search without ID constraints (all embeddings)
        r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, mode=gsm.GSM_MODE_COUNT, flags=gsm.GSM_FLAG_NO_SYMMETRY)
        rec["nosym_count_equal"] = r.count == c
    res = oracle_bounded(g, q, None, args.oracle_s)
    if res is not None:
        rec.update(parity="full", oracle_count=res[0], oracle_s=res[1], match=c == res[0])
    elif args.sample_roots <= 0:
        rec.update(parity="none (full oracle over time limit)", match=None)
    else:
        # strided over the vertices that can host query vertex 0 (its label, degree >= its
        # query degree): a sample of arbitrary vertices mostly counts 0 and proves nothing
        qdeg0 = sum(1 for e in q.edges if 0 in e)
        deg = np.diff(g.offsets)
        ok = deg >= qdeg0
        if q.labels is not None and g.labels is not None:
            ok &= g.labels == q.labels[0]
        cand = np.nonzero(ok)[0]
        cnt = min(len(cand), args.sample_roots)
        roots = np.unique(cand[(np.arange(cnt) * (len(cand) / max(cnt, 1))).astype(np.int64)]).astype(np.int32)
        cs, _, _ = time_match(G, q, 0, root_subset=roots)
        res = oracle_bounded(g, q, roots, 3 * args.oracle_s)
        if res is None:
            rec.update(parity="none (oracle sample over time limit)", match=None)
        else:
            rec.update(parity=f"root-sampled ({len(roots)} strided candidate roots of query vertex 0)", sample_count=cs,
                       oracle_count=res[0],
                       oracle_s=res[1], match=cs == res[0])
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")
    out.flush()
    return rec["match"] is not False


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--oracle-s", type=float, default=20.0)
    p.add_argument("--sample-roots", type=int, default=32)
    p.add_argument("--queries", type=int, default=10, help="random-walk queries per label count (P:220)")
    p.add_argument("--out", default="gpurun_out/fig3_sweep.jsonl")
    p.add_argument("--axis", default="both", choices=["both", "sizes", "labels"])
    p.add_argument("--label-scale", type=int, default=17, help="R-MAT scale of the label-axis graph")
    a = p.parse_args()
    ok = True
    with open(a.out, "w") as out:
        # (a) query size 3..13, 20 Zipf labels, random-walk queries with 2k-3 edges
        # (a tree plus k-2 non-tree edges when the walk's induced subgraph has them)
        base = gi.rmat(15, 8, 1)
        g = base.with_labels(gi.zipf_labels(base.num_nodes, 20, 1), tag="-Z20")
        G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0)
        for k in (range(3, 14) if a.axis in ("both", "sizes") else []):
            q = None
            for e in range(2 * k - 3, k - 2, -1):  # as dense as the walks allow
                try:
                    q = gi.random_walk_query(g, k, max(k - 1, e), seed=1000 + k)
                    break
                except RuntimeError:
                    continue
            ok &= point(out, g, G, q, "query_size", k, a)
        G.free()
        # (b) label count 20..200: 10 random-walk queries of 12 nodes / 22 edges each
        base = gi.rmat(a.label_scale, 8, 1)
        for L in ((20, 50, 100, 150, 200) if a.axis in ("both", "labels") else ()):
            g = base.with_labels(gi.zipf_labels(base.num_nodes, L, 1), tag=f"-Z{L}")
            G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0)
            made = 0
            for s in range(200):
                if made == a.queries:
                    break
                try:
                    q = gi.random_walk_query(g, 12, 22, seed=2000 + 97 * L + s)
                except RuntimeError:
                    continue
                made += 1
                ok &= point(out, g, G, q, "labels", L, a)
            G.free()
    print("ALL MATCH" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
