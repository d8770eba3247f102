"""Write tests/golden/<graph>_cliques.json: exact K3 / K4 counts of a generated
R-MAT graph from the ORACLE's independent degree-ordered clique counters
(oracle/oracle.c oracle_count_*_roots).  Calls only ``oracle`` and the seeded
input generators; nothing here touches the CUDA path (SURVEY §8(c) configs[4]
pin (ii): "exact triangle/K4 counts from an independent degree-ordered CPU
counter"; §4 validates counts against a CPU reference).

Stored per graph and clique size k:
  total          number of k-cliques (unique; all embeddings = k! x total)
  shards[P][s]   cliques whose lowest (degree, id)-ranked vertex v has
                 rank(v) % P == s   (the product's root shard)
  roots          {original id: count} for the 64 highest-degree vertices and
                 256 uniform (strided) vertices: cliques whose lowest vertex is it

Usage: python tools/make_golden_cliques.py --scale 24 [--threads 8]
(R-MAT-24 K4 takes about an hour on 8 cores.)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gsm_inputs as gi  # noqa: E402
import oracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--ks", default="3,4")
    args = ap.parse_args()
    g = gi.rmat(args.scale, args.ef, args.seed)
    n = g.num_nodes
    rank = oracle.rank_order(g)
    deg = np.diff(g.offsets)
    hubs = np.argsort(-deg, kind="stable")[:64]
    uni = np.arange(0, n, max(1, n // 256), dtype=np.int64)[:256]
    sample = np.unique(np.concatenate([hubs, uni]))
    name = f"rmat{args.scale}"
    path = os.path.join(ROOT, "tests", "golden", f"{name}_cliques.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out.update({
        "graph": f"gsm_inputs.rmat({args.scale}, {args.ef}, {args.seed})",
        "num_nodes": int(n), "nnz": int(g.nnz),
        "source": "tools/make_golden_cliques.py -> oracle.clique_counts_by_root (oracle/oracle.c, "
                  "degree-ordered forward counting; SURVEY 8(c) configs[4] pin (ii))",
        "hub_roots": [int(v) for v in hubs], "uniform_roots": [int(v) for v in uni],
    })
    for k in [int(x) for x in args.ks.split(",")]:
        t0 = time.time()
        total, per = oracle.clique_counts_by_root(g, k, None, args.threads)
        dt = time.time() - t0
        shards = {}
        for P in (2, 4, 8, 64):
            s = np.zeros(P, dtype=np.uint64)
            np.add.at(s, rank % P, per)
            shards[str(P)] = [int(x) for x in s]
        out[f"K{k}"] = {"total": int(total), "seconds": round(dt, 1), "threads": args.threads or oracle.num_threads(),
                        "shards": shards, "roots": {str(int(v)): int(per[v]) for v in sample}}
        print(f"{name} K{k}: {total} cliques in {dt:.1f} s", flush=True)
        json.dump(out, open(path + ".tmp", "w"), indent=1)
        os.replace(path + ".tmp", path)


if __name__ == "__main__":
    main()
