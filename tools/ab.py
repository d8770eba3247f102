"""Interleaved A/B of match-time switches on one resident graph (knobs are read at every
gsm_match, so variants alternate inside one process: box-to-box and run-to-run drift cancel).

    python tools/ab.py --workload rmat24 --reps 5 'GSM_CLIQUE_RANGES=1' 'GSM_CLIQUE_RANGES=0'

Prints per variant and query the median and min device ms (CUDA events on the match stream)."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="rmat24")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("variants", nargs="+")
    a = ap.parse_args()
    import torch

    from gsm_inputs import workloads
    from paper_2003_01527_b200 import gsm

    w = workloads.get(a.workload)
    g = w.graph()
    G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0)
    st = torch.cuda.current_stream()
    variants = []
    for v in a.variants:
        env = dict(kv.split("=", 1) for kv in v.split(",") if kv)
        variants.append((v, env))
    times = {(v, q.name): [] for v, _ in variants for q in w.queries}
    counts = {}
    base_env = dict(os.environ)
    for rep in range(a.reps + 1):
        for v, env in variants:
            os.environ.clear()
            os.environ.update(base_env)
            os.environ.update(env)
            for q in w.queries:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, mode=gsm.GSM_MODE_COUNT,
                                  mem_budget_bytes=w.mem_budget_bytes, stream=st.cuda_stream)
                e1.record(st)
                e1.synchronize()
                counts.setdefault(q.name, r.count)
                assert counts[q.name] == r.count, (v, q.name)
                if rep:
                    times[(v, q.name)].append(e0.elapsed_time(e1))
    os.environ.clear()
    os.environ.update(base_env)
    out = []
    for v, _ in variants:
        tot = 0.0
        row = {"variant": v}
        for q in w.queries:
            t = times[(v, q.name)]
            row[q.name] = {"median_ms": round(statistics.median(t), 3), "min_ms": round(min(t), 3)}
            tot += statistics.median(t)
        row["step_median_ms"] = round(tot, 3)
        out.append(row)
        print(json.dumps(row), flush=True)
    G.free()


if __name__ == "__main__":
    main()
