"""Diagnostic for the label-count sweep (tools/sweep_fig3.py): per-kernel times, launches,
chunks and level sizes of one COUNT match per label count, GSM_FLAG_PROFILE on."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gsm_inputs as gi
from paper_2003_01527_b200 import gsm

base = gi.rmat(13, 16, 1)
for L in (20, 50, 100, 200):
    g = base.with_labels(gi.zipf_labels(base.num_nodes, L, 1), tag=f"-Z{L}")
    G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0)
    q = gi.random_walk_query(g, 6, 9, seed=2000 + L)
    for rep in range(2):
        r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, mode=gsm.GSM_MODE_COUNT, flags=gsm.GSM_FLAG_PROFILE)
        print(json.dumps({"L": L, "rep": rep, "count": r.count, "ms": r.ms, "launches": r.kernel_launches,
                          "chunks": r.num_chunks, "cand": r.candidates, "level_rows": r.level_rows,
                          "prof": {k: v for k, v in r.prof.items() if v["launches"]}}), flush=True)
        r.free()
    G.free()
