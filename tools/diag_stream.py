import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import gsm_inputs as gi
from paper_2003_01527_b200 import gsm
base = gi.rmat(13, 16, 1)
for L in (50, 200):
    g = base.with_labels(gi.zipf_labels(base.num_nodes, L, 1), tag=f"-Z{L}")
    G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0)
    q = gi.random_walk_query(g, 6, 9, seed=2000 + L)
    s = torch.cuda.Stream()
    for name, st in (("default", None), ("stream", s.cuda_stream), ("default2", None)):
        ws = []
        for i in range(5):
            torch.cuda.synchronize(); t = time.perf_counter()
            r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, stream=st); r.free()
            torch.cuda.synchronize(); ws.append((time.perf_counter() - t) * 1e3)
        print(json.dumps({"L": L, "stream": name, "wall_ms": [round(x, 3) for x in ws]}), flush=True)
    G.free()
