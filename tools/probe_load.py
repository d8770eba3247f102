"""gsm_load_graph time (pinned host buffers, as bench.py's e2e) and a K3 count check."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from gsm_inputs import workloads
from paper_2003_01527_b200 import gsm
w = workloads.get(sys.argv[1] if len(sys.argv) > 1 else "rmat24")
g = w.graph()
off_h = torch.from_numpy(g.offsets).pin_memory(); cols_h = torch.from_numpy(g.cols).pin_memory()
lab_h = None if g.labels is None else torch.from_numpy(g.labels.view(np.int32)).pin_memory()
for it in range(4):
    torch.cuda.synchronize(); t = time.perf_counter()
    G = gsm.gsm_load_graph(g.num_nodes, off_h, cols_h, lab_h, device=0)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    msg = []
    for q in w.queries:
        t = time.perf_counter()
        r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, mem_budget_bytes=w.mem_budget_bytes)
        msg.append(f"{q.name} {r.count} {(time.perf_counter() - t) * 1e3:.1f} ms")
    t = time.perf_counter()
    G.free()
    torch.cuda.synchronize()
    print(f"load {dt*1e3:.1f} ms; " + "; ".join(msg) + f"; free {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
