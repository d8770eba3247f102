"""e2e variance probe: with the resident graph loaded (as bench.py), time 6 end-to-end steps
(gsm_load_graph from pinned host buffers + K3/K4 matches + gsm_free), host wall per phase."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from gsm_inputs import workloads  # noqa: E402
from paper_2003_01527_b200 import gsm  # noqa: E402

w = workloads.get("rmat24")
g = w.graph()
torch.cuda.set_device(0)
G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, None, device=0)
for q in w.queries:
    gsm.gsm_match(G, q.num_nodes, q.edges, None, mem_budget_bytes=w.mem_budget_bytes)
off_h = torch.from_numpy(g.offsets).pin_memory()
cols_h = torch.from_numpy(g.cols).pin_memory()
for it in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G2 = gsm.gsm_load_graph(g.num_nodes, off_h, cols_h, None, device=0)
    t1 = time.perf_counter()
    for q in w.queries:
        gsm.gsm_match(G2, q.num_nodes, q.edges, None, mem_budget_bytes=w.mem_budget_bytes)
    t2 = time.perf_counter()
    G2.free()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"e2e step {it}: load {1e3*(t1-t0):.1f} ms, matches {1e3*(t2-t1):.1f} ms, free {1e3*(t3-t2):.1f} ms, "
          f"total {1e3*(t3-t0):.1f} ms", flush=True)
G.free()
