"""Where the step time outside the kernels goes (R-MAT-24 K3+K4): wall time per gsm_match
call vs CUDA-event time of the step vs the per-kernel event sums."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import gsm_inputs as gi
from gsm_inputs import workloads
from paper_2003_01527_b200 import gsm

w = workloads.get(sys.argv[1] if len(sys.argv) > 1 else "rmat24")
g = w.graph() if callable(getattr(w, "graph", None)) else w.graph
G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0)
s = torch.cuda.current_stream().cuda_stream
for it in range(4):
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    walls = []
    for q in w.queries:
        t = time.perf_counter()
        r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, mode=gsm.GSM_MODE_COUNT, flags=int(sys.argv[2]) if len(sys.argv) > 2 else 0,
                          mem_budget_bytes=w.mem_budget_bytes, stream=s)
        walls.append((q.name, round((time.perf_counter() - t) * 1e3, 2), round(r.ms["total"], 2),
                      round(sum(v["ms"] for v in r.prof.values()), 2)))
    ev1.record(); ev1.synchronize()
    print("step event ms", round(ev0.elapsed_time(ev1), 2), walls, flush=True)
