"""Per-phase gsm_load_graph times (GSM_TRACE=1) from pinned host buffers, for the e2e path.
    python tools/load_phases.py [workload ...]"""
import os
import sys
import time

os.environ["GSM_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from gsm_inputs import workloads  # noqa: E402
from paper_2003_01527_b200 import gsm  # noqa: E402

for name in sys.argv[1:] or ["rmat24", "rmat22"]:
    g = workloads.get(name).graph()
    off = torch.from_numpy(g.offsets).pin_memory()
    cols = torch.from_numpy(g.cols).pin_memory()
    lab = None if g.labels is None else torch.from_numpy(g.labels.view(np.int32)).pin_memory()
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G = gsm.gsm_load_graph(g.num_nodes, off, cols, lab, device=0)
        t1 = time.perf_counter()
        G.free()
        print(f"{name} load {rep}: {1e3 * (t1 - t0):.1f} ms", file=sys.stderr, flush=True)
