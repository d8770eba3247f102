"""GSM_TRACE=1 of a few small random-walk queries (host allocations / syncs / chunks per match)."""
import os
import sys

os.environ["GSM_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gsm_inputs as gi  # noqa: E402
from paper_2003_01527_b200 import gsm  # noqa: E402

base = gi.rmat(15, 8, 1)
g = base.with_labels(gi.zipf_labels(base.num_nodes, 20, 1), tag="-Z20")
G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0)
for k in (4, 5):
    q = gi.random_walk_query(g, k, 2 * k - 3, seed=1000 + k)
    for rep in range(3):
        r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, mode=gsm.GSM_MODE_COUNT, flags=gsm.GSM_FLAG_PROFILE)
        print(q.name, r.count, {k2: round(v, 3) for k2, v in r.ms.items()}, r.num_chunks, r.kernel_launches, flush=True)
G.free()
