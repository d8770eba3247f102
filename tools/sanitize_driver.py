"""Small matches that exercise every hot kernel once, for compute-sanitizer
(memcheck / racecheck / synccheck): clique kernels (warp, shared-memory CTA, global
slab, hub lookups), pair tail (thread + warp pass), fused tail (+ block overflow),
generic expand (plain + compressed + look-ahead), count walk, ENUMERATE finalize."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gsm_inputs as gi  # noqa: E402
from paper_2003_01527_b200 import gsm  # noqa: E402


def m(G, q, **kw):
    r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, **kw)
    if r.num_rows:
        r.free()
    return r.count


def main():
    g = gi.random_gnp(700, 1, 2, 7)  # dense: |N+(u)| up to ~350 (CTA buckets)
    G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, None, validate=True)
    for q in (gi.query("K3"), gi.query("K4")):
        print(q.name, m(G, q))
    G.free()
    os.environ["GSM_ORDER"] = "1"  # approximate degeneracy order (k_adg_* at load)
    G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, None)
    print("K4 order1", m(G, gi.query("K4")))
    G.free()
    del os.environ["GSM_ORDER"]
    os.environ["GSM_NHASH_MIN"] = "1"  # hashed N+(v) lookups in every clique row
    os.environ["GSM_CLIQUE_NH_STREAM"] = "0"
    G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, None)
    print("K4 nh", m(G, gi.query("K4")), "K3 nh", m(G, gi.query("K3")))
    G.free()
    del os.environ["GSM_NHASH_MIN"], os.environ["GSM_CLIQUE_NH_STREAM"]
    os.environ["GSM_HUB_BITS"] = "0"
    os.environ["GSM_CLIQUE_DSMEM"] = "64"  # global-slab kernel
    G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, None)
    print("K4 slab", m(G, gi.query("K4")))
    G.free()
    del os.environ["GSM_CLIQUE_DSMEM"], os.environ["GSM_HUB_BITS"]
    h = gi.rmat(11, 8, seed=3).with_labels(gi.uniform_labels(2048, 3, 3))
    H = gsm.gsm_load_graph(h.num_nodes, h.offsets, h.cols, h.labels)
    for q in (gi.query("house", [0, 1, 2, 0, 1]), gi.query("P4", [0, 1, 1, 0]), gi.query("C4")):
        print(q.name, m(H, q), m(H, q, mode=gsm.GSM_MODE_ENUMERATE),
              m(H, q, mode=gsm.GSM_MODE_ENUMERATE, flags=gsm.GSM_FLAG_COMPRESSED_PARTIALS, lookahead=2,
                mem_budget_bytes=1 << 16))
    os.environ["GSM_PAIR_THREAD_MAX"] = "0"
    print("pair warp", m(H, gi.query("house", [0, 1, 2, 0, 1])))
    os.environ["GSM_CLIQUE"] = "0"
    os.environ["GSM_TAIL_CAP"] = "64"
    os.environ["GSM_TAIL_BLOCK_CAP"] = "256"
    print("tail", m(H, gi.query("K4")))
    H.free()


if __name__ == "__main__":
    main()
