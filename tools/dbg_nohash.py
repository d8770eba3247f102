import os, sys
sys.path.insert(0, os.getcwd())
import gsm_inputs as gi, oracle
from paper_2003_01527_b200 import gsm
g = gi.rmat(10, 16, seed=12)
G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, None, device=0)
ref = oracle.match(g, gi.query("K3"), count_only=True)[0]
print("oracle", ref)
for env in [{}, {"GSM_CLIQUE_HASH": "0"}, {"GSM_CLIQUE_HASH": "0", "GSM_CLIQUE_WARP": "0"}, {"GSM_CLIQUE_HASH": "0", "GSM_CLIQUE_DSMEM": "64"},
            {"GSM_CLIQUE_HASH": "0", "GSM_CLIQUE_STREAM": "0"}, {"GSM_CLIQUE_HASH": "0", "GSM_CLIQUE_STREAM": "100000000"}]:
    for k in ["GSM_CLIQUE_HASH", "GSM_CLIQUE_WARP", "GSM_CLIQUE_DSMEM", "GSM_CLIQUE_STREAM"]:
        os.environ.pop(k, None)
    os.environ.update(env)
    r = gsm.gsm_match(G, 3, gi.query("K3").edges, None, mode=gsm.GSM_MODE_COUNT)
    print(env, r.count, r.count == ref)
