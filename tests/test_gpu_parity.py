"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element on the same seeded inputs.  Integer work => bit-exact: equal counts
and identical sorted row lists.  Unique mode has several valid
representative sets, so it is compared after canonicalisation f -> min_σ f∘σ
(SURVEY §8(c) amb. 9/13) plus a check that the GPU rows are valid embeddings."""
import json
import os

import numpy as np
import pytest

import gsm_inputs as gi
import oracle
from oracle import closed_forms as cf
from paper_2003_01527_b200 import gsm

from gpu_helpers import assert_rows_equal, is_sorted_unique, load, run

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def check_all_modes(g, q, G=None, what="", budget=0):
    own = G is None
    if own:
        G = load(g)
    try:
        cnt, ref = oracle.match(g, q)
        aut = oracle.automorphisms(q)
        kw = {"mem_budget_bytes": budget} if budget else {}
        # all embeddings (symmetric search + Aut expansion)
        c, rows, r = run(G, q, "enumerate", **kw)
        assert c == cnt, (what, "all", c, cnt)
        assert_rows_equal(rows, ref, what + " all")
        c2, _, _ = run(G, q, "count", **kw)
        assert c2 == cnt, (what, "count", c2, cnt)
        # direct search, no ID constraints
        c3, rows3, _ = run(G, q, "enumerate", flags=gsm.GSM_FLAG_NO_SYMMETRY, **kw)
        assert c3 == cnt
        assert_rows_equal(rows3, ref, what + " nosym")
        # one per orbit
        cu, rowsu, ru = run(G, q, "enumerate", flags=gsm.GSM_FLAG_UNIQUE, **kw)
        uniq = oracle.unique(ref, aut)
        assert cu == len(uniq) and ru.automorphisms == len(aut), (what, cu, len(uniq))
        assert is_sorted_unique(rowsu)
        if len(rowsu):
            # canonical forms of the GPU representatives = the oracle's orbit set; with
            # cu == len(uniq) this also proves one representative per orbit, and each
            # representative is f∘σ of a valid embedding, hence valid itself
            assert_rows_equal(oracle.unique(rowsu, aut), uniq, what + " unique(canonical)")
        cuc, _, _ = run(G, q, "count", flags=gsm.GSM_FLAG_UNIQUE, **kw)
        assert cuc == len(uniq)
    finally:
        if own:
            G.free()


def test_spec_golden_on_gpu():
    ex = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))["examples"]
    for e in ex:
        d, qd = e["data"], e["query"]
        g = gi.from_edge_list(d["num_nodes"], d["edges"])
        if "labels" in d:
            g = g.with_labels(np.asarray(d["labels"], np.uint32))
        q = gi.Query(qd["num_nodes"], [tuple(x) for x in qd["edges"]], qd.get("labels"))
        G = load(g)
        try:
            c, rows, r = run(G, q, "enumerate")
            assert c == e["all"], e["cite"]
            cu, rowsu, _ = run(G, q, "enumerate", flags=gsm.GSM_FLAG_UNIQUE)
            assert cu == e["unique"], e["cite"]
            if "unique_node_sets" in e:
                assert sorted(sorted(x) for x in rowsu.tolist()) == e["unique_node_sets"]
        finally:
            G.free()


def test_random_instances_match_oracle():
    """SPEC acceptance criterion 2: >= 200 instances, G(30,0.2) and
    G(50,0.1), unlabeled and 3 labels, connected 3-5-node queries."""
    n_inst = 0
    for seed in range(1, 26):
        for (n, pn, pd) in [(30, 1, 5), (50, 1, 10)]:
            g0 = gi.random_gnp(n, pn, pd, seed)
            for nl in (0, 3):
                g = g0.with_labels(gi.uniform_labels(n, 3, seed)) if nl else g0
                G = load(g)
                try:
                    for j in range(2):
                        k = 3 + (seed + j) % 3
                        q = gi.random_connected_query(k, (seed + j) % 3, seed * 101 + j * 7 + n, nl)
                        check_all_modes(g, q, G, what=f"seed{seed} n{n} nl{nl} {q.name}")
                        n_inst += 1
                finally:
                    G.free()
    assert n_inst >= 200


@pytest.mark.parametrize("qname", ["K2", "K3", "P3", "P4", "S3", "C4", "K4", "C5", "house", "diamond", "tailed_triangle"])
def test_named_queries_on_random_graphs(qname):
    for seed in (1, 2):
        g = gi.random_gnp(60, 1, 6, seed)
        check_all_modes(g, gi.query(qname), what=f"{qname} s{seed}")
    g = gi.rmat(8, 8, seed=4)
    check_all_modes(g, gi.query(qname), what=f"{qname} rmat8")


def test_labeled_named_queries():
    g = gi.rmat(11, 8, seed=5).with_labels(gi.uniform_labels(2048, 3, 5))
    G = load(g)
    try:
        for qname, ql in [("P4", [0, 1, 2, 0]), ("P4", [1, 2, 2, 1]), ("S3", [0, 1, 1, 2]), ("S3", [0, 1, 2, 2]),
                          ("house", [0, 1, 2, 0, 1]), ("house", [0, 0, 1, 1, 2]), ("K3", [0, 0, 1]),
                          ("C4", [0, 1, 0, 1]), ("K4", [0, 0, 0, 0])]:
            check_all_modes(g, gi.query(qname, ql), G, what=f"{qname}{ql}")
    finally:
        G.free()


@pytest.mark.parametrize("tail", ["0", "1", "cap64", "cap64block256"])
def test_fused_tail_matches_generic_path(tail, monkeypatch):
    """The fused last-two-positions kernel (COUNT mode, clique-like tails) against the
    oracle, with the fusion disabled, enabled, and enabled with a tiny per-warp buffer
    (forcing the overflow hand-back to the generic path)."""
    monkeypatch.setenv("GSM_FUSED_TAIL", "0" if tail == "0" else "1")
    if tail.startswith("cap64"):
        monkeypatch.setenv("GSM_TAIL_CAP", "64")
    if tail == "cap64block256":
        monkeypatch.setenv("GSM_TAIL_BLOCK_CAP", "256")
    g = gi.rmat(10, 16, seed=12).with_labels(gi.uniform_labels(1024, 2, 12))
    G = load(g)
    try:
        for q in [gi.query("K3"), gi.query("K4"), gi.query("K3", [0, 0, 0]), gi.query("K3", [0, 0, 1]),
                  gi.query("K4", [1, 1, 1, 1]), gi.query("diamond"), gi.query("tailed_triangle"), gi.query("K2"),
                  gi.Query(5, [(a, b) for a in range(5) for b in range(a + 1, 5)], None, "K5")]:
            cnt, _ = oracle.match(g, q, count_only=True)
            for flags in (0, gsm.GSM_FLAG_UNIQUE, gsm.GSM_FLAG_NO_SYMMETRY):
                c, _, r = run(G, q, "count", flags=flags)
                want = cnt if flags != gsm.GSM_FLAG_UNIQUE else cnt // r.automorphisms
                assert c == want, (tail, q.name, flags, c, want)
    finally:
        G.free()


@pytest.fixture(scope="module")
def dense_gnp():
    """G(1200, 1/2): min degree > 512, so N+(u) of the lowest-ranked vertices exceeds 512
    (the shared-memory CTA bucket above 512); exact counts from the oracle's independent
    degree-ordered clique counters."""
    g = gi.random_gnp(1200, 1, 2, 7)
    return g, oracle.count_triangles(g), oracle.count_k4(g)


@pytest.mark.parametrize("variant", ["default", "nohub", "hubmix", "hubmix_warp0", "warp0", "dsmem64", "search",
                                     "stream", "nohash", "handback", "off", "nh_all", "nh_all_warp0", "nh_dsmem64",
                                     "ranges", "ranges_dsmem64", "occ1", "occ0", "eagerck"])
def test_clique_bitmap_path(variant, dense_gnp, monkeypatch):
    """K3/K4 COUNT through the per-root local-bitmap kernels (gsm_clique.cu) in every
    bucket (warp per root; CTA with shared memory; CTA with a global slab via a tiny
    GSM_CLIQUE_DSMEM) and both row-construction strategies, against the oracle (DFS on an
    R-MAT graph, independent clique counters on a dense G(n, p)).  "off" = the fused-tail
    path (GSM_CLIQUE=0) on the same inputs; "handback" = roots beyond GSM_CLIQUE_DMAX handed
    back to the breadth-first path inside the same call.  Hub bitmap (read at load time):
    "default" = every vertex of these small graphs is a hub, so every row is built by
    bitmap lookups; "hubmix" = only the top 256 ranks are hubs (lookup, stream and search
    rows mixed in one root); every other variant switches the bitmap off (GSM_HUB_BITS=0)
    so its stream / search / bucket path is the one under test.  Hashed N+(v) tables (read at
    load time, GSM_NHASH_MIN): "nh_all*" give every non-empty list a table and force every row
    onto table lookups (GSM_CLIQUE_NH_STREAM=0) in the warp, shared-memory and global-slab
    kernels; the stream / search variants switch the tables off."""
    env = {"nohub": {}, "hubmix": {"GSM_HUB_BITS": "256"},
           "hubmix_warp0": {"GSM_HUB_BITS": "256", "GSM_CLIQUE_WARP": "0", "GSM_CLIQUE_DSMEM": "64"},
           "warp0": {"GSM_CLIQUE_WARP": "0"}, "dsmem64": {"GSM_CLIQUE_DSMEM": "64"},
           "search": {"GSM_CLIQUE_STREAM": "0"}, "stream": {"GSM_CLIQUE_STREAM": "1000000000"},
           "nohash": {"GSM_CLIQUE_HASH": "0"}, "handback": {"GSM_CLIQUE_DMAX": "64"},
           "off": {"GSM_CLIQUE": "0"},
           "nh_all": {"GSM_NHASH_MIN": "1", "GSM_CLIQUE_NH_STREAM": "0"},
           "nh_all_warp0": {"GSM_NHASH_MIN": "1", "GSM_CLIQUE_NH_STREAM": "0", "GSM_CLIQUE_WARP": "0"},
           "nh_dsmem64": {"GSM_NHASH_MIN": "1", "GSM_CLIQUE_NH_STREAM": "0", "GSM_CLIQUE_DSMEM": "64"},
           "ranges": {"GSM_CLIQUE_RANGES": "1"},
           "ranges_dsmem64": {"GSM_CLIQUE_RANGES": "1", "GSM_CLIQUE_DSMEM": "64"},
           "occ1": {"GSM_CLIQUE_OCC": "1"}, "occ0": {"GSM_CLIQUE_OCC": "0"}, "eagerck": {"GSM_CLIQUE_LAZYCK": "0"}}.get(variant, {})
    if variant not in ("default", "hubmix", "hubmix_warp0"):
        env = {"GSM_HUB_BITS": "0", **env}
    if variant not in ("default", "hubmix", "hubmix_warp0") and not variant.startswith("nh_"):
        env = {"GSM_NHASH_MIN": "0", **env}
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = gi.rmat(10, 16, seed=12)
    G = load(g)
    try:
        for q in [gi.query("K3"), gi.query("K4")]:
            cnt, _ = oracle.match(g, q, count_only=True)
            c, _, r = run(G, q, "count")
            assert c == cnt, (variant, q.name, c, cnt)
            assert (r.prof["clique"]["launches"] > 0) == (variant != "off"), r.prof
            cu, _, _ = run(G, q, "count", flags=gsm.GSM_FLAG_UNIQUE)
            assert cu * r.automorphisms == cnt
    finally:
        G.free()
    gd, T, K4 = dense_gnp
    G = load(gd)
    try:
        assert run(G, gi.query("K3"), "count", flags=gsm.GSM_FLAG_UNIQUE)[0] == T, variant
        assert run(G, gi.query("K4"), "count", flags=gsm.GSM_FLAG_UNIQUE)[0] == K4, variant
        c4, _, r4 = run(G, gi.query("K4"), "count")
        assert c4 == 24 * K4, variant
        if variant == "handback":  # roots with |N+(u)| > 64 went to the breadth-first path
            assert r4.prof["tail"]["launches"] + r4.prof["expand"]["launches"] > 0, r4.prof
    finally:
        G.free()


@pytest.mark.parametrize("pair", ["1", "warp", "0", "plan_groups", "nohub", "swap1", "swap1_warp", "nolidx", "lidx_all"])
def test_pair_tail(pair, monkeypatch):
    """COUNT mode with the last two positions an independent pair (k_pair: |Cp||Cq| - |Cp∩Cq|)
    against the oracle's count, labeled and unlabeled, with and without symmetry; "0" =
    the pair ordering disabled (GSM_PAIR_TAIL=0) on the same inputs; "warp" = every row through
    the warp-per-row kernel (no thread-per-row pass)."""
    if pair == "plan_groups":  # row plans by lane groups instead of one thread per row (the default)
        monkeypatch.setenv("GSM_PLAN_GROUPS", "1")
    # label index of the keyed lists (read at load): "nolidx" = binary searches for every label
    # segment, "lidx_all" = every vertex indexed
    if pair == "nolidx":
        monkeypatch.setenv("GSM_LIDX_MIN", "0")
    if pair == "lidx_all":
        monkeypatch.setenv("GSM_LIDX_MIN", "1")
    # membership tests: these small graphs are all hubs by default (bitmap tests); "nohub" = binary
    # searches only; "swap1" = search the image in N(v) whenever v's list is the shorter one
    if pair in ("nohub", "swap1", "swap1_warp"):
        monkeypatch.setenv("GSM_HUB_BITS", "0")
    if pair.startswith("swap1"):
        monkeypatch.setenv("GSM_MEMBER_SWAP", "1")
    if pair == "swap1_warp":
        monkeypatch.setenv("GSM_PAIR_THREAD_MAX", "0")
    monkeypatch.setenv("GSM_PAIR_TAIL", "0" if pair == "0" else "1")
    if pair == "warp":
        monkeypatch.setenv("GSM_PAIR_THREAD_MAX", "0")
    g = gi.rmat(9, 8, seed=31).with_labels(gi.uniform_labels(512, 3, 31))
    G = load(g)
    try:
        qs = [gi.query("P3"), gi.query("P4"), gi.query("S3"), gi.query("house"), gi.query("tailed_triangle"),
              gi.query("P4", [0, 1, 2, 0]), gi.query("P4", [0, 1, 1, 2]), gi.query("S3", [0, 1, 1, 2]),
              gi.query("house", [0, 1, 2, 0, 1]), gi.query("house", [0, 0, 1, 1, 2]), gi.query("C4", [0, 1, 0, 2])]
        qs += [gi.random_connected_query(k, e, seed, 3) for (k, e, seed) in [(4, 1, 1), (5, 1, 2), (5, 2, 3), (6, 2, 4)]]
        used = 0
        for q in qs:  # unlabeled queries ignore the data labels
            cnt, _ = oracle.match(g, q, count_only=True)
            for flags in (0, gsm.GSM_FLAG_NO_SYMMETRY):
                c, _, r = run(G, q, "count", flags=flags)
                assert c == cnt, (pair, q.name, q.labels, flags, c, cnt)
                a, b = r.order[-2], r.order[-1]
                adj = any({a, b} == {x, y} for x, y in q.edges)
                used += (not adj) and r.prof["tail"]["launches"] > 0
        assert (used > 0) == (pair != "0"), used
    finally:
        G.free()


def test_lookahead_results_unchanged():
    """k-look-ahead: a necessary condition, so the sorted
    row lists and counts are identical for lookahead = 0, 1, 2 (SPEC criterion 4) on
    random labeled / unlabeled instances and named queries, in every mode."""
    n_inst = 0
    for seed in range(1, 16):
        g0 = gi.random_gnp(40, 1, 6, 300 + seed)
        for nl in (0, 3):
            g = g0.with_labels(gi.uniform_labels(40, 3, seed)) if nl else g0
            G = load(g)
            try:
                for j in range(2):
                    q = gi.random_connected_query(4 + (seed + j) % 3, (seed + j) % 3, seed * 31 + j, nl)
                    cnt, ref = oracle.match(g, q)
                    for la in (1, 2):
                        c, rows, _ = run(G, q, "enumerate", lookahead=la)
                        assert c == cnt, (q.name, la)
                        assert_rows_equal(rows, ref, f"{q.name} la={la}")
                        for flags in (0, gsm.GSM_FLAG_UNIQUE, gsm.GSM_FLAG_NO_SYMMETRY):
                            cc, _, r = run(G, q, "count", flags=flags, lookahead=la)
                            want = cnt if flags != gsm.GSM_FLAG_UNIQUE else cnt // r.automorphisms
                            assert cc == want, (q.name, la, flags)
                    n_inst += 1
            finally:
                G.free()
    assert n_inst >= 60


def test_lookahead_prunes_on_road_like_graph():
    """SPEC criterion 4: summed intermediate rows satisfy rows(2) <= rows(1) <= rows(0)
    on every instance, strictly on the sparse chain-with-tails graph (road_central's low
    average degree, where Table 2 shows the largest look-ahead gain)."""
    graphs = [gi.chain_with_tails(400, 6, seed=3), gi.grid(40, 40, seed=5), gi.rmat(10, 4, seed=8)]
    queries = [gi.query("P4"), gi.query("tailed_triangle"), gi.query("S3"), gi.query("C4"), gi.query("house"),
               gi.Query(5, [(0, 1), (1, 2), (2, 3), (3, 4)], None, "P5"),
               gi.Query(5, [(0, 1), (1, 2), (2, 3), (1, 4)], None, "chair")]
    strict = {}
    for gi_, g in enumerate(graphs):
        G = load(g)
        try:
            for q in queries:
                cnt, _ = oracle.match(g, q, count_only=True)
                rows = []
                for la in (0, 1, 2):
                    c, _, r = run(G, q, "enumerate", lookahead=la)
                    r_rows = sum(r.level_rows[1:q.num_nodes - 1])
                    assert c == cnt, (g.name, q.name, la)
                    rows.append(r_rows)
                assert rows[2] <= rows[1] <= rows[0], (g.name, q.name, rows)
                strict[(gi_, q.name)] = rows[1] < rows[0] or rows[2] < rows[1]
        finally:
            G.free()
    assert any(v for (gi_, _), v in strict.items() if gi_ == 0), strict


def test_ne_refinement_is_sound():
    """NE filter + refinement rounds (Alg. 1 lines 7-8): results
    identical for R = 0..3; |C(u)| non-increasing in R and never below the number of
    distinct images of u in the oracle's embeddings (filter soundness)."""
    g = gi.rmat(11, 8, seed=21).with_labels(gi.uniform_labels(2048, 3, 21))
    G = load(g)
    try:
        for q in [gi.query("K3"), gi.query("K4"), gi.query("house", [0, 1, 2, 0, 1]), gi.query("P4", [1, 2, 2, 1]),
                  gi.query("C4"), gi.query("S3", [0, 1, 1, 2])]:
            cnt, ref = oracle.match(g, q)
            images = [len(np.unique(ref[:, u])) for u in range(q.num_nodes)]
            prev = None
            for R in range(4):
                c, rows, r = run(G, q, "enumerate", refine_rounds=R)
                assert c == cnt, (q.name, R)
                assert_rows_equal(rows, ref, f"{q.name} R={R}")
                assert run(G, q, "count", refine_rounds=R)[0] == cnt
                for u in range(q.num_nodes):
                    assert r.candidates[u] >= images[u], (q.name, R, u)
                    if prev is not None:
                        assert r.candidates[u] <= prev[u]
                prev = r.candidates
    finally:
        G.free()


def test_random_walk_queries_zipf_labels():
    """Paper-shaped queries (random-walk queries on power-law labels):
    GPU == oracle (count and rows) for 5..12-node queries; every query has >= 1 embedding
    (the walk's own vertices)."""
    g = gi.rmat(9, 8, seed=41).with_labels(gi.zipf_labels(512, 20, 41))  # oracle < 2 s per query
    G = load(g)
    try:
        for k, m in [(5, 6), (6, 8), (8, 12), (10, 16), (12, 22)]:
            for s in range(3):
                q = gi.random_walk_query(g, k, m, seed=97 * k + s)
                cnt, ref = oracle.match(g, q)
                assert cnt >= 1
                c, rows, _ = run(G, q, "enumerate")
                assert c == cnt, (q.name, c, cnt)
                assert_rows_equal(rows, ref, q.name)
                assert run(G, q, "count")[0] == cnt
    finally:
        G.free()


def test_closed_forms_on_gpu():
    for n in (5, 8):
        G = load(gi.complete(n))
        try:
            for qname in ["K3", "P4", "C4", "K4", "house"]:
                q = gi.query(qname)
                assert run(G, q)[0] == cf.complete_graph(n, q.num_nodes)
        finally:
            G.free()
    G = load(gi.petersen())
    try:
        assert run(G, gi.query("C5"))[0] == 120
        assert run(G, gi.query("K3"))[0] == 0
    finally:
        G.free()
    gg = gi.grid(80, 60, seed=3)
    G = load(gg)
    try:
        assert run(G, gi.query("K4"))[0] == cf.grid_diag_k4(gg.meta["d2"])
        assert run(G, gi.query("K3"))[0] == cf.grid_diag_k3(gg.meta["d1"], gg.meta["d2"])
        assert run(G, gi.query("C4"))[0] == cf.cycle4(gg)
    finally:
        G.free()


def test_candidate_counts_match_cpu_predicate():
    """K1 filter: |C(u)| = #{v : label(v) = label_Q(u) and deg(v) >= deg_Q(u)}."""
    g = gi.rmat(12, 8, seed=9).with_labels(gi.uniform_labels(4096, 4, 9))
    deg = np.diff(g.offsets)
    G = load(g)
    try:
        for qname, ql in [("S3", [0, 1, 2, 3]), ("house", [1, 1, 2, 3, 0]), ("K4", None)]:
            q = gi.query(qname, ql)
            _, _, r = run(G, q)
            qdeg = np.zeros(q.num_nodes, int)
            for a, b in q.edges:
                qdeg[a] += 1
                qdeg[b] += 1
            for u in range(q.num_nodes):
                lab_ok = np.ones(g.num_nodes, bool) if ql is None else (g.labels == ql[u])
                assert r.candidates[u] == int(np.sum(lab_ok & (deg >= qdeg[u]))), (qname, u)
    finally:
        G.free()


@pytest.mark.parametrize("variant", ["plain_budget", "budget", "tailcap", "pair_warp"])
def test_compressed_partials(variant, monkeypatch):
    """Compressed partial results (level-wise (parent row, vertex) pairs; PAPER P:136/P:151,
    SURVEY §8(f) row 3): sorted row lists and counts identical to the oracle in every mode,
    under tiny budgets (chains across many chunks), with the fused tail's overflow hand-back
    and the pair tail's warp pass reading compressed rows; and the stored bytes of every
    intermediate width w >= 3 shrink from 4w to 8 per partial result."""
    if variant == "tailcap":
        monkeypatch.setenv("GSM_TAIL_CAP", "64")
        monkeypatch.setenv("GSM_TAIL_BLOCK_CAP", "256")
    if variant == "pair_warp":
        monkeypatch.setenv("GSM_PAIR_THREAD_MAX", "0")
    budget = 0 if variant == "plain_budget" else 1 << 16
    g = gi.rmat(9, 8, seed=31).with_labels(gi.uniform_labels(512, 2, 31))
    G = load(g)
    try:
        qs = [gi.query("house"), gi.query("K4"), gi.query("P4", [0, 1, 1, 0]), gi.query("C5"),
              # labeled: the unlabeled C6+chord has 1.7e9 embeddings here (40 GB of rows, ~550 s per variant)
              gi.Query(6, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 0), (0, 3)], [0, 1, 0, 1, 0, 1], "C6+chord"),
              gi.random_connected_query(6, 2, 77, 2)]
        for q in qs:
            cnt, ref = oracle.match(g, q)
            c0, rows0, r0 = run(G, q, "enumerate", mem_budget_bytes=budget)
            c1, rows1, r1 = run(G, q, "enumerate", flags=gsm.GSM_FLAG_COMPRESSED_PARTIALS, mem_budget_bytes=budget)
            assert r1.compressed and not r0.compressed
            assert c0 == c1 == cnt, (variant, q.name)
            assert_rows_equal(rows1, ref, f"{q.name} compressed")
            for flags in (0, gsm.GSM_FLAG_UNIQUE, gsm.GSM_FLAG_NO_SYMMETRY):
                cc, _, r = run(G, q, "count", flags=flags | gsm.GSM_FLAG_COMPRESSED_PARTIALS,
                               mem_budget_bytes=budget)
                want = cnt if flags != gsm.GSM_FLAG_UNIQUE else cnt // r.automorphisms
                assert cc == want, (variant, q.name, flags)
            k = q.num_nodes
            for w in range(2, k - 1):  # stored intermediate widths w+1 = 3 .. k-1
                assert r0.level_rows[w] == r1.level_rows[w]
                assert r0.level_frontier_bytes[w] == 4 * (w + 1) * r0.level_rows[w]
                assert r1.level_frontier_bytes[w] == 8 * r1.level_rows[w]
    finally:
        G.free()


def test_filter_masks_bit_exact():
    """K1 (vectorised filter): the candidate mask of EVERY vertex equals the CPU predicate
    label(v) = label_Q(u) and deg(v) >= deg_Q(u) bit for bit — on labeled and
    unlabeled graphs whose vertex counts are not multiples of 4 (the scalar tail) — and the
    refined masks are subsets that keep every vertex some oracle embedding uses (soundness)."""
    cases = [(gi.rmat(12, 8, seed=9).with_labels(gi.uniform_labels(4096, 4, 9)), [("S3", [0, 1, 2, 3]),
              ("house", [1, 1, 2, 3, 0]), ("K4", None)]),
             (gi.erdos_renyi(1003, 4000, 2), [("K3", None), ("P4", None), ("C5", None)]),
             (gi.random_gnp(37, 1, 4, 5).with_labels(gi.uniform_labels(37, 3, 5)), [("tailed_triangle", [0, 1, 2, 0])])]
    for g, qs in cases:
        deg = np.diff(g.offsets)
        G = load(g)
        try:
            for qname, ql in qs:
                q = gi.query(qname, ql)
                qdeg = np.zeros(q.num_nodes, int)
                for a, b in q.edges:
                    qdeg[a] += 1
                    qdeg[b] += 1
                want = np.zeros(g.num_nodes, np.uint32)
                for u in range(q.num_nodes):
                    lab_ok = np.ones(g.num_nodes, bool) if ql is None else (g.labels == ql[u])
                    want |= ((lab_ok & (deg >= qdeg[u])).astype(np.uint32) << np.uint32(u))
                got = gsm.gsm_filter_candidates(G, q.num_nodes, q.edges, q.labels)
                np.testing.assert_array_equal(got, want, err_msg=qname)
                _, _, r = run(G, q)
                for u in range(q.num_nodes):
                    assert r.candidates[u] == int(np.sum((want >> np.uint32(u)) & 1)), (qname, u)
                _, ref = oracle.match(g, q)
                for R in (1, 2):
                    ref_mask = gsm.gsm_filter_candidates(G, q.num_nodes, q.edges, q.labels, refine_rounds=R)
                    assert np.all((ref_mask & ~want) == 0), (qname, R)
                    for u in range(q.num_nodes):
                        assert np.all((ref_mask[ref[:, u]] >> np.uint32(u)) & 1), (qname, R, u)
        finally:
            G.free()


def test_chunking_invariance():
    """Tiny memory budgets force many chunks per level; results must not change."""
    g = gi.rmat(9, 8, seed=2)
    G = load(g)
    try:
        for qname in ["K4", "C4", "diamond"]:
            q = gi.query(qname)
            cnt, ref = oracle.match(g, q)
            for budget in (64 << 10, 1 << 20, 0):
                c, rows, r = run(G, q, "enumerate", mem_budget_bytes=budget)
                assert c == cnt
                assert_rows_equal(rows, ref, f"{qname} budget {budget}")
                c2, _, r2 = run(G, q, "count", mem_budget_bytes=budget)
                assert c2 == cnt
            assert r.num_chunks >= 1
            # the small budget really chunks the breadth-first frontier (ENUMERATE; COUNT-mode
            # cliques take the per-root bitmap path, which has no frontier to chunk)
            r_small = run(G, q, "enumerate", mem_budget_bytes=64 << 10)[2]
            assert r_small.num_chunks > r.num_chunks
    finally:
        G.free()


def test_shard_invariance():
    """P root shards run sequentially on one GPU: counts add up, rows union = all rows."""
    g = gi.rmat(10, 8, seed=3).with_labels(gi.uniform_labels(1024, 2, 3))
    G = load(g)
    try:
        for q in [gi.query("K3"), gi.query("P4", [0, 1, 1, 0]), gi.query("K4")]:
            cnt, ref = oracle.match(g, q)
            for P in (2, 3, 8):
                tot = 0
                parts = []
                for s in range(P):
                    c, rows, _ = run(G, q, "enumerate", shard_index=s, num_shards=P)
                    tot += c
                    parts.append(rows)
                assert tot == cnt
                assert_rows_equal(oracle.sort_rows(np.concatenate(parts)), ref, f"{q.name} P={P}")
    finally:
        G.free()


def test_level1_shard_invariance(monkeypatch):
    """GSM_FLAG_SHARD_LEVEL1 (SURVEY §8(e) skew mitigation): P shards of the level-1 pairs run
    sequentially on one GPU — counts add up to the oracle's, the rows' union is the oracle's
    list, each shard really was pair-sharded (where level 1 is a breadth-first expand) and a
    single hub root's embeddings are split over several shards."""
    g = gi.rmat(10, 8, seed=3).with_labels(gi.uniform_labels(1024, 2, 3))
    G = load(g)
    F = gsm.GSM_FLAG_SHARD_LEVEL1
    try:
        for q in [gi.query("P4", [0, 1, 1, 0]), gi.query("house", [0, 1, 0, 1, 0]), gi.query("C4"), gi.query("K4")]:
            cnt, ref = oracle.match(g, q)
            for P in (2, 3, 8):
                tot = tot_c = 0
                parts = []
                for s in range(P):
                    c, rows, r = run(G, q, "enumerate", flags=F, shard_index=s, num_shards=P)
                    assert r.level1_sharded
                    cc, _, rc = run(G, q, "count", flags=F, shard_index=s, num_shards=P)
                    if rc.level1_sharded:  # COUNT-mode K4 takes the root-sharded clique path
                        assert cc == c, (q.name, P, s)
                    tot += c
                    tot_c += cc
                    parts.append(rows)
                assert tot == cnt and tot_c == cnt
                assert_rows_equal(oracle.sort_rows(np.concatenate(parts)), ref, f"{q.name} P={P} level1")
        # the COUNT-mode clique path stays root-sharded (flag ignored), still exact
        q = gi.query("K4")
        cnt, _ = oracle.match(g, q, count_only=True)
        tot = 0
        for s in range(4):
            c, _, r = run(G, q, "count", flags=F, shard_index=s, num_shards=4)
            assert not r.level1_sharded and r.prof["clique"]["launches"] > 0
            tot += c
        assert tot == cnt
    finally:
        G.free()


def test_root_subset_sampling():
    g = gi.rmat(12, 16, seed=6).with_labels(gi.uniform_labels(4096, 3, 6))
    G = load(g)
    try:
        rng = np.random.default_rng(1)
        roots = np.unique(rng.integers(0, 4096, 300)).astype(np.int32)
        for q in [gi.query("house", [0, 1, 2, 0, 1]), gi.query("K3"), gi.query("C4", [0, 1, 0, 1])]:
            cnt, ref = oracle.match(g, q, roots=roots)
            c, rows, _ = run(G, q, "enumerate", root_subset=roots)
            assert c == cnt
            assert_rows_equal(rows, ref, q.name)
    finally:
        G.free()


def test_relabel_invariance():
    g = gi.rmat(10, 8, seed=8)
    perm = np.random.default_rng(3).permutation(g.num_nodes).astype(np.int32)
    src = np.repeat(np.arange(g.num_nodes), np.diff(g.offsets))
    g2 = gi.csr_from_edges(g.num_nodes, perm[src], perm[g.cols])
    G1, G2 = load(g), load(g2)
    try:
        for qname in ["K3", "C4", "P4"]:
            q = gi.query(qname)
            _, r1, _ = run(G1, q, "enumerate")
            _, r2, _ = run(G2, q, "enumerate")
            assert_rows_equal(oracle.sort_rows(perm[r1]), r2, qname)
    finally:
        G1.free()
        G2.free()


def test_edge_cases():
    # single vertex query -> n; K2 -> 2m; k > n -> 0; label absent -> 0
    g = gi.random_gnp(20, 1, 4, 1)
    G = load(g)
    try:
        assert run(G, gi.Query(1, [], None))[0] == 20
        c, rows, _ = run(G, gi.Query(1, [], None), "enumerate")
        assert rows[:, 0].tolist() == list(range(20))
        assert run(G, gi.query("K2"))[0] == 2 * g.num_edges
        with pytest.raises(gsm.GsmError) as e:
            run(G, gi.Query(3, [(0, 1)], None))
        assert e.value.status == 3  # disconnected query
        with pytest.raises(gsm.GsmError) as e:
            run(G, gi.query("K3", [0, 0, 0]))
        assert e.value.status == 1  # labels on an unlabeled graph
        with pytest.raises(gsm.GsmError):
            run(G, gi.Query(3, [(0, 1), (1, 1)], None))  # self-loop in Q
        with pytest.raises(gsm.GsmError):
            run(G, gi.Query(33, [(i, i + 1) for i in range(32)], None))  # k > 32
    finally:
        G.free()
    G = load(gi.complete(4))
    try:
        assert run(G, gi.query("C5"))[0] == 0  # k > n
    finally:
        G.free()
    gl = gi.complete(5).with_labels(np.array([1, 1, 2, 2, 2], np.uint32))
    G = load(gl)
    try:
        assert run(G, gi.query("K3", [1, 2, 7]))[0] == 0
        c, rows, _ = run(G, gi.query("K3", [1, 2, 7]), "enumerate")
        assert c == 0 and rows.shape[0] == 0
    finally:
        G.free()
    # graph without edges, isolated vertices
    ge = gi.csr_from_edges(10, np.zeros(0, np.int32), np.zeros(0, np.int32))
    G = load(ge)
    try:
        assert run(G, gi.query("K2"))[0] == 0
        assert run(G, gi.Query(1, [], None))[0] == 10
    finally:
        G.free()


def test_invalid_graphs_rejected():
    g = gi.complete(4)
    bad_unsorted = g.cols.copy()
    bad_unsorted[0], bad_unsorted[1] = bad_unsorted[1], bad_unsorted[0]
    cases = [
        (g.offsets, bad_unsorted),
        (g.offsets, np.where(g.cols == 3, 9, g.cols).astype(np.int32)),  # out of range
    ]
    # asymmetric: drop one direction
    off = np.array([0, 1, 1], np.int64)
    cases.append((off, np.array([1], np.int32)))
    # self-loop
    cases.append((np.array([0, 1], np.int64), np.array([0], np.int32)))
    for o, c in cases:
        with pytest.raises(gsm.GsmError) as e:
            gsm.gsm_load_graph(len(o) - 1, o, c, validate=True)
        assert e.value.status == 2
    with pytest.raises(gsm.GsmError) as e:
        gsm.gsm_load_graph(0, np.zeros(1, np.int64), np.zeros(0, np.int32))
    assert e.value.status == 2


def test_device_pointer_load_and_profile():
    import torch
    g = gi.rmat(12, 8, seed=1)
    off = torch.from_numpy(g.offsets).cuda()
    cols = torch.from_numpy(g.cols).cuda()
    G = gsm.gsm_load_graph(g.num_nodes, off, cols, None, device=0, validate=True)
    try:
        c, _, r = run(G, gi.query("K3"), flags=gsm.GSM_FLAG_PROFILE)
        assert c == 6 * oracle.count_triangles(g)
        hot = [r.prof[k] for k in ("expand", "tail", "clique")]
        assert sum(h["launches"] for h in hot) >= 1 and sum(h["ms"] for h in hot) > 0
        assert sum(h["alg_bytes"] for h in hot) > 0 and r.prof["filter"]["ms"] > 0
        rt = run(G, gi.query("K3"), "enumerate")[1]
        re = gsm.gsm_match(G, 3, gi.query("K3").edges, mode=gsm.GSM_MODE_ENUMERATE)
        t = re.rows_torch()
        assert t.is_cuda and t.shape[0] == c
        assert np.array_equal(t.cpu().numpy(), rt)
        re.free()
    finally:
        G.free()


@pytest.mark.parametrize("hub", ["hub", "nohub"])
def test_degeneracy_order(hub, dense_gnp, monkeypatch):
    """GSM_ORDER=1 (read at gsm_load_graph): data vertices ranked by an approximate
    degeneracy (peeling-round) order instead of (degree, id).  Any strict total order is a
    valid ≺ (SURVEY §8(c) amb. 9): every mode's rows equal the oracle's, the clique kernels'
    counts equal the independent clique counters."""
    monkeypatch.setenv("GSM_ORDER", "1")
    if hub == "nohub":
        monkeypatch.setenv("GSM_HUB_BITS", "0")
    g = gi.rmat(9, 8, seed=12)  # house: 4.3e7 rows (R-MAT-10 ef16: 1.5e9 — 20 min per variant)
    G = load(g)
    try:
        for qn in ["K3", "K4", "C4", "P4", "house"]:
            check_all_modes(g, gi.query(qn), G, f"order1 {qn}")
    finally:
        G.free()
    h = gi.rmat(11, 8, seed=3).with_labels(gi.uniform_labels(2048, 3, 3))
    H = load(h)
    try:
        check_all_modes(h, gi.query("house", [0, 1, 2, 0, 1]), H, "order1 labeled house")
    finally:
        H.free()
    gd, T, K4 = dense_gnp
    G = load(gd)
    try:
        assert run(G, gi.query("K3"), "count", flags=gsm.GSM_FLAG_UNIQUE)[0] == T
        assert run(G, gi.query("K4"), "count", flags=gsm.GSM_FLAG_UNIQUE)[0] == K4
    finally:
        G.free()


def test_merge_rows():
    """gsm_merge_rows (merge path): two sorted row blocks -> the sorted
    concatenation, element by element against oracle.sort_rows; empty sides, ragged sizes,
    equal rows across the blocks, widths 1..5."""
    import torch
    rng = np.random.default_rng(17)
    for w, na, nb, hi in [(1, 0, 5, 9), (3, 7, 0, 9), (2, 1000, 3, 4), (3, 12345, 54321, 50), (5, 200000, 150001, 1 << 24),
                          (4, 1, 1, 2)]:
        a = oracle.sort_rows(rng.integers(0, hi, size=(na, w)).astype(np.int32))
        b = oracle.sort_rows(rng.integers(0, hi, size=(nb, w)).astype(np.int32))
        ta = torch.from_numpy(a).cuda().reshape(na, w)
        tb = torch.from_numpy(b).cuda().reshape(nb, w)
        out = gsm.gsm_merge_rows(ta, tb).cpu().numpy()
        assert_rows_equal(out, oracle.sort_rows(np.concatenate([a, b]).reshape(-1, w)), f"merge w={w} {na}+{nb}")


@pytest.mark.parametrize("bigsort", ["0", "1"])
def test_long_lists_relabel(bigsort, monkeypatch):
    """gsm_load_graph's relabel with lists of degree >= 8192: by the segmented sort (default) or
    by one radix sort of (list, id) keys (GSM_BIGSORT=1): a hub of degree 12,000 plus a second
    one of 9,000 over random edges — K3 / P3 / C4 counts and K3 rows equal the oracle's."""
    monkeypatch.setenv("GSM_BIGSORT", bigsort)
    rng = np.random.default_rng(21)
    n = 12500
    src = [np.zeros(12000, np.int64), np.ones(9000, np.int64)]
    dst = [np.arange(1, 12001), np.arange(2, 9002)]
    e = rng.integers(2, n, size=(30000, 2))
    src.append(e[:, 0])
    dst.append(e[:, 1])
    g = gi.csr_from_edges(n, np.concatenate(src), np.concatenate(dst))
    G = load(g)
    try:
        for qn in ["K3", "P3", "C4"]:
            q = gi.query(qn)
            cnt, ref = oracle.match(g, q, count_only=qn != "K3")
            c, rows, _ = run(G, q, "enumerate" if qn == "K3" else "count")
            assert c == cnt, (qn, c, cnt)
            if qn == "K3":
                assert_rows_equal(rows, ref, "hub K3")
    finally:
        G.free()
