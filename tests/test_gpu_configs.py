"""GPU parity on the five BASELINE.json configs at full size.

Full sorted row lists vs the oracle where the oracle finishes (configs 0-2);
for configs 3-4 (R-MAT-22 house, R-MAT-24 K3/K4): root-sampled oracle parity
(exercises the direct search), exact counts from independent counters, and
the symmetry identities that pin the production (ID-constrained) path:
count_all = |Aut| x count_unique = count of the direct search."""
import numpy as np
import pytest

import gsm_inputs as gi
import oracle
from gsm_inputs import workloads
from oracle import closed_forms as cf
from paper_2003_01527_b200 import gsm

from gpu_helpers import assert_rows_equal, is_sorted_unique, load, run

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_config0_er1000_triangle(seed):
    g = gi.erdos_renyi(1000, 4000, seed)
    q = gi.query("K3")
    G = load(g)
    try:
        cnt, ref = oracle.match(g, q)
        c, rows, _ = run(G, q, "enumerate")
        assert c == cnt == cf.triangle_trace(cf.dense_adj(g))
        assert_rows_equal(rows, ref, "er1000 all")
        cu, rowsu, _ = run(G, q, "enumerate", flags=gsm.GSM_FLAG_UNIQUE)
        aut = oracle.automorphisms(q)
        assert cu * 6 == cnt
        assert_rows_equal(oracle.unique(rowsu, aut), oracle.unique(ref, aut), "er1000 unique")
    finally:
        G.free()


@pytest.fixture(scope="module")
def rmat16():
    w = workloads.get("rmat16")
    g = w.graph()
    G = load(g)
    yield w, g, G
    G.free()


@pytest.mark.parametrize("qi", [0, 1, 2, 3])
def test_config1_rmat16_labeled_path_and_star(rmat16, qi):
    w, g, G = rmat16
    q = w.queries[qi]
    if q.name.startswith("P4"):
        closed = cf.path4_labeled_vectorised(g, *q.labels, num_labels=8)
    else:
        closed = cf.star_vectorised(g, q.labels[0], q.labels[1:], 8)
    c_count, _, r = run(G, q, "count")
    assert c_count == closed, (q.name, c_count, closed)
    cnt, ref = oracle.match(g, q)
    assert cnt == closed
    c, rows, _ = run(G, q, "enumerate")
    assert c == cnt
    assert_rows_equal(rows, ref, q.name)
    del rows, ref
    cu, _, ru = run(G, q, "count", flags=gsm.GSM_FLAG_UNIQUE)
    assert cu * ru.automorphisms == cnt


@pytest.fixture(scope="module")
def grid1m():
    w = workloads.get("grid1m")
    g = w.graph()
    G = load(g)
    yield w, g, G
    G.free()


def test_config2_grid_k4(grid1m):
    w, g, G = grid1m
    q = gi.query("K4")
    c, rows, _ = run(G, q, "enumerate")
    assert c == cf.grid_diag_k4(g.meta["d2"])
    cnt, ref = oracle.match(g, q)
    assert c == cnt
    assert_rows_equal(rows, ref, "grid K4")
    assert run(G, gi.query("K3"))[0] == cf.grid_diag_k3(g.meta["d1"], g.meta["d2"])


def test_config2_grid_c4(grid1m):
    w, g, G = grid1m
    q = gi.query("C4")
    c, rows, _ = run(G, q, "enumerate")
    cnt, ref = oracle.match(g, q)
    assert c == cnt == cf.cycle4(g)
    assert_rows_equal(rows, ref, "grid C4")
    assert is_sorted_unique(rows)


@pytest.fixture(scope="module")
def rmat22():
    w = workloads.get("rmat22")
    g = w.graph()
    G = load(g, validate=True)
    yield w, g, G
    G.free()


def _root_sample(g, label, n_uniform, seed, n_high=16):
    """Uniform sample of label-matching vertices + n_high moderately high-degree ones
    (around the 99.9th degree percentile: hubs make the plain DFS infeasible)."""
    rng = np.random.default_rng(seed)
    cand = np.nonzero(g.labels == label)[0] if label is not None else np.arange(g.num_nodes)
    uni = rng.choice(cand, size=min(n_uniform, len(cand)), replace=False)
    deg = np.diff(g.offsets)[cand]
    order = cand[np.argsort(deg, kind="stable")]
    hi = order[int(len(order) * 0.999): int(len(order) * 0.999) + n_high]
    return np.unique(np.concatenate([uni, hi])).astype(np.int32)


def _hubs(g, label, n):
    """The n highest-degree vertices (carrying `label` when given)."""
    cand = np.nonzero(g.labels == label)[0] if label is not None else np.arange(g.num_nodes)
    deg = np.diff(g.offsets)[cand]
    return cand[np.argsort(-deg, kind="stable")[:n]].astype(np.int32)


@pytest.mark.parametrize("qi", [0, 1])
def test_config3_rmat22_house_exact_full_scale(rmat22, qi):
    """configs[3] at full scale against the oracle's independent house counter (counts
    roof x 4-path choices per edge; oracle.house_counts_by_root): the production COUNT
    path (symmetric search + pair tail, k_pair) must give the exact total."""
    w, g, G = rmat22
    q = w.queries[qi]
    total, _ = oracle.house_counts_by_root(g, q.labels)
    c_all, _, r = run(G, q, "count")
    assert r.prof["tail"]["launches"] > 0, "pair tail (k_pair) did not run"
    assert c_all == total, (q.name, c_all, total)
    c_uni, _, ru = run(G, q, "count", flags=gsm.GSM_FLAG_UNIQUE)
    c_direct, _, _ = run(G, q, "count", flags=gsm.GSM_FLAG_NO_SYMMETRY)
    aut = oracle.automorphisms(q)
    assert r.automorphisms == len(aut)
    assert c_all == len(aut) * c_uni == c_direct


@pytest.mark.parametrize("qi", [0, 1])
def test_config3_rmat22_house_roots_with_pair_tail(rmat22, qi):
    """Root-sampled parity of the pair-tail kernel (k_pair) at full scale: 4,096 uniform
    label-matching roots + the 64 highest-degree label-matching roots (SURVEY §8(c) pin
    (i)), per-root counts from the oracle's house counter.  root_subset pins π[0] = 0 and
    keeps the pair tail on (the pair is chosen among the other vertices)."""
    w, g, G = rmat22
    q = w.queries[qi]
    rng = np.random.default_rng(100 + qi)
    cand = np.nonzero(g.labels == q.labels[0])[0]
    uni = np.sort(rng.choice(cand, size=4096, replace=False)).astype(np.int32)
    hubs = _hubs(g, q.labels[0], 64)
    for roots, what in ((uni, "4096 uniform roots"), (hubs, "64 hubs")):
        total, per = oracle.house_counts_by_root(g, q.labels, roots)
        c, _, r = run(G, q, "count", root_subset=roots)
        assert r.prof["tail"]["launches"] > 0, "pair tail (k_pair) did not run under root_subset"
        assert r.order[0] == 0
        assert c == total, (q.name, what, c, total)
    for h in hubs[:8]:  # the largest hubs one by one
        total, _ = oracle.house_counts_by_root(g, q.labels, np.array([h], dtype=np.int32))
        assert run(G, q, "count", root_subset=[h])[0] == total, (q.name, int(h))


@pytest.mark.parametrize("qi", [0, 1])
def test_config3_rmat22_house_enumerate_sample(rmat22, qi):
    """Sorted row lists of a root sample against the plain DFS oracle (ENUMERATE path)."""
    w, g, G = rmat22
    q = w.queries[qi]
    roots = _root_sample(g, q.labels[0], 1024, 7 + qi, n_high=4)  # bounded oracle time (~minutes)
    cnt, ref = oracle.match(g, q, roots=roots)
    c, rows, _ = run(G, q, "enumerate", root_subset=roots)
    assert c == cnt and cnt > 0
    assert_rows_equal(rows, ref, q.name + " root sample")


@pytest.fixture(scope="module")
def rmat24():
    w = workloads.get("rmat24")
    g = w.graph()
    G = load(g)
    yield w, g, G
    G.free()


def _golden24():
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "rmat24_cliques.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/rmat24_cliques.json absent (tools/make_golden_cliques.py --scale 24)")
    return json.load(open(path))


@pytest.mark.parametrize("k", [3, 4])
def test_config4_rmat24_cliques_exact(rmat24, k):
    """configs[4] at full scale: the clique kernels' counts equal the oracle's independent
    degree-ordered counter (tests/golden/rmat24_cliques.json, written by
    tools/make_golden_cliques.py, which calls only oracle/) — total, every shard of P = 64
    (root rank % 64), and the 64 largest hubs + 256 strided vertices one root at a time
    (num_shards = n isolates one root)."""
    w, g, G = rmat24
    gold = _golden24()
    if f"K{k}" not in gold:
        pytest.skip(f"golden K{k} not computed yet")
    gk = gold[f"K{k}"]
    assert gold["num_nodes"] == g.num_nodes and gold["nnz"] == g.nnz
    q = gi.query(f"K{k}")
    fact = 6 if k == 3 else 24
    c, _, r = run(G, q, "count", mem_budget_bytes=w.mem_budget_bytes)
    assert r.prof["clique"]["launches"] > 0
    assert c == fact * gk["total"], (c, fact * gk["total"])
    P = 64
    for s in range(P):
        cs, _, _ = run(G, q, "count", shard_index=s, num_shards=P, mem_budget_bytes=w.mem_budget_bytes)
        assert cs == fact * gk["shards"][str(P)][s], ("shard", s)
    rank = oracle.rank_order(g)
    n = g.num_nodes
    for v, want in gk["roots"].items():
        cv, _, rv = run(G, q, "count", flags=gsm.GSM_FLAG_UNIQUE, shard_index=int(rank[int(v)]), num_shards=n)
        assert cv == want, ("root", v, cv, want)


def test_config4_rmat24_cliques_degeneracy_order(rmat24, monkeypatch):
    """GSM_ORDER=1 (approximate degeneracy rank, another valid ≺): K3 and K4 totals at full
    scale still equal the oracle's independent counter (golden file)."""
    w, g, _ = rmat24
    gold = _golden24()
    monkeypatch.setenv("GSM_ORDER", "1")
    G = load(g, validate=False)
    monkeypatch.delenv("GSM_ORDER")
    try:
        for k, fact in ((3, 6), (4, 24)):
            if f"K{k}" not in gold:
                continue
            c, _, r = run(G, gi.query(f"K{k}"), "count", mem_budget_bytes=w.mem_budget_bytes)
            assert r.prof["clique"]["launches"] > 0
            assert c == fact * gold[f"K{k}"]["total"], (k, c)
    finally:
        G.free()


def test_config4_rmat24_k4_chunked_bfs_and_samples(rmat24, monkeypatch):
    """The north_star's breadth-first path (GSM_CLIQUE=0: chunked frontier under the fixed
    16 GiB budget) on the same graph, and root-sampled sorted-row parity vs the DFS oracle."""
    w, g, G = rmat24
    q = gi.query("K4")
    c_all, _, r = run(G, q, "count", mem_budget_bytes=w.mem_budget_bytes)  # clique bitmap path
    assert c_all == 24 * r.count_unique and c_all > 0
    monkeypatch.setenv("GSM_CLIQUE", "0")
    c_bfs, _, r2 = run(G, q, "count", mem_budget_bytes=w.mem_budget_bytes)
    monkeypatch.delenv("GSM_CLIQUE")
    assert r2.num_chunks > 1  # the fixed budget forces a chunked frontier
    assert c_bfs == c_all
    roots = _root_sample(g, None, 128, 11, n_high=0)  # the plain DFS needs ~0.2 s per R-MAT-24 root
    cnt, ref = oracle.match(g, q, roots=roots)
    c, rows, _ = run(G, q, "enumerate", root_subset=roots)
    assert c == cnt
    assert_rows_equal(rows, ref, "rmat24 K4 root sample")
    cnt3, ref3 = oracle.match(g, gi.query("K3"), roots=roots)
    c3, rows3, _ = run(G, gi.query("K3"), "enumerate", root_subset=roots)
    assert c3 == cnt3
    assert_rows_equal(rows3, ref3, "rmat24 K3 root sample")


def test_config4_k4_exact_at_scale20():
    """K4 exact count against the independent CPU counter where it finishes (scale 20)."""
    g = gi.rmat(20, 16, 1)
    G = load(g)
    try:
        c, _, _ = run(G, gi.query("K4"), mem_budget_bytes=1 << 30)
        assert c == 24 * oracle.count_k4(g)
    finally:
        G.free()
