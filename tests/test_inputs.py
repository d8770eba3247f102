"""Seeded input generators (gsm_inputs): determinism and CSR invariants
(SPEC CsrGraph S:22-29; SURVEY §8(d) workload recipe)."""
import numpy as np

import gsm_inputs as gi


def check_csr(g):
    off, cols, n = g.offsets, g.cols, g.num_nodes
    assert off[0] == 0 and off[-1] == len(cols)
    assert np.all(np.diff(off) >= 0)
    src = np.repeat(np.arange(n), np.diff(off))
    assert np.all(src != cols)  # no self-loops
    same = src[1:] == src[:-1]
    assert np.all(cols[1:][same] > cols[:-1][same])  # strictly ascending lists
    fwd = np.sort(src.astype(np.int64) * n + cols)
    bwd = np.sort(cols.astype(np.int64) * n + src)
    assert np.array_equal(fwd, bwd)  # symmetric


def test_generators_deterministic_and_canonical(tmp_path, monkeypatch):
    monkeypatch.setenv("GSM_CACHE_DIR", "off")
    a = gi.rmat(12, 16, seed=7)
    b = gi.rmat(12, 16, seed=7)
    c = gi.rmat(12, 16, seed=8)
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.cols, b.cols)
    assert not np.array_equal(a.cols, c.cols)
    for g in (a, gi.grid(50, 40, seed=3), gi.erdos_renyi(1000, 4000, 1), gi.petersen()):
        check_csr(g)
    er = gi.erdos_renyi(1000, 4000, 1)
    assert er.num_edges == 4000
    lab = gi.uniform_labels(100000, 8, 1)
    assert lab.max() == 7 and lab.min() == 0
    assert np.array_equal(lab, gi.uniform_labels(100000, 8, 1))
    hist = np.bincount(lab, minlength=8) / 1e5
    assert np.all(np.abs(hist - 0.125) < 0.01)


def test_rmat_shape_statistics(monkeypatch):
    monkeypatch.setenv("GSM_CACHE_DIR", "off")
    g = gi.rmat(16, 16, seed=1)
    deg = g.degrees()
    # SURVEY §8(d) config [1] sizing: nnz ~1.82M, max deg ~1e4, ~29% isolated
    assert 1.7e6 < g.nnz < 1.95e6
    assert 5000 < deg.max() < 20000
    assert 0.25 < (deg == 0).mean() < 0.33


def test_grid_diagonal_counts(monkeypatch):
    monkeypatch.setenv("GSM_CACHE_DIR", "off")
    W, H = 60, 50
    g = gi.grid(W, H, seed=9)
    adj = set(zip(np.repeat(np.arange(W * H), np.diff(g.offsets)).tolist(), g.cols.tolist()))
    d1 = d2 = 0
    for y in range(H - 1):
        for x in range(W - 1):
            i = y * W + x
            m = (i, i + W + 1) in adj
            a = (i + 1, i + W) in adj
            d1 += m ^ a
            d2 += m and a
    assert (d1, d2) == (g.meta["d1"], g.meta["d2"])
    cells = (W - 1) * (H - 1)
    assert abs(d2 / cells - 0.05) < 0.02 and abs(d1 / cells - 0.30) < 0.04
    assert g.num_edges == (W - 1) * H + W * (H - 1) + d1 + 2 * d2


def test_zipf_labels_and_random_walk_queries(monkeypatch):
    """SPEC assign_powerlaw_labels and random_walk_query."""
    monkeypatch.setenv("GSM_CACHE_DIR", "off")
    lab = gi.zipf_labels(200000, 20, seed=4)
    assert lab.min() >= 0 and lab.max() <= 19
    assert np.array_equal(lab, gi.zipf_labels(200000, 20, seed=4))
    freq = np.bincount(lab, minlength=20) / len(lab)
    h = sum(1.0 / (l + 1) for l in range(20))
    for l in (0, 1, 4, 19):  # P(l) = (l+1)^-1 / H_20
        assert abs(freq[l] - 1.0 / ((l + 1) * h)) < 0.01
    assert np.all(gi.zipf_labels(1000, 1, 2) == 0)  # one label = unlabeled semantics
    g = gi.rmat(12, 16, seed=2).with_labels(gi.zipf_labels(4096, 20, 2))
    for seed in range(5):
        q = gi.random_walk_query(g, 12, 22, seed)
        assert q.num_nodes == 12 and len(q.edges) == 22 and len(set(q.edges)) == 22
        # connected
        seen, stack = {0}, [0]
        adj = {u: set() for u in range(12)}
        for a, b in q.edges:
            adj[a].add(b)
            adj[b].add(a)
        while stack:
            for w in adj[stack.pop()]:
                if w not in seen:
                    seen.add(w)
                    stack.append(w)
        assert len(seen) == 12
        assert q.labels is not None and len(q.labels) == 12
        assert q.edges == gi.random_walk_query(g, 12, 22, seed).edges  # deterministic
    # a triangle from K4
    q3 = gi.random_walk_query(gi.complete(4), 3, 3, 1)
    assert sorted(q3.edges) == [(0, 1), (0, 2), (1, 2)]
