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
