"""Closed-form embedding counts — TEST INFRASTRUCTURE ONLY (pins for the oracle
and full-scale pins for the CUDA path).  Formulas from SURVEY.md §8(c) "What
pins each part"; each one is an independent counting argument, not a search.

All counts are of ALL embeddings (injective, edge-preserving, label-respecting
maps; non-induced), SURVEY §8(b).
"""
from __future__ import annotations

from math import prod

import numpy as np


def falling(x: int, m: int) -> int:
    """x (x-1) ... (x-m+1); 0 when x < m."""
    r = 1
    for i in range(m):
        r *= max(x - i, 0)
    return r


def complete_graph(n: int, k: int) -> int:
    """Any connected k-vertex Q in K_n: n!/(n-k)! (every injective map works)."""
    return falling(n, k)


def complete_graph_labeled(label_counts: dict, query_labels) -> int:
    """Labeled K_n with c_l vertices of label l; Q with m_l vertices of label l:
    prod_l falling(c_l, m_l)."""
    m = {}
    for l in query_labels:
        m[l] = m.get(l, 0) + 1
    return prod(falling(label_counts.get(l, 0), ml) for l, ml in m.items())


def _neighbour_label_counts(graph, v: int) -> dict:
    out = {}
    for e in range(graph.offsets[v], graph.offsets[v + 1]):
        w = int(graph.cols[e])
        l = 0 if graph.labels is None else int(graph.labels[w])
        out[l] = out.get(l, 0) + 1
    return out


def star(graph, centre_label, leaf_labels) -> int:
    """Star K_{1,s}: sum over v with L(v) = L_centre of prod_l falling(n_l(v), m_l),
    n_l(v) = neighbours of v with label l, m_l = leaves with label l.
    Labels None => unlabeled (all labels 0)."""
    m = {}
    for l in leaf_labels:
        m[l] = m.get(l, 0) + 1
    deg = np.diff(graph.offsets)
    total = 0
    for v in range(graph.num_nodes):
        if deg[v] == 0:
            continue
        lv = 0 if graph.labels is None else int(graph.labels[v])
        if lv != centre_label:
            continue
        nl = _neighbour_label_counts(graph, v)
        total += prod(falling(nl.get(l, 0), ml) for l, ml in m.items())
    return total


def star_vectorised(graph, centre_label, leaf_labels, num_labels: int) -> int:
    """Same formula as :func:`star`, with numpy per-vertex label histograms
    (for full-scale graphs).  Exact integer arithmetic (Python ints in the sum)."""
    n = graph.num_nodes
    lab = np.zeros(n, dtype=np.int64) if graph.labels is None else graph.labels.astype(np.int64)
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(graph.offsets))
    hist = np.zeros((n, num_labels), dtype=np.int64)
    np.add.at(hist, (src, lab[graph.cols.astype(np.int64)]), 1)
    m = {}
    for l in leaf_labels:
        m[l] = m.get(l, 0) + 1
    sel = np.nonzero(lab == centre_label)[0]
    terms = np.ones(len(sel), dtype=object)
    for l, ml in m.items():
        x = hist[sel, l]
        f = np.ones(len(sel), dtype=object)
        for i in range(ml):
            f = f * np.maximum(x - i, 0).astype(object)
        terms = terms * f
    return int(terms.sum()) if len(sel) else 0


def path4_labeled(graph, la, lb, lc, ld) -> int:
    """P4 a-b-c-d: sum over directed (b,c) in E with L(b)=lb, L(c)=lc of
    (n_la(b) - [L(c)=la]) * (n_ld(c) - [L(b)=ld]) - [la=ld] * #{x in N(b) & N(c) : L(x)=la}."""
    lab = (lambda v: 0) if graph.labels is None else (lambda v: int(graph.labels[v]))
    total = 0
    for b in range(graph.num_nodes):
        if lab(b) != lb:
            continue
        nb = _neighbour_label_counts(graph, b)
        Nb = set(int(x) for x in graph.cols[graph.offsets[b]:graph.offsets[b + 1]])
        for e in range(graph.offsets[b], graph.offsets[b + 1]):
            c = int(graph.cols[e])
            if lab(c) != lc:
                continue
            nc = _neighbour_label_counts(graph, c)
            a_choices = nb.get(la, 0) - (1 if lab(c) == la else 0)
            d_choices = nc.get(ld, 0) - (1 if lab(b) == ld else 0)
            t = a_choices * d_choices
            if la == ld:
                common = sum(1 for x in graph.cols[graph.offsets[c]:graph.offsets[c + 1]]
                             if int(x) in Nb and lab(int(x)) == la)
                t -= common
            total += t
    return total


def path4_labeled_vectorised(graph, la, lb, lc, ld, num_labels: int) -> int:
    """:func:`path4_labeled` with numpy, for full-scale graphs.  The common
    neighbour term (only when la == ld) is counted by sorting 2-path keys."""
    n = graph.num_nodes
    lab = np.zeros(n, dtype=np.int64) if graph.labels is None else graph.labels.astype(np.int64)
    deg = np.diff(graph.offsets)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    dst = graph.cols.astype(np.int64)
    hist = np.zeros((n, num_labels), dtype=np.int64)
    np.add.at(hist, (src, lab[dst]), 1)
    sel = (lab[src] == lb) & (lab[dst] == lc)
    b, c = src[sel], dst[sel]
    a_ch = hist[b, la] - (lab[c] == la)
    d_ch = hist[c, ld] - (lab[b] == ld)
    total = int(np.sum(a_ch.astype(object) * d_ch.astype(object))) if len(b) else 0
    if la == ld and len(b):
        # sum over selected directed (b,c) of #{x in N(b) & N(c): L(x)=la}
        #   = number of 2-paths b - x - c with L(x)=la and (b,c) selected
        xs = np.nonzero(lab == la)[0]
        cnt = 0
        keys = np.sort(b * n + c)
        for x in xs:
            nb = graph.cols[graph.offsets[x]:graph.offsets[x + 1]].astype(np.int64)
            if len(nb) < 2:
                continue
            bb = nb[lab[nb] == lb]
            cc = nb[lab[nb] == lc]
            if len(bb) == 0 or len(cc) == 0:
                continue
            k2 = (bb[:, None] * n + cc[None, :]).ravel()
            k2 = k2[(k2 // n) != (k2 % n)]
            pos = np.minimum(np.searchsorted(keys, k2), len(keys) - 1)
            cnt += int(np.sum(keys[pos] == k2))
        total -= cnt
    return total


def path4_unlabeled(graph, triangles: int) -> int:
    """Unlabeled P4: sum over directed (b,c) of (d_b - 1)(d_c - 1) - 6T."""
    deg = np.diff(graph.offsets).astype(np.int64)
    src = np.repeat(np.arange(graph.num_nodes), np.diff(graph.offsets))
    return int(np.sum((deg[src] - 1) * (deg[graph.cols] - 1))) - 6 * triangles


def cycle4(graph) -> int:
    """C4 all = sum over ordered pairs a != c of cn(a,c) (cn(a,c) - 1), cn = number
    of common neighbours (f(0)=a, f(2)=c, f(1) != f(3) both common)."""
    n = graph.num_nodes
    # all 2-paths a - b - c with a != c
    a_list, c_list = [], []
    for b in range(n):
        nb = graph.cols[graph.offsets[b]:graph.offsets[b + 1]].astype(np.int64)
        if len(nb) < 2:
            continue
        aa = np.repeat(nb, len(nb))
        cc = np.tile(nb, len(nb))
        keep = aa != cc
        a_list.append(aa[keep])
        c_list.append(cc[keep])
    if not a_list:
        return 0
    keys = np.concatenate(a_list) * n + np.concatenate(c_list)
    _, cn = np.unique(keys, return_counts=True)
    return int(np.sum(cn.astype(np.int64) * (cn.astype(np.int64) - 1)))


def cycle4_dense(adj: np.ndarray) -> int:
    """tr(A^4) - 2 sum_v d(d-1) - 2m  (closed walks of length 4 minus degenerate ones)."""
    A = adj.astype(object)
    A2 = A.dot(A)
    tr4 = int(sum(A2[i, j] * A2[j, i] for i in range(len(A)) for j in range(len(A))))
    d = adj.sum(axis=1).astype(object)
    m = int(adj.sum()) // 2
    return tr4 - 2 * int(sum(x * (x - 1) for x in d)) - 2 * m


def triangle_trace(adj: np.ndarray) -> int:
    """All K3 embeddings = 6T = tr(A^3)."""
    A = adj.astype(np.int64)
    return int(np.trace(A @ A @ A))


def grid_plain_c4(W: int, H: int) -> int:
    """Plain W x H grid: C4 all = 8 (W-1)(H-1) (one 4-cycle per cell, |Aut(C4)|=8)."""
    return 8 * (W - 1) * (H - 1)


def grid_diag_k4(d2: int) -> int:
    """Grid + diagonals: a 4-clique needs both diagonals of one cell: K4 all = 24 D2."""
    return 24 * d2


def grid_diag_k3(d1: int, d2: int) -> int:
    """Grid + diagonals: 2 triangles per one-diagonal cell, 4 per two-diagonal
    cell; K3 all = 6 (2 D1 + 4 D2)."""
    return 6 * (2 * d1 + 4 * d2)


def kab_c4(a: int, b: int) -> int:
    """K_{a,b}: C4 all = 2 a(a-1) b(b-1)."""
    return 2 * a * (a - 1) * b * (b - 1)


def dense_adj(graph) -> np.ndarray:
    n = graph.num_nodes
    A = np.zeros((n, n), dtype=np.int64)
    src = np.repeat(np.arange(n), np.diff(graph.offsets))
    A[src, graph.cols] = 1
    return A
