"""oracle — the plain, slow, obviously-correct CPU reference.  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2003_01527_b200``) never imports it, and the two share no code: the
only common dependency is ``gsm_inputs`` (seeded input generators, no method
arithmetic).

Contents (each cites the passage it follows):
  * :func:`match` — all embeddings (injective, edge-preserving, label-respecting;
    SURVEY §8(b) semantics, §3.2) by plain DFS backtracking in C
    (``oracle.c``; §2.1, SURVEY §8(c) "Oracle algorithm"), rows
    sorted lexicographically (SURVEY §8(c) amb. 13).
  * :func:`automorphisms` — Aut(Q) by brute force over all k! permutations.
  * :func:`unique` — one representative per Aut(Q) orbit, canonical form
    f -> min_sigma f∘sigma (SURVEY §8(c) "Unique mode"; SPEC S:294 dedup, PAPER
    P:169 footnote "filters out duplicate results").
  * :func:`brute_force` — every injective map of a tiny instance, filtered by
    the definition (a second, independent check).
  * :func:`count_triangles`, :func:`count_k4` — independent exact clique
    counters (C, degree-ordered forward algorithm) for full-scale pins.
  * :mod:`oracle.closed_forms` — closed-form counts used to pin the oracle.

Pins: see tests/test_oracle_pins.py.  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_oracle.so")
_lib = None


class _Result(ctypes.Structure):
    _fields_ = [("count", ctypes.c_uint64), ("nrows", ctypes.c_int64), ("k", ctypes.c_int32),
                ("rows", ctypes.POINTER(ctypes.c_int32)), ("status", ctypes.c_int32)]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, src])
        os.replace(tmp, _SO)
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        p, i64 = ctypes.c_void_p, ctypes.c_int64
        lib.oracle_match.restype = ctypes.c_int
        lib.oracle_match.argtypes = [i64, p, p, p, ctypes.c_int, ctypes.c_int, p, p, p, i64, ctypes.c_int,
                                     ctypes.c_int, ctypes.POINTER(_Result)]
        lib.oracle_result_free.restype = None
        lib.oracle_result_free.argtypes = [ctypes.POINTER(_Result)]
        lib.oracle_count_triangles.restype = ctypes.c_uint64
        lib.oracle_count_triangles.argtypes = [i64, p, p, ctypes.c_int]
        lib.oracle_count_k4.restype = ctypes.c_uint64
        lib.oracle_count_k4.argtypes = [i64, p, p, ctypes.c_int]
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_L().oracle_num_threads())


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def sort_rows(rows: np.ndarray) -> np.ndarray:
    """Lexicographic sort of int32 rows as unsigned tuples (SURVEY §8(c) amb. 13)."""
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    if rows.shape[0] <= 1:
        return rows
    k = rows.shape[1]
    keys = rows.view(np.uint32)
    top = int(keys.max())
    bits = max(1, top.bit_length())
    if bits * k <= 64:  # one packed uint64 key per row (same order as the tuple order)
        packed = np.zeros(rows.shape[0], dtype=np.uint64)
        for j in range(k):
            packed = (packed << np.uint64(bits)) | keys[:, j].astype(np.uint64)
        order = np.argsort(packed, kind="stable")
    else:
        order = np.lexsort(keys.T[::-1])
    return rows[order]


def match(graph, query, roots: Optional[np.ndarray] = None, count_only: bool = False,
          threads: int = 0):
    """All embeddings of ``query`` in ``graph`` (the plain definition, computed by
    DFS).  Returns ``(count, rows)``; rows is ``None`` when ``count_only``, else an
    int32 array (count x k), column j = f(query vertex j), sorted lexicographically.
    ``roots`` restricts f(query vertex 0) to the given vertices (root sampling)."""
    k = query.num_nodes
    qe = np.ascontiguousarray(np.asarray(query.edges, dtype=np.int32).reshape(-1, 2))
    ql = None if query.labels is None else np.ascontiguousarray(query.labels, dtype=np.uint32)
    gl = None if graph.labels is None else np.ascontiguousarray(graph.labels, dtype=np.uint32)
    rt = None if roots is None else np.ascontiguousarray(roots, dtype=np.int32)
    res = _Result()
    rc = _L().oracle_match(graph.num_nodes, _p(graph.offsets), _p(graph.cols), _p(gl), k, len(qe), _p(qe), _p(ql),
                           _p(rt), 0 if rt is None else len(rt), threads, 0 if count_only else 1,
                           ctypes.byref(res))
    try:
        if rc != 0:
            raise ValueError(f"oracle_match failed (status {res.status})")
        count = int(res.count)
        if count_only:
            return count, None
        if res.nrows:
            rows = np.ctypeslib.as_array(res.rows, shape=(res.nrows * k,)).reshape(res.nrows, k).copy()
        else:
            rows = np.zeros((0, k), dtype=np.int32)
    finally:
        _L().oracle_result_free(ctypes.byref(res))
    return count, sort_rows(rows)


def count_triangles(graph, threads: int = 0) -> int:
    """Exact number of (unlabeled) triangles T; all K3 embeddings = 6T."""
    return int(_L().oracle_count_triangles(graph.num_nodes, _p(graph.offsets), _p(graph.cols), threads))


def count_k4(graph, threads: int = 0) -> int:
    """Exact number of (unlabeled) 4-cliques; all K4 embeddings = 24 * this."""
    return int(_L().oracle_count_k4(graph.num_nodes, _p(graph.offsets), _p(graph.cols), threads))


# ------------------------------------------------------------------ automorphisms
def automorphisms(query) -> np.ndarray:
    """Aut(Q): every permutation sigma of V_Q with (u,w) in E_Q <=> (sigma u, sigma w)
    in E_Q and label(sigma u) = label(u).  Brute force over all k! permutations
    (queries here have k <= 9).  Returns an int array (|Aut| x k), sigma[u]."""
    k = query.num_nodes
    E = {frozenset(e) for e in query.edges}
    lab = query.labels
    out = []
    for s in itertools.permutations(range(k)):
        if lab is not None and any(lab[s[u]] != lab[u] for u in range(k)):
            continue
        if all(frozenset((s[a], s[b])) in E for a, b in query.edges):
            out.append(s)
    return np.asarray(out, dtype=np.int64).reshape(-1, k)


def canonical(rows: np.ndarray, aut: np.ndarray) -> np.ndarray:
    """Canonical form of each embedding: the lexicographic minimum over sigma in
    Aut(Q) of f∘sigma, i.e. of the tuple (f(sigma 0), ..., f(sigma (k-1)))."""
    rows = np.asarray(rows, dtype=np.int32)
    if rows.shape[0] == 0:
        return rows.copy()
    best = rows[:, aut[0]].copy()
    for s in aut[1:]:
        cand = rows[:, s]
        # lexicographic (unsigned) comparison cand < best, row by row
        less = np.zeros(rows.shape[0], dtype=bool)
        decided = np.zeros(rows.shape[0], dtype=bool)
        for j in range(rows.shape[1]):
            cj = cand[:, j].view(np.uint32)
            bj = best[:, j].view(np.uint32)
            lt = (~decided) & (cj < bj)
            gt = (~decided) & (cj > bj)
            less |= lt
            decided |= lt | gt
        best[less] = cand[less]
    return best


def unique(rows: np.ndarray, aut: np.ndarray) -> np.ndarray:
    """One representative per Aut(Q) orbit (canonical forms), sorted."""
    c = canonical(rows, aut)
    if c.shape[0] == 0:
        return c
    c = sort_rows(c)
    keep = np.ones(c.shape[0], dtype=bool)
    keep[1:] = np.any(c[1:] != c[:-1], axis=1)
    return c[keep]


def expand_orbits(canon_rows: np.ndarray, aut: np.ndarray) -> np.ndarray:
    """{f∘sigma : f in rows, sigma in Aut(Q)}, deduplicated and sorted."""
    if canon_rows.shape[0] == 0:
        return canon_rows.copy()
    allr = np.concatenate([canon_rows[:, s] for s in aut], axis=0)
    allr = sort_rows(allr)
    keep = np.ones(allr.shape[0], dtype=bool)
    keep[1:] = np.any(allr[1:] != allr[:-1], axis=1)
    return allr[keep]


# ------------------------------------------------------------------ brute force
def brute_force(graph, query) -> np.ndarray:
    """Every injective map V_Q -> V_G (n!/(n-k)! of them, n <= 10) filtered by the
    definition.  Independent of :func:`match` (no DFS, no CSR binary search)."""
    n, k = graph.num_nodes, query.num_nodes
    adj = set()
    for u in range(n):
        for e in range(graph.offsets[u], graph.offsets[u + 1]):
            adj.add((u, int(graph.cols[e])))
    out = []
    for f in itertools.permutations(range(n), k):
        if query.labels is not None:
            if graph.labels is None:
                raise ValueError("query labels need data labels")
            if any(int(graph.labels[f[u]]) != query.labels[u] for u in range(k)):
                continue
        if all((f[a], f[b]) in adj for a, b in query.edges):
            out.append(f)
    return sort_rows(np.asarray(out, dtype=np.int32).reshape(-1, k))
