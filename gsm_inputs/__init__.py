"""gsm_inputs — seeded synthetic inputs shared by the oracle and the CUDA path.

This package is deliberately separate from both ``oracle/`` and
``paper_2003_01527_b200/``: it holds none of the matching method's arithmetic,
only the graph / label / query generators (SURVEY.md §2.7 "deterministic,
counter-based generators", §8(d) workloads).  Both sides of every parity test
receive their inputs from here.

Graphs are returned as :class:`Graph` (canonical undirected CSR: int64
offsets, int32 ascending neighbour lists, both directions stored, no loops, no
duplicates — SPEC CsrGraph S:22-29) with optional uint32 labels.
"""
from __future__ import annotations

import ctypes
import dataclasses
import hashlib
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_gen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile gen.c into an in-tree shared library (host code, OpenMP)."""
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-shared", "-fPIC",
                               "-o", tmp, src])
        os.replace(tmp, _SO)
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, u64, u32, p = ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p
        lib.gen_draw.restype = u64
        lib.gen_draw.argtypes = [u64, u64, u64]
        lib.gen_rmat_edges.restype = ctypes.c_int
        lib.gen_rmat_edges.argtypes = [ctypes.c_int, i64, u64, u32, u32, u32, p, p]
        lib.gen_grid_edges.restype = i64
        lib.gen_grid_edges.argtypes = [i64, i64, u64, u32, u32, p, p, p, p]
        lib.gen_er_edges.restype = i64
        lib.gen_er_edges.argtypes = [i64, i64, u64, p, p]
        lib.gen_uniform_labels.restype = None
        lib.gen_uniform_labels.argtypes = [i64, u32, u64, p]
        lib.gen_csr_build.restype = i64
        lib.gen_csr_build.argtypes = [i64, i64, p, p, p, p]
        lib.gen_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _threshold(num: int, den: int = 100) -> int:
    """floor(num/den * 2^32) as an exact integer (no float compares)."""
    return (num << 32) // den


@dataclasses.dataclass
class Graph:
    num_nodes: int
    offsets: np.ndarray  # int64[n+1]
    cols: np.ndarray  # int32[nnz]
    labels: Optional[np.ndarray] = None  # uint32[n] or None
    name: str = ""
    meta: dict = dataclasses.field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.offsets[-1])

    @property
    def num_edges(self) -> int:
        return self.nnz // 2

    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets)

    def with_labels(self, labels: Optional[np.ndarray], tag: str = "") -> "Graph":
        return dataclasses.replace(self, labels=None if labels is None else np.ascontiguousarray(labels, np.uint32),
                                   name=self.name + tag)


def csr_from_edges(n: int, src, dst, name: str = "") -> Graph:
    src = np.ascontiguousarray(src, dtype=np.int32)
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    m = len(src)
    offsets = np.empty(n + 1, dtype=np.int64)
    cols = np.empty(max(2 * m, 1), dtype=np.int32)
    nnz = _L().gen_csr_build(n, m, _ptr(src), _ptr(dst), _ptr(offsets), _ptr(cols))
    if nnz < 0:
        raise ValueError("edge id out of range")
    return Graph(n, offsets, cols[:nnz].copy(), None, name)


# ------------------------------------------------------------------ cache
def _cache_dir() -> Optional[str]:
    d = os.environ.get("GSM_CACHE_DIR", "/tmp/gsm_inputs_cache")
    if d in ("", "0", "off"):
        return None
    try:
        os.makedirs(d, exist_ok=True)
    except OSError:
        return None
    return d


def _cached(key: str, make):
    d = _cache_dir()
    h = hashlib.sha1(key.encode()).hexdigest()[:16]
    if d is not None:
        path = os.path.join(d, f"{h}.npz")
        if os.path.exists(path):
            try:
                z = np.load(path)
                meta = {k[5:]: int(z[k]) for k in z.files if k.startswith("meta_")}
                return Graph(int(z["n"]), z["offsets"], z["cols"], None, key, meta)
            except Exception:
                pass
    g = make()
    if d is not None:
        tmp = os.path.join(d, f"{h}.tmp{os.getpid()}.npz")
        try:
            np.savez(tmp, n=np.int64(g.num_nodes), offsets=g.offsets, cols=g.cols,
                     **{f"meta_{k}": np.int64(v) for k, v in g.meta.items()})
            os.replace(tmp, os.path.join(d, f"{h}.npz"))
        except OSError:
            pass
    g.name = key
    return g


# ------------------------------------------------------------------ generators
def rmat(scale: int, edge_factor: int = 16, seed: int = 1, abc_percent=(57, 19, 19)) -> Graph:
    """Graph500-style R-MAT (SURVEY §8(d) configs [1],[3],[4]): 2^scale vertices,
    edge_factor * 2^scale samples, quadrant probabilities a,b,c,d in percent,
    random vertex permutation, symmetrised / deduplicated / loop-free."""
    a, b, c = abc_percent
    key = f"rmat-s{scale}-ef{edge_factor}-seed{seed}-{a}.{b}.{c}"

    def make():
        n = 1 << scale
        m = edge_factor * n
        src = np.empty(m, dtype=np.int32)
        dst = np.empty(m, dtype=np.int32)
        rc = _L().gen_rmat_edges(scale, m, seed, _threshold(a), _threshold(a + b), _threshold(a + b + c),
                                 _ptr(src), _ptr(dst))
        if rc != 0:
            raise RuntimeError(f"gen_rmat_edges failed ({rc})")
        g = csr_from_edges(n, src, dst)
        del src, dst
        return g

    return _cached(key, make)


def grid(W: int, H: int, seed: int = 1, p_none_percent: int = 65, p_one_percent: int = 30) -> Graph:
    """Road-like W x H lattice with random diagonals (SURVEY §8(d) config [2]).
    meta['d1'] / meta['d2'] = number of cells with one / both diagonals."""
    key = f"grid-{W}x{H}-seed{seed}-{p_none_percent}.{p_one_percent}"

    def make():
        cap = 2 * W * H + 2 * max(W - 1, 0) * max(H - 1, 0)
        src = np.empty(cap, dtype=np.int32)
        dst = np.empty(cap, dtype=np.int32)
        d1 = ctypes.c_int64(0)
        d2 = ctypes.c_int64(0)
        m = _L().gen_grid_edges(W, H, seed, _threshold(p_none_percent), _threshold(p_none_percent + p_one_percent),
                                _ptr(src), _ptr(dst), ctypes.byref(d1), ctypes.byref(d2))
        if m < 0:
            raise ValueError("bad grid size")
        g = csr_from_edges(W * H, src[:m], dst[:m])
        g.meta = {"W": W, "H": H, "d1": d1.value, "d2": d2.value}
        return g

    return _cached(key, make)


def erdos_renyi(n: int, m: int, seed: int = 1) -> Graph:
    """G(n, m): m distinct undirected edges drawn uniformly (config [0])."""
    src = np.empty(m, dtype=np.int32)
    dst = np.empty(m, dtype=np.int32)
    if _L().gen_er_edges(n, m, seed, _ptr(src), _ptr(dst)) < 0:
        raise ValueError("bad G(n,m) parameters")
    g = csr_from_edges(n, src, dst, name=f"er-n{n}-m{m}-seed{seed}")
    return g


def uniform_labels(n: int, num_labels: int, seed: int = 1) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    _L().gen_uniform_labels(n, num_labels, seed, _ptr(out))
    return out


def zipf_labels(n: int, num_labels: int, seed: int = 1, alpha_num: int = 1, alpha_den: int = 1) -> np.ndarray:
    """Power-law node labels (SPEC assign_powerlaw_labels S:54-62; "seeds the data
    graph with power-law-distributed node ... labels"): label l in [0, L) with probability
    proportional to (l+1)^-alpha (alpha = 1 by default).  The CDF is quantised to
    32-bit integer thresholds so every caller draws identical labels."""
    if num_labels < 1:
        raise ValueError("num_labels must be >= 1")
    alpha = alpha_num / alpha_den
    w = np.array([(l + 1) ** (-alpha) for l in range(num_labels)], dtype=np.float64)
    cdf = np.cumsum(w) / w.sum()
    thr = np.minimum((cdf * 2 ** 32).astype(np.uint64), np.uint64(2 ** 32))
    thr[-1] = np.uint64(2 ** 32)
    u = uniform_labels(n, 1 << 31, seed).astype(np.uint64) << np.uint64(1)  # 32-bit uniform draw
    return np.searchsorted(thr, u, side="right").astype(np.uint32)


def random_walk_query(graph: "Graph", num_nodes: int, num_edges: int, seed: int = 1, max_tries: int = 1000) -> "Query":
    """Query from a random walk in the data graph (SPEC random_walk_query S:63-71; PAPER P:220,
    "uses random walks in the data graph to create a query graph of a specified size"): the
    first num_nodes distinct vertices of a walk, the walk's edges kept first (connected), then
    further edges of the induced subgraph in a seeded order until num_edges.  Labels are
    inherited from the data graph (None if unlabeled).  Raises if no start succeeds."""
    deg = np.diff(graph.offsets)
    for t in range(max_tries):
        start = int(draw(seed, 0x5257414c, t) % graph.num_nodes)
        if deg[start] == 0:
            continue
        order, pos = [start], {start: 0}
        edges = set()
        cur = start
        for step in range(64 * num_nodes):
            if len(order) == num_nodes:
                break
            d = int(deg[cur])
            if d == 0:
                break
            nxt = int(graph.cols[graph.offsets[cur] + draw(seed, 0x52574e58, t * 1_000_003 + step) % d])
            if nxt not in pos:
                pos[nxt] = len(order)
                order.append(nxt)
            a, b = pos[cur], pos[nxt]
            if a != b:
                edges.add((min(a, b), max(a, b)))
            cur = nxt
        if len(order) < num_nodes:
            continue
        # induced edges among the chosen vertices, in a seeded order
        chosen = np.array(order, dtype=np.int64)
        induced = []
        for i, v in enumerate(order):
            nb = graph.cols[graph.offsets[v]:graph.offsets[v + 1]]
            for w in nb[np.isin(nb, chosen)]:
                j = pos[int(w)]
                if i < j:
                    induced.append((i, j))
        extra = [e for e in induced if e not in edges]
        extra.sort(key=lambda e: draw(seed, 0x52574544, e[0] * 4096 + e[1]))
        if len(edges) > num_edges or len(edges) + len(extra) < num_edges:
            continue
        edges = sorted(edges | set(extra[:num_edges - len(edges)]))
        labels = None if graph.labels is None else [int(graph.labels[v]) for v in order]
        return Query(num_nodes, edges, labels, f"rw{num_nodes}-{num_edges}-s{seed}")
    raise RuntimeError("random walk did not reach the requested size; try another seed")


def draw(seed: int, stream: int, idx: int) -> int:
    return int(_L().gen_draw(seed, stream, idx))


# ------------------------------------------------------------------ textbook graphs
def from_edge_list(n: int, edges: Sequence[Sequence[int]], name: str = "") -> Graph:
    e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
    return csr_from_edges(n, e[:, 0], e[:, 1], name=name)


def complete(n: int) -> Graph:
    return from_edge_list(n, [(i, j) for i in range(n) for j in range(i + 1, n)], f"K{n}")


def complete_bipartite(a: int, b: int) -> Graph:
    return from_edge_list(a + b, [(i, a + j) for i in range(a) for j in range(b)], f"K{a},{b}")


def cycle(n: int) -> Graph:
    return from_edge_list(n, [(i, (i + 1) % n) for i in range(n)], f"C{n}")


def path(n: int) -> Graph:
    return from_edge_list(n, [(i, i + 1) for i in range(n - 1)], f"P{n}")


def petersen() -> Graph:
    outer = [(i, (i + 1) % 5) for i in range(5)]
    spokes = [(i, i + 5) for i in range(5)]
    inner = [(5 + i, 5 + (i + 2) % 5) for i in range(5)]
    return from_edge_list(10, outer + spokes + inner, "petersen")


def chain_with_tails(num_chains: int, length: int, seed: int = 1, tail_percent: int = 50) -> Graph:
    """Road-like sparse graph ("chain-with-tails", mimicking road_central's
    low average degree): num_chains disjoint paths of `length` vertices, each
    chain vertex carrying a pendant degree-1 tail with probability tail_percent %, and
    consecutive chains joined end to end with probability 1/2 (longer roads)."""
    src, dst = [], []
    n = 0
    prev_end = -1
    thr = _threshold(tail_percent)
    for c in range(num_chains):
        first = n
        for i in range(length):
            v = n
            n += 1
            if i:
                src.append(v - 1)
                dst.append(v)
        if prev_end >= 0 and (draw(seed, 0x4a4f494e, c) & 1):
            src.append(prev_end)
            dst.append(first)
        prev_end = n - 1
        for i in range(length):
            if (draw(seed, 0x5441494c, first + i) & 0xffffffff) < thr:
                src.append(first + i)
                dst.append(n)
                n += 1
    return csr_from_edges(n, np.asarray(src, np.int32), np.asarray(dst, np.int32), f"chain-tails-{num_chains}x{length}")


def plain_grid(W: int, H: int) -> Graph:
    e = []
    for y in range(H):
        for x in range(W):
            i = y * W + x
            if x + 1 < W:
                e.append((i, i + 1))
            if y + 1 < H:
                e.append((i, i + W))
    return from_edge_list(W * H, e, f"grid{W}x{H}")


def random_gnp(n: int, p_num: int, p_den: int, seed: int) -> Graph:
    """Small G(n, p) for property tests (integer threshold p_num/p_den)."""
    t = (p_num << 32) // p_den
    e = [(i, j) for i in range(n) for j in range(i + 1, n)
         if (draw(seed, 0x474e50, i * n + j) >> 32) < t]
    return from_edge_list(n, e, f"gnp{n}-{p_num}/{p_den}-s{seed}")


# ------------------------------------------------------------------ queries
@dataclasses.dataclass
class Query:
    """Small query graph Q: k vertices 0..k-1, undirected edge list, optional labels."""
    num_nodes: int
    edges: list
    labels: Optional[list] = None
    name: str = ""

    def with_labels(self, labels):
        return Query(self.num_nodes, list(self.edges), None if labels is None else list(labels),
                     self.name + ("" if labels is None else "(" + ",".join(map(str, labels)) + ")"))


QUERIES = {
    "K1": Query(1, [], None, "K1"),
    "K2": Query(2, [(0, 1)], None, "K2"),
    "K3": Query(3, [(0, 1), (1, 2), (0, 2)], None, "K3"),
    "P3": Query(3, [(0, 1), (1, 2)], None, "P3"),
    "P4": Query(4, [(0, 1), (1, 2), (2, 3)], None, "P4"),
    "S3": Query(4, [(0, 1), (0, 2), (0, 3)], None, "S3"),  # star K_{1,3}, centre 0
    "C4": Query(4, [(0, 1), (1, 2), (2, 3), (3, 0)], None, "C4"),
    "K4": Query(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)], None, "K4"),
    "C5": Query(5, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0)], None, "C5"),
    "diamond": Query(4, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)], None, "diamond"),
    "tailed_triangle": Query(4, [(0, 1), (1, 2), (0, 2), (2, 3)], None, "tailed_triangle"),
    # house: square 0-1-2-3 plus roof vertex 4 on edge 0-1 (SURVEY §8(d) config [3])
    "house": Query(5, [(0, 1), (1, 2), (2, 3), (3, 0), (0, 4), (1, 4)], None, "house"),
}


def query(name: str, labels=None) -> Query:
    q = QUERIES[name]
    return q if labels is None else q.with_labels(labels)


def random_connected_query(k: int, extra_edges: int, seed: int, num_labels: int = 0) -> Query:
    """Random connected query: a random spanning tree plus extra random edges."""
    edges = set()
    for v in range(1, k):
        u = draw(seed, 0x51545245, v) % v
        edges.add((u, v))
    t = 0
    possible = k * (k - 1) // 2
    while len(edges) < min(possible, k - 1 + extra_edges):
        r = draw(seed, 0x51455854, t)
        t += 1
        a, b = (r >> 32) % k, (r & 0xffffffff) % k
        if a == b:
            continue
        edges.add((min(a, b), max(a, b)))
    labels = None
    if num_labels:
        labels = [int(draw(seed, 0x514c4142, v) % num_labels) for v in range(k)]
    return Query(k, sorted(edges), labels, f"rq{k}-{extra_edges}-s{seed}")
