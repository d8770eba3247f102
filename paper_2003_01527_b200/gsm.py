"""Thin ctypes binding for libgsm.so (include/gsm.h).  Argument marshalling only:
every step of the hot path runs inside the library's CUDA kernels.  There is no
CPU fallback — if libgsm.so (or a CUDA device) is missing, calls raise.

The functions keep the C names: :func:`gsm_load_graph`, :func:`gsm_match`,
:func:`gsm_free`, :func:`gsm_result_free`, :func:`gsm_result_copy_rows`,
:func:`gsm_graph_info`, :func:`gsm_plan_query`, :func:`gsm_last_error`.
Arrays may be numpy (host) or torch tensors (host or CUDA)."""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# GSM_LIB=checked selects the device-index-checked test build (libgsm_checked.so)
SO_PATH = os.path.join(HERE, "libgsm_checked.so" if os.environ.get("GSM_LIB") == "checked" else "libgsm.so")

MAX_K = 32

GSM_OK = 0
STATUS_NAMES = {0: "GSM_OK", 1: "GSM_ERR_INVALID_ARGUMENT", 2: "GSM_ERR_INVALID_GRAPH", 3: "GSM_ERR_INVALID_QUERY",
                4: "GSM_ERR_OUT_OF_MEMORY", 5: "GSM_ERR_CUDA", 6: "GSM_ERR_NO_DEVICE"}
GSM_MODE_COUNT = 0
GSM_MODE_ENUMERATE = 1
GSM_FLAG_UNIQUE = 1
GSM_FLAG_NO_SYMMETRY = 2
GSM_FLAG_PROFILE = 4
GSM_FLAG_PLAN_COUNT = 8
GSM_FLAG_COMPRESSED_PARTIALS = 16
GSM_FLAG_SHARD_LEVEL1 = 32
KERNEL_NAMES = ["filter", "roots", "plan", "scan", "expand", "finalize", "tail", "clique"]


class GsmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class gsm_load_opts(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("device", ctypes.c_int32), ("validate", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("stream", ctypes.c_void_p)]


class gsm_query(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_int32), ("num_edges", ctypes.c_int32),
                ("edges", ctypes.POINTER(ctypes.c_int32)), ("labels", ctypes.POINTER(ctypes.c_uint32))]


class gsm_match_opts(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("mode", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("shard_index", ctypes.c_int32), ("num_shards", ctypes.c_int32), ("refine_rounds", ctypes.c_int32),
                ("lookahead", ctypes.c_int32), ("root_subset", ctypes.POINTER(ctypes.c_int32)), ("root_subset_len", ctypes.c_int64),
                ("mem_budget_bytes", ctypes.c_uint64), ("stream", ctypes.c_void_p)]


class gsm_kernel_prof(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_uint64), ("ms", ctypes.c_double), ("alg_bytes", ctypes.c_double)]


class gsm_result(ctypes.Structure):
    _fields_ = [("count", ctypes.c_uint64), ("count_unique", ctypes.c_uint64), ("automorphisms", ctypes.c_uint64),
                ("width", ctypes.c_int32), ("num_levels", ctypes.c_int32), ("num_rows", ctypes.c_uint64),
                ("rows", ctypes.c_void_p),
                ("ms_total", ctypes.c_float), ("ms_plan", ctypes.c_float), ("ms_filter", ctypes.c_float),
                ("ms_expand", ctypes.c_float), ("ms_finalize", ctypes.c_float),
                ("order", ctypes.c_int32 * MAX_K), ("candidates", ctypes.c_uint64 * MAX_K),
                ("level_rows", ctypes.c_uint64 * MAX_K), ("level_work", ctypes.c_uint64 * MAX_K),
                ("num_chunks", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64),
                ("prof", gsm_kernel_prof * 8), ("device", ctypes.c_int32), ("symmetric", ctypes.c_int32),
                ("level_frontier_bytes", ctypes.c_uint64 * MAX_K), ("compressed", ctypes.c_int32),
                ("level1_sharded", ctypes.c_int32)]


class gsm_plan_info(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("order", ctypes.c_int32 * MAX_K), ("parent", ctypes.c_int32 * MAX_K),
                ("backward", ctypes.c_uint32 * MAX_K), ("num_conditions", ctypes.c_int32),
                ("cond_lo", ctypes.c_int32 * (MAX_K * MAX_K // 2)), ("cond_hi", ctypes.c_int32 * (MAX_K * MAX_K // 2)),
                ("automorphisms", ctypes.c_uint64)]


_lib = None

EXPORTS = ["gsm_load_graph", "gsm_free", "gsm_graph_info", "gsm_match", "gsm_result_free", "gsm_result_copy_rows",
           "gsm_plan_query", "gsm_sort_rows", "gsm_merge_rows", "gsm_filter_candidates", "gsm_last_error",
           "gsm_version"]


def lib():
    """Load libgsm.so (fails loudly if it was not built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"libgsm.so not built at {SO_PATH}; run __graft_entry__.build()")
        L = ctypes.CDLL(SO_PATH)
        P, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.gsm_load_graph.argtypes = [i64, P, P, P, i32, ctypes.POINTER(gsm_load_opts), ctypes.POINTER(ctypes.c_void_p)]
        L.gsm_free.argtypes = [P]
        L.gsm_graph_info.argtypes = [P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                     ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
        L.gsm_match.argtypes = [P, ctypes.POINTER(gsm_query), ctypes.POINTER(gsm_match_opts), ctypes.POINTER(gsm_result)]
        L.gsm_result_free.argtypes = [ctypes.POINTER(gsm_result)]
        L.gsm_result_copy_rows.argtypes = [ctypes.POINTER(gsm_result), P, i32]
        L.gsm_plan_query.argtypes = [ctypes.POINTER(gsm_query), P, ctypes.c_uint32, ctypes.POINTER(gsm_plan_info)]
        L.gsm_sort_rows.argtypes = [P, ctypes.c_uint64, i32, i64, i32, P]
        L.gsm_merge_rows.argtypes = [P, ctypes.c_uint64, P, ctypes.c_uint64, i32, P, i32, P]
        L.gsm_filter_candidates.argtypes = [P, ctypes.POINTER(gsm_query), i32, P, i32]
        L.gsm_last_error.restype = ctypes.c_char_p
        L.gsm_version.restype = ctypes.c_char_p
        for name in EXPORTS:
            if name not in ("gsm_last_error", "gsm_version"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def gsm_last_error() -> str:
    return lib().gsm_last_error().decode()


def _check(status: int):
    if status != GSM_OK:
        raise GsmError(status, gsm_last_error())


def _ptr(a):
    """(pointer, on_device, keepalive) for a numpy array or torch tensor (or None)."""
    if a is None:
        return None, 0, None
    if hasattr(a, "data_ptr"):  # torch tensor
        a = a.contiguous()
        return ctypes.c_void_p(a.data_ptr()), int(a.is_cuda), a
    a = np.ascontiguousarray(a)
    return ctypes.c_void_p(a.ctypes.data), 0, a


def _check_array(name, a, dtypes, length):
    """dtype and length of a numpy array / torch tensor passed to the C ABI by pointer."""
    dt = str(a.dtype).replace("torch.", "")
    if dt not in dtypes:
        raise ValueError(f"{name}: dtype {dt}, expected {' or '.join(dtypes)}")
    n = int(a.numel()) if hasattr(a, "numel") else int(np.asarray(a).size)
    if len(getattr(a, "shape", (n,))) != 1 or n != length:
        raise ValueError(f"{name}: expected a 1-D array of {length} elements, got shape {tuple(a.shape)}")


class Graph:
    """Handle returned by :func:`gsm_load_graph` (wraps ``gsm_graph*``)."""

    def __init__(self, handle: ctypes.c_void_p):
        self.handle = handle

    def info(self):
        return gsm_graph_info(self)

    def free(self):
        if self.handle:
            gsm_free(self)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()


def gsm_load_graph(num_nodes: int, row_offsets, col_indices, labels=None, device: int = 0, validate: bool = False,
                   stream: Optional[int] = None) -> Graph:
    """int64 offsets[n+1], int32 cols, optional uint32 labels; numpy/host or torch (host or CUDA).

    The arrays must already have exactly these dtypes and sizes (the C ABI reads raw
    pointers): a mismatch raises ValueError here instead of reading out of bounds."""
    _check_array("row_offsets", row_offsets, ("int64",), int(num_nodes) + 1)
    nnz = int(row_offsets[-1]) if int(num_nodes) >= 0 and len(row_offsets) else 0
    _check_array("col_indices", col_indices, ("int32",), nnz)
    if labels is not None:
        _check_array("labels", labels, ("uint32", "int32"), int(num_nodes))
    ro, od1, k1 = _ptr(row_offsets)
    co, od2, k2 = _ptr(col_indices)
    lo, od3, k3 = _ptr(labels)
    on_dev = od1 or od2 or (od3 if labels is not None else 0)
    if on_dev and not (od1 and od2 and (labels is None or od3)):
        raise ValueError("offsets, cols and labels must all be host or all be device arrays")
    opts = gsm_load_opts(ctypes.sizeof(gsm_load_opts), device, 1 if validate else 0, 0, stream)
    h = ctypes.c_void_p()
    _check(lib().gsm_load_graph(int(num_nodes), ro, co, lo, on_dev, ctypes.byref(opts), ctypes.byref(h)))
    del k1, k2, k3
    return Graph(h)


def gsm_free(g: Graph):
    _check(lib().gsm_free(g.handle))
    g.handle = None


def gsm_graph_info(g: Graph):
    n, m, lab, dev = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib().gsm_graph_info(g.handle, ctypes.byref(n), ctypes.byref(m), ctypes.byref(lab), ctypes.byref(dev)))
    return {"num_nodes": n.value, "num_directed_edges": m.value, "labeled": bool(lab.value), "device": dev.value}


def _query(num_nodes: int, edges: Sequence, labels):
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1))
    lab = None if labels is None else np.ascontiguousarray(np.asarray(labels, dtype=np.uint32))
    q = gsm_query(int(num_nodes), len(e) // 2, e.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)) if len(e) else None,
                  None if lab is None else lab.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
    return q, (e, lab)


class Result:
    """A finished gsm_match: counts, per-level statistics and (ENUMERATE) device rows."""

    def __init__(self, r: gsm_result):
        self.raw = r
        self.count = int(r.count)
        self.count_unique = int(r.count_unique)
        self.automorphisms = int(r.automorphisms)
        self.width = int(r.width)
        self.num_rows = int(r.num_rows)
        k = self.width
        self.order = list(r.order[:k])
        self.candidates = [int(x) for x in r.candidates[:k]]
        self.level_rows = [int(x) for x in r.level_rows[:k]]
        self.level_frontier_bytes = [int(x) for x in r.level_frontier_bytes[:k]]
        self.compressed = bool(r.compressed)
        self.level1_sharded = bool(r.level1_sharded)
        self.level_work = [int(x) for x in r.level_work[:k]]
        self.num_chunks = int(r.num_chunks)
        self.kernel_launches = int(r.kernel_launches)
        self.ms = {"total": r.ms_total, "plan": r.ms_plan, "filter": r.ms_filter, "expand": r.ms_expand,
                   "finalize": r.ms_finalize}
        self.prof = {name: {"launches": int(r.prof[i].launches), "ms": float(r.prof[i].ms),
                            "alg_bytes": float(r.prof[i].alg_bytes)} for i, name in enumerate(KERNEL_NAMES)}
        self.symmetric = bool(r.symmetric)

    def rows_numpy(self) -> np.ndarray:
        out = np.empty((self.num_rows, max(self.width, 1)), dtype=np.int32)
        if self.num_rows:
            _check(lib().gsm_result_copy_rows(ctypes.byref(self.raw), ctypes.c_void_p(out.ctypes.data), 0))
        return out

    def rows_torch(self, device=None):
        import torch
        out = torch.empty((self.num_rows, max(self.width, 1)), dtype=torch.int32,
                          device=device or f"cuda:{self.raw.device}")
        if self.num_rows:
            _check(lib().gsm_result_copy_rows(ctypes.byref(self.raw), ctypes.c_void_p(out.data_ptr()), 1))
        return out

    def free(self):
        gsm_result_free(self)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.free()


def gsm_match(g: Graph, num_nodes: int, edges: Sequence, labels=None, mode: int = GSM_MODE_COUNT, flags: int = 0,
              shard_index: int = 0, num_shards: int = 1, root_subset=None, mem_budget_bytes: int = 0,
              stream: Optional[int] = None, refine_rounds: int = 0, lookahead: int = 0) -> Result:
    """Count (mode=GSM_MODE_COUNT) or enumerate (GSM_MODE_ENUMERATE) the embeddings of the
    query (num_nodes, edges, labels) in g.  Rows are freed with gsm_result_free / Result.free."""
    q, keep = _query(num_nodes, edges, labels)
    rs = None if root_subset is None else np.ascontiguousarray(np.asarray(root_subset, dtype=np.int32))
    opts = gsm_match_opts(ctypes.sizeof(gsm_match_opts), mode, flags, shard_index, num_shards, refine_rounds, lookahead,
                          None if rs is None else rs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                          0 if rs is None else len(rs), mem_budget_bytes, stream)
    r = gsm_result()
    _check(lib().gsm_match(g.handle, ctypes.byref(q), ctypes.byref(opts), ctypes.byref(r)))
    del keep, rs
    return Result(r)


def gsm_result_free(res: Result):
    _check(lib().gsm_result_free(ctypes.byref(res.raw)))
    res.num_rows = 0


def gsm_result_copy_rows(res: Result, dst, dst_on_device: bool):
    p, _, keep = _ptr(dst)
    _check(lib().gsm_result_copy_rows(ctypes.byref(res.raw), p, 1 if dst_on_device else 0))
    del keep


def gsm_sort_rows(rows, max_id: int, stream: Optional[int] = None):
    """In-place lexicographic sort of a CUDA int32 tensor (num_rows x width), values in [0, max_id]."""
    if not (hasattr(rows, "is_cuda") and rows.is_cuda and rows.is_contiguous() and rows.dim() == 2):
        raise ValueError("gsm_sort_rows needs a contiguous 2-D CUDA int32 tensor")
    _check(lib().gsm_sort_rows(ctypes.c_void_p(rows.data_ptr()), rows.shape[0], rows.shape[1], int(max_id),
                               rows.device.index or 0, stream))
    return rows


def gsm_merge_rows(a, b, stream: Optional[int] = None):
    """Merge two lexicographically sorted CUDA int32 row tensors (na x w, nb x w) on the same
    device into a new (na + nb) x w tensor (the library's merge-path kernel)."""
    import torch
    for name, t in (("a", a), ("b", b)):
        if not (hasattr(t, "is_cuda") and t.is_cuda and t.is_contiguous() and t.dim() == 2 and t.dtype == torch.int32):
            raise ValueError(f"gsm_merge_rows: {name} must be a contiguous 2-D CUDA int32 tensor")
    if a.shape[1] != b.shape[1] or a.device != b.device:
        raise ValueError("gsm_merge_rows: a and b need the same width and device")
    out = torch.empty((a.shape[0] + b.shape[0], a.shape[1]), dtype=torch.int32, device=a.device)
    _check(lib().gsm_merge_rows(ctypes.c_void_p(a.data_ptr()), a.shape[0], ctypes.c_void_p(b.data_ptr()), b.shape[0],
                                a.shape[1], ctypes.c_void_p(out.data_ptr()), a.device.index or 0, stream))
    return out


def gsm_filter_candidates(g: Graph, num_nodes: int, edges: Sequence, labels=None, refine_rounds: int = 0):
    """Candidate masks of the filter step (Alg. 1 lines 6-9): uint32 array, entry v (original
    id) has bit u set iff v is a candidate of query vertex u."""
    q, keep = _query(num_nodes, edges, labels)
    n = gsm_graph_info(g)["num_nodes"]
    out = np.zeros(n, dtype=np.uint32)
    _check(lib().gsm_filter_candidates(g.handle, ctypes.byref(q), int(refine_rounds), ctypes.c_void_p(out.ctypes.data), 0))
    del keep
    return out


def gsm_plan_query(num_nodes: int, edges: Sequence, labels=None, candidates=None, flags: int = 0) -> dict:
    """Host-only query plan (order, parents, backward masks, ID constraints, |Aut(Q)|)."""
    q, keep = _query(num_nodes, edges, labels)
    cand = None if candidates is None else np.ascontiguousarray(np.asarray(candidates, dtype=np.uint64))
    info = gsm_plan_info()
    _check(lib().gsm_plan_query(ctypes.byref(q), None if cand is None else ctypes.c_void_p(cand.ctypes.data),
                                flags, ctypes.byref(info)))
    k = info.k
    return {"order": list(info.order[:k]), "parent": list(info.parent[:k]), "backward": list(info.backward[:k]),
            "conditions": [(info.cond_lo[c], info.cond_hi[c]) for c in range(info.num_conditions)],
            "automorphisms": int(info.automorphisms)}
