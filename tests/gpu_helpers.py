"""Helpers for the GPU parity tests: run the CUDA path through the C ABI
(paper_2003_01527_b200.gsm) on inputs from gsm_inputs, and compare with oracle."""
import numpy as np

from paper_2003_01527_b200 import gsm


def load(g, validate=True):
    return gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0, validate=validate)


def run(G, q, mode="count", flags=0, **kw):
    """Returns (count, rows or None, Result)."""
    m = gsm.GSM_MODE_ENUMERATE if mode == "enumerate" else gsm.GSM_MODE_COUNT
    r = gsm.gsm_match(G, q.num_nodes, q.edges, q.labels, mode=m, flags=flags, **kw)
    rows = None
    if m == gsm.GSM_MODE_ENUMERATE:
        rows = r.rows_numpy()
        r.free()
        assert rows.shape[0] == r.count
    return r.count, rows, r


def assert_rows_equal(gpu_rows, ref_rows, what=""):
    assert gpu_rows.shape == ref_rows.shape, (what, gpu_rows.shape, ref_rows.shape)
    if not np.array_equal(gpu_rows, ref_rows):
        bad = np.nonzero(np.any(gpu_rows != ref_rows, axis=1))[0]
        i = int(bad[0])
        raise AssertionError(f"{what}: {len(bad)} rows differ; first at {i}: gpu {gpu_rows[i].tolist()} "
                             f"oracle {ref_rows[i].tolist()}")


def is_sorted_unique(rows):
    if len(rows) < 2:
        return True
    k = rows.shape[1]
    a = rows[:-1].view(np.uint32)
    b = rows[1:].view(np.uint32)
    less = np.zeros(len(a), bool)
    decided = np.zeros(len(a), bool)
    for j in range(k):
        lt = (~decided) & (a[:, j] < b[:, j])
        gt = (~decided) & (a[:, j] > b[:, j])
        less |= lt
        decided |= lt | gt
    return bool(np.all(less))
