"""Multi-GPU GSM: one process per GPU, data graph replicated, root candidates
sharded (BASELINE north_star).

Embeddings are partitioned by the image of the first query position π[0]:
each rank keeps the roots whose (degree, id) rank r satisfies r % P == rank
(hubs spread round-robin), runs the whole hot path on them with no exchange,
and the ranks meet once at the end:
  * COUNT      — one all-reduce of the uint64 counts (16 B);
  * ENUMERATE  — all-gather of the per-rank row counts, all-gather of the rows
                 padded to the largest shard, then one lexicographic sort of
                 the concatenation (gsm_sort_rows, the library's radix sort).
torch.distributed is the plumbing (NCCL over NVLink on GPUs; gloo in the CPU
tests of the collective logic); the matching itself is libgsm's kernels.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

from . import gsm


def _host_collectives(dist) -> bool:
    """gloo (CPU tests, single-GPU functional checks) moves tensors through host memory."""
    return dist.get_backend() == "gloo"


def allreduce_counts(values: Sequence[int], dist, device) -> list:
    """Sum a few non-negative integer counts over all ranks (int64 tensor all-reduce)."""
    import torch
    dev = "cpu" if _host_collectives(dist) else device
    t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=dev)
    dist.all_reduce(t)
    return [int(x) for x in t.tolist()]


def allgather_rows(rows, dist):
    """All-gather variable-length row blocks (N_r x k int32 tensors) -> concatenation in rank order."""
    import torch
    if _host_collectives(dist) and rows.is_cuda:
        return allgather_rows(rows.cpu(), dist).to(rows.device)
    world = dist.get_world_size()
    k = rows.shape[1]
    n = torch.tensor([rows.shape[0]], dtype=torch.int64, device=rows.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    if mx == 0:
        return rows.new_zeros((0, k))
    padded = rows.new_zeros((mx, k))
    padded[: rows.shape[0]] = rows
    bufs = [rows.new_zeros((mx, k)) for _ in range(world)]
    dist.all_gather(bufs, padded)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0)


def match_sharded(G: "gsm.Graph", num_nodes: int, edges, labels=None, mode: int = gsm.GSM_MODE_COUNT, flags: int = 0,
                  dist=None, num_graph_nodes: Optional[int] = None, mem_budget_bytes: int = 0,
                  stream: Optional[int] = None, sort_fn: Optional[Callable] = None):
    """Run gsm_match on this rank's root shard and combine across ranks.
    Returns (count, count_unique, rows or None); rows (ENUMERATE) are the full,
    sorted embedding list on every rank."""
    import torch
    rank = dist.get_rank() if dist is not None else 0
    world = dist.get_world_size() if dist is not None else 1
    r = gsm.gsm_match(G, num_nodes, edges, labels, mode=mode, flags=flags, shard_index=rank, num_shards=world,
                      mem_budget_bytes=mem_budget_bytes, stream=stream)
    try:
        dev = torch.device("cuda", r.raw.device)
        count, count_unique = r.count, r.count_unique
        if dist is not None:
            count, count_unique = allreduce_counts([count, count_unique], dist, dev)
        rows = None
        if mode == gsm.GSM_MODE_ENUMERATE:
            local = r.rows_torch(dev)
            rows = allgather_rows(local, dist) if dist is not None else local
            if world > 1 and rows.shape[0]:
                n = num_graph_nodes if num_graph_nodes is not None else int(rows.max().item()) + 1
                (sort_fn or (lambda t: gsm.gsm_sort_rows(t, n - 1, stream)))(rows)
        return count, count_unique, rows
    finally:
        r.free()
