"""Multi-GPU GSM: one process per GPU, data graph replicated, root candidates
sharded (BASELINE north_star).

Embeddings are partitioned by the image of the first query position π[0]:
each rank keeps the roots whose (degree, id) rank r satisfies r % P == rank
(hubs spread round-robin), runs the whole hot path on them with no exchange,
and the ranks meet once at the end:
  * COUNT      — one all-reduce of the uint64 counts (16 B);
  * ENUMERATE  — all-gather of the per-rank row counts, then every rank's
                 exact-size row block by one broadcast per source rank (an
                 all-gather-v: no padding to the largest shard), then a tree
                 of pairwise merges of the locally sorted shards
                 (gsm_merge_rows, the library's merge-path kernel): log2 P
                 rounds, no re-sort of the concatenation.
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


def gather_row_blocks(rows, dist) -> list:
    """All-gather-v of variable-length row blocks (N_r x k int32 tensors): the per-rank counts
    first, then each rank's block at its exact size by a broadcast from that rank.  Returns
    the list of blocks in rank order (this rank's own block is ``rows`` itself)."""
    import torch
    if _host_collectives(dist) and rows.is_cuda:
        return [b.to(rows.device) for b in gather_row_blocks(rows.cpu(), dist)]
    world, me = dist.get_world_size(), dist.get_rank()
    k = rows.shape[1]
    n = torch.tensor([rows.shape[0]], dtype=torch.int64, device=rows.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(x.item()) for x in sizes]
    blocks = []
    for r in range(world):
        if sizes[r] == 0:
            blocks.append(rows.new_zeros((0, k)))
            continue
        buf = rows.contiguous() if r == me else rows.new_empty((sizes[r], k))
        dist.broadcast(buf, src=r)
        blocks.append(buf)
    return blocks


def merge_sorted_blocks(blocks: list, merge_fn: Callable):
    """Tree of pairwise merges of lexicographically sorted row blocks (ceil(log2 P) rounds)."""
    blocks = [b for b in blocks if b.shape[0] > 0] or blocks[:1]
    while len(blocks) > 1:
        nxt = [merge_fn(blocks[i], blocks[i + 1]) for i in range(0, len(blocks) - 1, 2)]
        if len(blocks) % 2:
            nxt.append(blocks[-1])
        blocks = nxt
    return blocks[0]


def allgather_rows(rows, dist, merge_fn: Optional[Callable] = None):
    """All sorted row blocks of every rank merged into one sorted block (on every rank)."""
    blocks = gather_row_blocks(rows, dist)
    if merge_fn is None:
        if not rows.is_cuda:
            raise ValueError("allgather_rows: host row blocks need an explicit merge_fn (the library merges on the GPU)")
        merge_fn = gsm.gsm_merge_rows
    return merge_sorted_blocks(blocks, merge_fn)


def match_sharded(G: "gsm.Graph", num_nodes: int, edges, labels=None, mode: int = gsm.GSM_MODE_COUNT, flags: int = 0,
                  dist=None, num_graph_nodes: Optional[int] = None, mem_budget_bytes: int = 0,
                  stream: Optional[int] = None, merge_fn: Optional[Callable] = None):
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
            local = r.rows_torch(dev)  # sorted by gsm_match
            if dist is not None and world > 1:
                rows = allgather_rows(local, dist, merge_fn)
            else:
                rows = local
        return count, count_unique, rows
    finally:
        r.free()
