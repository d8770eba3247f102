"""N>1 host logic on CPU: world_size-2 gloo process group.
Each rank produces its root shard's embeddings (here with the oracle, since
there is no GPU in this container), then the product's collective code
(paper_2003_01527_b200.multigpu) combines them; the result must equal the
unsharded oracle result (count and sorted rows)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_roots(g, world, rank):
    # same rule as the product: rank the vertices by (degree, id), keep r % P == rank
    deg = np.diff(g.offsets)
    order = np.lexsort((np.arange(g.num_nodes), deg))
    return np.sort(order[rank::world]).astype(np.int32)


def _merge_host(a, b):
    """Two-pointer merge of two sorted host row blocks (stands in for gsm_merge_rows, GPU);
    unsigned lexicographic order, a first on ties."""
    A, B = a.numpy().view(np.uint32), b.numpy().view(np.uint32)
    out, i, j = [], 0, 0
    while i < len(A) or j < len(B):
        if j >= len(B) or (i < len(A) and tuple(A[i]) <= tuple(B[j])):
            out.append(a[i])
            i += 1
        else:
            out.append(b[j])
            j += 1
    return torch.stack(out) if out else a.new_zeros((0, a.shape[1]))


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gsm_inputs as gi
        import oracle
        from paper_2003_01527_b200 import multigpu

        g = gi.rmat(8, 8, seed=7)
        res = {}
        for qname in ["K3", "P4", "C4"]:
            q = gi.query(qname)
            c, rows = oracle.match(g, q, roots=_shard_roots(g, world, rank))
            tot, tot2 = multigpu.allreduce_counts([c, 2 * c], dist, "cpu")
            merged = multigpu.allgather_rows(torch.from_numpy(rows), dist, _merge_host).numpy()
            res[qname] = (tot, tot2, merged)
        # empty shard on one rank
        empty = torch.zeros((0, 3), dtype=torch.int32) if rank == 0 else torch.tensor([[1, 2, 3]], dtype=torch.int32)
        res["empty"] = multigpu.allgather_rows(empty, dist, _merge_host).numpy()
        if rank == 0:
            out_q.put({k: (v if k == "empty" else (v[0], v[1], v[2].tolist())) for k, v in res.items()})
    finally:
        dist.destroy_process_group()


def test_merge_tree_of_sorted_blocks():
    """merge_sorted_blocks: any number of sorted blocks (odd counts, empty ones) -> one
    sorted block equal to the sorted concatenation."""
    from paper_2003_01527_b200 import multigpu
    rng = np.random.default_rng(5)
    for nb in (1, 2, 3, 5, 8):
        blocks = []
        for _ in range(nb):
            x = rng.integers(0, 6, size=(int(rng.integers(0, 40)), 3)).astype(np.int32)
            blocks.append(torch.from_numpy(x[np.lexsort(x.T[::-1])].copy()))
        got = multigpu.merge_sorted_blocks(blocks, _merge_host).numpy()
        cat = np.concatenate([b.numpy() for b in blocks])
        assert np.array_equal(got, cat[np.lexsort(cat.T[::-1])])


def test_two_rank_gloo_combine():
    import gsm_inputs as gi
    import oracle

    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q_out)) for r in range(2)]
    for p in procs:
        p.start()
    got = q_out.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = gi.rmat(8, 8, seed=7)
    for qname in ["K3", "P4", "C4"]:
        cnt, rows = oracle.match(g, gi.query(qname))
        tot, tot2, merged = got[qname]
        assert tot == cnt and tot2 == 2 * cnt
        assert np.array_equal(np.asarray(merged, np.int32).reshape(-1, rows.shape[1]), rows)
    assert got["empty"].tolist() == [[1, 2, 3]]
