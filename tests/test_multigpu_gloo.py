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
            allr = multigpu.allgather_rows(torch.from_numpy(rows), dist)
            merged = oracle.sort_rows(allr.numpy())  # stands in for gsm_sort_rows (GPU)
            res[qname] = (tot, tot2, merged)
        # empty shard on one rank
        empty = torch.zeros((0, 3), dtype=torch.int32) if rank == 0 else torch.tensor([[1, 2, 3]], dtype=torch.int32)
        res["empty"] = multigpu.allgather_rows(empty, dist).numpy()
        if rank == 0:
            out_q.put({k: (v if k == "empty" else (v[0], v[1], v[2].tolist())) for k, v in res.items()})
    finally:
        dist.destroy_process_group()


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
