"""Multi-rank path on one GPU (functional): two processes share cuda:0 and
talk over gloo.  multigpu.match_sharded must reproduce the single-process
result (count and the full sorted row list, merged by the gsm_merge_rows tree), and
bench.py under torchrun must report the same total as one rank."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gsm_inputs as gi
        from paper_2003_01527_b200 import gsm, multigpu
        g = gi.rmat(11, 8, seed=31).with_labels(gi.uniform_labels(2048, 2, 31))
        G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=0)
        res = {}
        for name, q in [("K3", gi.query("K3")), ("P4", gi.query("P4", [0, 1, 1, 0])), ("K4", gi.query("K4"))]:
            c, cu, _ = multigpu.match_sharded(G, q.num_nodes, q.edges, q.labels, mode=gsm.GSM_MODE_COUNT, dist=dist)
            ce, _, rows = multigpu.match_sharded(G, q.num_nodes, q.edges, q.labels, mode=gsm.GSM_MODE_ENUMERATE,
                                                 dist=dist, num_graph_nodes=g.num_nodes)
            res[name] = (c, cu, ce, rows.cpu().numpy().tolist())
        G.free()
        if rank == 0:
            out_q.put(res)
    finally:
        dist.destroy_process_group()


def test_match_sharded_two_ranks_one_gpu():
    import gsm_inputs as gi
    import oracle
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q_out)) for r in range(2)]
    for p in procs:
        p.start()
    got = q_out.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = gi.rmat(11, 8, seed=31).with_labels(gi.uniform_labels(2048, 2, 31))
    for name, q in [("K3", gi.query("K3")), ("P4", gi.query("P4", [0, 1, 1, 0])), ("K4", gi.query("K4"))]:
        cnt, ref = oracle.match(g, q)
        c, cu, ce, rows = got[name]
        assert c == ce == cnt
        assert np.array_equal(np.asarray(rows, np.int32).reshape(-1, q.num_nodes), ref)


def test_bench_two_ranks_one_gpu_counts_match():
    env = dict(os.environ, GSM_BENCH_ONE_DEVICE="1")
    base = [sys.executable, "bench.py", "--workload", "rmat16", "--steps", "1", "--warmup", "1",
            "--no-cpu-baseline", "--e2e-steps", "0"]
    one = subprocess.run(base, cwd=ROOT, capture_output=True, text=True, timeout=900)
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_free_port())] + base[1:] + ["--gpus", "2"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert one.returncode == 0, one.stderr[-2000:]
    assert two.returncode == 0, two.stderr[-2000:]
    j1 = json.loads(one.stdout.strip().splitlines()[-1])
    j2 = json.loads(two.stdout.strip().splitlines()[-1])
    assert j2["n_gpus"] == 2 and j2["counts_per_step"] == j1["counts_per_step"]
