#!/usr/bin/env python
"""bench.py — device-timed GSM hot path (BASELINE.json metric: embeddings/s and
query ms at 1/2/4/8 B200; achieved HBM GB/s vs peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload rmat24] [--impl ours|reference]

A step = one pass of the whole hot path over the workload: gsm_match (COUNT)
of every query of the workload on the resident data graph
(filter -> roots -> per-position plan/scan/partition/expand -> count).  Default
workload = BASELINE configs[4] (R-MAT-24, K3 + K4, chunked frontier), the
configuration the metric is quoted on at 1/2/4/8 GPUs.  Multi-GPU: one process
per GPU (torchrun), data graph replicated (each rank regenerates it), root
candidates sharded round-robin by (degree, id) rank, one NCCL all-reduce of
the counts per step (inside the timed region); time = max over ranks.
value = UNIQUE embeddings/s (one per Aut(Q) orbit — what the kernels search for;
the all-embeddings figure |Aut(Q)| x unique is reported as all_per_s).

--impl reference: the CPU oracle (oracle/, plain DFS) timed on this host's
cores on a bounded root sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--workload", default=os.environ.get("GSM_BENCH_WORKLOAD", "rmat24"))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--e2e-steps", type=int, default=2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=8.0, help="oracle sample budget per pass (cpu_baseline)")
    p.add_argument("--refine-rounds", type=int, default=0, help="NE filter rounds (Alg. 1 lines 7-8)")
    p.add_argument("--mode", default="count", choices=["count", "enumerate"],
                   help="enumerate: rows materialised, sorted (device-timed) and copied D2H (e2e)")
    p.add_argument("--clique", type=int, default=1, help="0: K3/K4 take the breadth-first path (GSM_CLIQUE=0)")
    p.add_argument("--lookahead", type=int, default=0, help="k-look-ahead depth (0/1/2)")
    p.add_argument("--compressed", action="store_true", help="compressed partial results")
    p.add_argument("--shard-level", type=int, default=1, choices=[0, 1],
                   help="N>1: shard by root (0) or by level-1 pair where level 1 is a breadth-first expand (1)")
    return p.parse_args()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # let nvidia-smi finish its NVML start-up before the timed region: measured, its
            # start-up overlapping a short timed region added 2-40 ms of host-side gaps per step
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:  # timed region shorter than one 200 ms sample: one query right after it
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=30)
                parts = [x.strip() for x in out.stdout.strip().split(",")]
                reasons = sorted(nm for nm, v in zip(names, parts[3:7]) if v.lower().startswith("active"))
                return {"sm_mhz": float(parts[0]), "sm_max_mhz": float(parts[1]), "reasons": reasons,
                        "samples": 0, "note": "timed region < 200 ms; sampled once right after it"}
            except Exception:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- distributed
# GSM_BENCH_ONE_DEVICE=1: every rank uses cuda:0 and the collectives go over gloo — a
# functional check of the multi-rank path on a single-GPU box (NCCL needs one GPU per rank);
# never a scaling measurement.
ONE_DEVICE = os.environ.get("GSM_BENCH_ONE_DEVICE", "0") == "1"


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if ONE_DEVICE else int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if (args.impl == "ours" and not ONE_DEVICE) else "gloo"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
        pg = dist
    return world, rank, local, pg


def load_peaks():
    """MEASURED_PEAKS.json (driver-written); if absent, the fallback the profiling guide
    states (6.65 TB/s copy, an earlier measurement on this pool) marked as such."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        d["_source"] = "MEASURED_PEAKS.json hbm_gbs (copy, burst) - of measured"
        return d
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "_source": "fallback 6.65 TB/s (B200_PROFILING.md; MEASURED_PEAKS.json absent) - of fallback"}


KERNELS_OF = {"expand": ["k_expand", "k_count_walk"], "tail": ["k_tail", "k_tail_block"],
              "clique": ["k_clique_cta", "k_clique_warp"], "filter": ["k_filter"],
              "plan": ["k_plan_rows", "k_plan_rows_grp"], "roots": ["k_root_count", "k_root_write"]}


def ncu_traffic(workload: str, kind: str, launches_per_step: float):
    """DRAM bytes (ncu dram__bytes_read.sum + dram__bytes_write.sum) per recorder launch of this
    kind: the bytes of all its kernels in the one-step capture (profiles/ncu_summary.json, written
    by tools/ncu_summary.py metrics from `bench.py --steps 1 --warmup 0` under ncu) divided by
    the recorder launches per step — the unit `alg_bytes_per_launch` is in.  (None if absent.)"""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(path)).get(workload, {})
    except (OSError, ValueError):
        return None, None
    names = [n for n in KERNELS_OF.get(kind, []) if d.get(n, {}).get("dram_bytes_total_in_capture") is not None]
    if not names or not launches_per_step:
        return None, None
    tot = sum(d[n]["dram_bytes_total_in_capture"] for n in names)
    return tot / launches_per_step, "+".join(names)


# ----------------------------------------------------------------------------- oracle baseline
METRIC = "embeddings/s (unique: one per Aut(Q) orbit, i.e. per matched subgraph)"


def strided_roots(n: int, count: int):
    import numpy as np
    count = max(1, min(n, int(count)))
    stride = n / count
    return np.unique((np.arange(count) * stride + stride / 2).astype(np.int64).clip(0, n - 1)).astype(np.int32)


def oracle_pass(g, queries, roots):
    """One oracle pass (plain DFS, all embeddings with f(query vertex 0) in roots) over the
    workload's queries; returns (unique-equivalent embeddings = sum all/|Aut(Q)|, seconds)."""
    import oracle
    t0 = time.perf_counter()
    uni = 0.0
    for q in queries:
        c = oracle.match(g, q, roots=roots, count_only=True)[0]
        uni += c / len(oracle.automorphisms(q))
    return uni, time.perf_counter() - t0


_SHM = {}  # id(graph) -> (graph, directory of its .npy arrays) for spawned oracle children;
# the graph itself is kept referenced so its id cannot be reused by a later graph


def _graph_files(g):
    """The graph's arrays as .npy files (in /dev/shm when present) for a spawned child to mmap."""
    import tempfile

    import numpy as np
    key = id(g)
    if key not in _SHM or _SHM[key][0] is not g:
        d = tempfile.mkdtemp(prefix="gsm_oracle_", dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
        np.save(os.path.join(d, "offsets.npy"), g.offsets)
        np.save(os.path.join(d, "cols.npy"), g.cols)
        if g.labels is not None:
            np.save(os.path.join(d, "labels.npy"), g.labels)
        import atexit
        import shutil
        atexit.register(shutil.rmtree, d, True)
        _SHM[key] = (g, d)
    return _SHM[key][1]


def _pass_child(conn, d, n, queries, roots):
    import numpy as np

    import gsm_inputs as gi
    lab = os.path.join(d, "labels.npy")
    g = gi.Graph(n, np.load(os.path.join(d, "offsets.npy"), mmap_mode="r"),
                 np.load(os.path.join(d, "cols.npy"), mmap_mode="r"),
                 np.load(lab, mmap_mode="r") if os.path.exists(lab) else None)
    conn.send(oracle_pass(g, queries, roots))
    conn.close()


def oracle_pass_bounded(g, queries, roots, limit_s: float):
    """oracle_pass in a SPAWNED child (the graph mmapped from .npy files), killed after limit_s:
    per-root DFS cost is heavy-tailed (one R-MAT hub root can take hours), so a calibration pass
    must be interruptible without touching the oracle.  Spawn, not fork: a forked child of a
    process whose OpenMP runtime (input generator) or CUDA context is live hangs (measured: every
    forked pass timed out and the sample shrank to one root).  None on timeout."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    a, b = ctx.Pipe(duplex=False)
    p = ctx.Process(target=_pass_child, args=(b, _graph_files(g), g.num_nodes, queries, roots), daemon=True)
    p.start()
    b.close()
    res = a.recv() if a.poll(limit_s + 10.0) else None  # + interpreter start-up
    if p.is_alive():
        p.kill()
    p.join()
    return res


def oracle_sample(g, queries, target_s: float):
    """A FIXED evenly strided root sample sized so one oracle pass takes about target_s:
    start at 16 roots, grow geometrically while a pass is < target/3, shrink on a pass
    over 1.5 x target (such a pass is killed at that limit, so calibration stays bounded
    even when the sample hits a hub).  Returns (roots, unique, seconds, threads)."""
    import oracle
    n = g.num_nodes
    cnt = 16
    best = None
    for _ in range(16):
        roots = strided_roots(n, cnt)
        res = oracle_pass_bounded(g, queries, roots, 1.5 * target_s)
        if res is None:  # over the limit: shrink, and never grow past this size again
            cnt = max(1, cnt // 2) if cnt > 1 else 1
            if cnt == 1 and best is None:
                roots = strided_roots(n, 1)
                uni, dt = oracle_pass(g, queries, roots)
                return roots, uni, dt, oracle.num_threads()
            continue
        uni, dt = res
        best = (roots, uni, dt)
        if dt < target_s / 3 and cnt < n:
            cnt = min(n, int(cnt * min(8.0, max(1.5, 0.9 * target_s / max(dt, 1e-4)))))
            continue
        break
    roots, uni, dt = best
    return roots, uni, dt, oracle.num_threads()


def cpu_baseline(g, w, budget_s):
    roots, uni, dt, threads = oracle_sample(g, w.queries, budget_s)
    return {"value": uni / dt if (dt > 0 and uni > 0) else None, "unit": METRIC, "cores": threads, "kind": "oracle",
            "sample": f"all embeddings of {[q.name for q in w.queries]} with f(query vertex 0) in a fixed evenly "
                      f"strided sample of {len(roots)} of {g.num_nodes} vertices, counted as all/|Aut(Q)|; "
                      f"{uni:.6g} unique-equivalent embeddings in {dt:.2f} s (one pass)"}


def run_reference(args, world, rank):
    """Reference arm = the CPU oracle as it stands (plain DFS, oracle/), rank 0 only, on a
    fixed root sample whose per-step cost is sized so the WHOLE run (calibration, W warm-up
    and K timed passes) stays within ~240 s whatever --steps/--warmup are."""
    import oracle  # noqa: F401  (reference arm = the CPU oracle)
    from gsm_inputs import workloads

    if rank != 0:
        return
    w = workloads.get(args.workload)
    g = w.graph()
    per_step = max(0.3, min(8.0, 240.0 / (args.steps + args.warmup + 4)))
    roots, _, _, threads = oracle_sample(g, w.queries, per_step)
    for _ in range(max(0, args.warmup - 1)):  # the accepted calibration pass was one warm-up
        oracle_pass(g, w.queries, roots)
    tot = 0.0
    times = []
    for _ in range(args.steps):  # same deterministic sample as the accepted calibration pass
        uni, dt = oracle_pass(g, w.queries, roots)
        tot += uni
        times.append(dt)
    dt = sum(times)
    value = tot / dt
    sample = (f"all embeddings of {[q.name for q in w.queries]} with f(query vertex 0) in a fixed evenly strided "
              f"sample of {len(roots)} of {g.num_nodes} vertices per step, counted as all/|Aut(Q)|")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
           "ms_median": 1000 * statistics.median(times),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
           "data": "synthetic", "config": config_of(w, g),
           "cpu_baseline": {"value": value, "unit": METRIC, "cores": threads, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def config_of(w, g, refine_rounds=0, args=None):
    extra = {}
    if args is not None:
        extra = {"match_mode": args.mode, "clique_path": bool(args.clique), "lookahead": args.lookahead,
                 "compressed_partials": bool(args.compressed),
                 "sharding": "level-1 pairs where level 1 is a breadth-first expand, else roots"
                             if args.shard_level == 1 else "roots (rank % P)"}
    return {"workload": f"{w.name} (BASELINE configs[{w.config_index}]): {w.description}",
            "refine_rounds": refine_rounds, **extra,
            "graph": {"name": g.name, "num_nodes": g.num_nodes, "directed_edges": g.nnz,
                      "csr_bytes": int(g.offsets.nbytes + g.cols.nbytes + (0 if g.labels is None else g.labels.nbytes))},
            "queries": [q.name for q in w.queries],
            "mode": "count; value = unique embeddings (one per Aut(Q) orbit, what the kernels find); "
                    "all embeddings = |Aut(Q)| x unique in counts_per_step / all_per_s",
            "mem_budget_bytes": w.mem_budget_bytes,
            "l2": "inputs larger than L2 (no flush)" if g.offsets.nbytes + g.cols.nbytes > 126e6
                  else "graph smaller than L2: L2 flushed (256 MiB write) before every timed step"}


# ----------------------------------------------------------------------------- ours
def run_ours(args, world, rank, local, dist):
    import numpy as np
    import torch

    from gsm_inputs import workloads
    from paper_2003_01527_b200 import gsm

    if not args.clique:
        os.environ["GSM_CLIQUE"] = "0"  # read by the library at every gsm_match
    w = workloads.get(args.workload)
    if dist is not None:  # rank 0 generates (all host cores) and fills the on-disk cache; the others load it
        if rank == 0:
            g = w.graph()
        dist.barrier()
        if rank != 0:
            g = w.graph()
    else:
        g = w.graph()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    G = gsm.gsm_load_graph(g.num_nodes, g.offsets, g.cols, g.labels, device=local)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    graph_bytes = g.offsets.nbytes + g.cols.nbytes
    flush = None
    if graph_bytes <= 126e6:
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    per_query = {}

    enumerate_ = args.mode == "enumerate"
    extra_flags = gsm.GSM_FLAG_COMPRESSED_PARTIALS if args.compressed else 0
    if world > 1 and args.shard_level == 1:
        extra_flags |= gsm.GSM_FLAG_SHARD_LEVEL1
    host_rows = {}  # e2e (enumerate): pinned destination of each query's rows

    def step(flags, G_=None, d2h=False):
        G_ = G_ or G
        tot_all = tot_unique = launches = 0
        profs = []
        for q in w.queries:
            r = gsm.gsm_match(G_, q.num_nodes, q.edges, q.labels,
                              mode=gsm.GSM_MODE_ENUMERATE if enumerate_ else gsm.GSM_MODE_COUNT,
                              flags=flags | extra_flags, shard_index=rank, num_shards=world,
                              mem_budget_bytes=w.mem_budget_bytes, stream=sptr, refine_rounds=args.refine_rounds,
                              lookahead=args.lookahead)
            tot_all += r.count
            tot_unique += r.count_unique
            launches += r.kernel_launches
            profs.append(r.prof)
            if enumerate_:
                if d2h and r.num_rows:  # rows to pinned host memory through the C ABI
                    hb = host_rows.get(q.name)
                    if hb is None or hb.numel() < r.num_rows * r.width:
                        hb = torch.empty(r.num_rows * r.width, dtype=torch.int32).pin_memory()
                        host_rows[q.name] = hb
                    gsm.gsm_result_copy_rows(r, hb, False)
                    host_rows[q.name + ":bytes"] = r.num_rows * r.width * 4
                r.free()
            if G_ is not G:
                continue  # e2e steps (fresh graph each step) do not overwrite the resident-graph stats
            per_query[q.name] = {"count": r.count, "unique": r.count_unique, "automorphisms": r.automorphisms,
                                 "order": r.order, "candidates": r.candidates, "level_work": r.level_work,
                                 "level_rows": r.level_rows, "chunks": r.num_chunks,
                                 "level_frontier_bytes": r.level_frontier_bytes, "compressed": r.compressed,
                                 "ms": {k: round(v, 3) for k, v in r.ms.items()},
                                 "kernel_ms": {k: round(v["ms"], 3) for k, v in r.prof.items()}}
        return tot_all, tot_unique, launches, profs

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        if flush is not None:
            flush.zero_()
        step(gsm.GSM_FLAG_PROFILE)
    barrier()
    ms_steps = []
    counts = None
    launches = 0
    prof_tot = {}
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            if flush is not None:
                flush.zero_()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            c_all, c_uni, nl, profs = step(gsm.GSM_FLAG_PROFILE)
            if dist is not None and not ONE_DEVICE:  # the step's count all-reduce (NCCL) is in the timed region
                red = torch.tensor([c_all, c_uni], dtype=torch.int64, device=dev)
                dist.all_reduce(red)
            ev1.record(stream)
            ev1.synchronize()
            ms_steps.append(ev0.elapsed_time(ev1))
            counts = (c_all, c_uni)
            launches += nl
            for p in profs:
                for kname, d in p.items():
                    t = prof_tot.setdefault(kname, {"launches": 0, "ms": 0.0, "alg_bytes": 0.0})
                    for key in t:
                        t[key] += d[key]
    barrier()
    ms = sum(ms_steps) / len(ms_steps)
    ms_med = statistics.median(ms_steps)
    c_all, c_uni = counts
    cdev = "cpu" if ONE_DEVICE else dev
    per_rank_ms = [ms]
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=cdev)
        gathered = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        per_rank_ms = [float(x.item()) for x in gathered]
        ms = max(per_rank_ms)
        t = torch.tensor([ms_med], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_med = float(t.item())
        c = torch.tensor([c_all, c_uni, launches], dtype=torch.int64, device=cdev)
        dist.all_reduce(c)
        c_all, c_uni, launches = (int(x) for x in c.tolist())

    # ---- end to end through the C ABI with host buffers (pinned), per step:
    #      H2D CSR + relabel (gsm_load_graph) + matches + D2H counts + gsm_free
    e2e = None
    if args.e2e_steps > 0:
        off_h = torch.from_numpy(g.offsets).pin_memory()
        cols_h = torch.from_numpy(g.cols).pin_memory()
        lab_h = None if g.labels is None else torch.from_numpy(g.labels.view(np.int32)).pin_memory()
        # one untimed end-to-end step first (the W warm-up rule): the first upload of a fresh
        # graph maps the memory pool's pages (measured ~120 ms extra on R-MAT-24)
        G2 = gsm.gsm_load_graph(g.num_nodes, off_h, cols_h, lab_h, device=local, stream=sptr)
        step(0, G2, d2h=True)
        G2.free()
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        e_cnt = 0
        for _ in range(args.e2e_steps):
            G2 = gsm.gsm_load_graph(g.num_nodes, off_h, cols_h, lab_h, device=local, stream=sptr)
            e_cnt = step(0, G2, d2h=True)[1]
            G2.free()
        ev1.record(stream)
        ev1.synchronize()
        e_ms = ev0.elapsed_time(ev1) / args.e2e_steps
        if dist is not None:
            t = torch.tensor([e_ms], dtype=torch.float64, device=cdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
            c = torch.tensor([e_cnt], dtype=torch.int64, device=cdev)
            dist.all_reduce(c)
            e_cnt = int(c.item())
        h2d = (g.offsets.nbytes + g.cols.nbytes + (0 if g.labels is None else g.labels.nbytes)) * world
        rows_d2h = sum(v for k, v in host_rows.items() if k.endswith(":bytes"))
        e2e = {"value": e_cnt / (e_ms / 1000.0), "unit": METRIC, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(8 * len(w.queries) * world + rows_d2h)}
    G.free()

    if rank != 0:
        return
    peaks = load_peaks()
    ex = prof_tot.get("expand", {"ms": 0, "alg_bytes": 0, "launches": 0})
    # dominant kernel = the one with the largest share of device time
    dom = max(prof_tot.items(), key=lambda kv: kv[1]["ms"])[0] if prof_tot else "expand"
    kp = prof_tot.get(dom, ex)
    achieved = (kp["alg_bytes"] / (kp["ms"] / 1e3)) / 1e9 if kp["ms"] > 0 else None
    peak = peaks.get("hbm_gbs")
    traffic, traffic_kernel = ncu_traffic(args.workload, dom, kp["launches"] / args.steps)
    roof = {"kernel": f"k_{dom}", "bound": "hbm", "achieved": achieved,
            "peak": peak, "unit": "GB/s", "frac": (achieved / peak) if (achieved and peak) else None,
            "traffic": traffic, "traffic_kernel": traffic_kernel,
            "traffic_source": "profiles/ncu_summary.json: ncu dram__bytes_read.sum+dram__bytes_write.sum of all "
                              "kernels of this kind in a one-step capture / recorder launches per step",
            "peak_source": peaks.get("_source", "absent"),
            "dram_gbs": (traffic / (kp["ms"] / max(1, kp["launches"]) / 1e3)) / 1e9
                        if (traffic and kp["ms"] > 0) else None,
            "dram_frac": (traffic / (kp["ms"] / max(1, kp["launches"]) / 1e3)) / 1e9 / peak
                         if (traffic and kp["ms"] > 0 and peak) else None,
            "launches_per_step": kp["launches"] / args.steps,
            "kernel_ms_per_step": kp["ms"] / args.steps,
            "alg_bytes_per_launch": kp["alg_bytes"] / max(1, kp["launches"]),
            "share_of_step": (kp["ms"] / args.steps) / ms if ms > 0 else None,
            "per_kernel_ms_per_step": {k: v["ms"] / args.steps for k, v in prof_tot.items()}}
    out = {"metric": METRIC, "value": c_uni / (ms / 1000.0), "unit": METRIC, "n_gpus": world,
           **({"one_device_functional_check": True} if ONE_DEVICE else {}),
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_median": ms_med,
           "per_rank_ms": per_rank_ms, "imbalance_max_over_mean": max(per_rank_ms) / (sum(per_rank_ms) / len(per_rank_ms)),
           "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
           "config": config_of(w, g, args.refine_rounds, args),
           "counts_per_step": {"all": c_all, "unique": c_uni},
           "all_per_s": c_all / (ms / 1000.0),
           "query_ms": ms, "per_query_rank0": per_query, "roofline": roof, "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e}
    # the oracle baseline runs AFTER the timed GPU work (its 16-thread passes must not share the
    # host with the timed steps), in spawned children (oracle_pass_bounded): spawn is safe from a
    # process with a live CUDA context, fork was not
    if world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline(g, w, args.cpu_seconds)
        except Exception as e:  # baseline failure must not hide the measurement
            out["cpu_baseline"] = {"value": None, "error": repr(e)}
    print(json.dumps(out), flush=True)


def main():
    args = parse_args()
    world, rank, local, dist = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
