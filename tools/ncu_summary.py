#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) or launch-list CSV into profiles/.

    python tools/ncu_summary.py full  gpurun_out/prof.ncu-rep  <workload> [alg_bytes_per_launch]
    python tools/ncu_summary.py launches gpurun_out/launches.csv <out.md>

`full` merges the per-kernel metrics of a `--set full` capture into
profiles/ncu_summary.json under <workload> (bench.py reads `traffic` from it).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct": "ld_sector_efficiency_pct",
    "launch__registers_per_thread": "registers",
    "launch__occupancy_limit_registers": "occ_limit_regs",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__maximum_warps_per_active_cycle_pct": "theoretical_occupancy_pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard": "stall_long_scoreboard",
}


def raw_rows(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rd = list(csv.reader(io.StringIO(out)))
    header, units, rows = rd[0], rd[1], rd[2:]
    return header, units, rows


def kname(raw):
    """'void gsm::k_tail<unsigned char>(TailArgs, ...)' -> 'k_tail'"""
    base = raw.split("(")[0].split("<")[0].strip()
    return base.split()[-1].split("::")[-1]


def to_float(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def full(rep, workload, alg=None):
    header, units, rows = raw_rows(rep)
    idx = {h: i for i, h in enumerate(header)}
    kidx = idx.get("Kernel Name")
    per = defaultdict(list)
    for r in rows:
        name = kname(r[kidx])
        d = {}
        for m, key in METRICS.items():
            if m in idx:
                v = to_float(r[idx[m]])
                u = units[idx[m]]
                if v is not None and key == "duration":
                    v = v * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(u, 1e-9)
                if v is not None and key in ("dram_read", "dram_write"):
                    v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                             "GB": 1e9}.get(u, 1)
                d[key] = v
        per[name].append(d)
    summ = {}
    for name, lst in per.items():
        agg = {k: sum(x.get(k) or 0 for x in lst) / len(lst) for k in lst[0]}
        agg["launches_captured"] = len(lst)
        if "dram_read" in agg:
            agg["dram_bytes_per_launch"] = agg["dram_read"] + agg.get("dram_write", 0)
        summ[name] = agg
    if alg is not None and "k_expand" in summ:
        summ["k_expand"]["alg_bytes_per_launch"] = alg
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        allp = json.load(open(path))
    except (OSError, ValueError):
        allp = {}
    allp[workload] = summ
    json.dump(allp, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(summ, indent=1))


def launches(csvpath, outmd):
    txt = open(csvpath).read()
    start = txt.find('"ID"')
    rd = list(csv.reader(io.StringIO(txt[start:])))
    header, rows = rd[0], rd[1:]
    idx = {h: i for i, h in enumerate(header)}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if len(r) < len(header) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = kname(r[idx["Kernel Name"]])
        v = to_float(r[idx["Metric Value"]]) or 0.0
        unit = r[idx["Metric Unit"]]
        v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(unit, 1e-3)
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| {name} | {cnt[name]} | {v:.1f} | {v / total:.1%} |")
    open(outmd, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def metrics(csvpath, workload):
    """Per-kernel mean DRAM bytes / duration per launch from an `ncu --metrics ... --csv` log;
    merged into profiles/ncu_summary.json under <workload> (bench.py reads `traffic`)."""
    txt = open(csvpath).read()
    start = txt.find('"ID"')
    rd = list(csv.reader(io.StringIO(txt[start:])))
    header, rows = rd[0], rd[1:]
    idx = {h: i for i, h in enumerate(header)}
    per = defaultdict(lambda: defaultdict(list))
    for r in rows:
        if len(r) < len(header):
            continue
        name = kname(r[idx["Kernel Name"]])
        m = r[idx["Metric Name"]]
        v = to_float(r[idx["Metric Value"]])
        u = r[idx["Metric Unit"]]
        if v is None:
            continue
        if m.startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
        if m == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(u, 1e-9)
        per[name][m].append(v)
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        allp = json.load(open(path))
    except (OSError, ValueError):
        allp = {}
    summ = allp.get(workload, {})
    for name, ms in per.items():
        n = max(len(v) for v in ms.values())
        rd_ = sum(ms.get("dram__bytes_read.sum", [0])) / n
        wr_ = sum(ms.get("dram__bytes_write.sum", [0])) / n
        dur = sum(ms.get("gpu__time_duration.sum", [0])) / n
        e = summ.setdefault(name, {})
        e.update({"launches_measured": n, "dram_read_per_launch": rd_, "dram_write_per_launch": wr_,
                  "dram_bytes_per_launch": rd_ + wr_, "duration_s_per_launch_ncu": dur,
                  "dram_bytes_total_in_capture": (rd_ + wr_) * n, "source": os.path.basename(csvpath)})
    allp[workload] = summ
    json.dump(allp, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "metrics":
        metrics(sys.argv[2], sys.argv[3])
        sys.exit(0)
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
