import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.check_output(["ncu", "-i", rep, "--page", "details", "--csv"], text=True, stderr=subprocess.DEVNULL)
r = list(csv.reader(out.splitlines()))
h = r[0]
iN, iV, iU, iK = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Kernel Name")
want = ["Duration", "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Compute (SM) Throughput", "Memory Throughput",
        "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Grid Size", "L2 Cache Throughput", "Issue Slots Busy", "Block Limit Shared Mem", "Block Limit Registers"]
seen = set()
for x in r[1:]:
    key = (x[0], x[iN])
    if x[iN] in want and key not in seen:
        seen.add(key)
        print(x[0], x[iK][:40], x[iN], x[iV], x[iU])
src = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv"], text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(src.splitlines()))
hh = rows[1]
iS, iE = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
def _isint(v):
    try:
        int(v)
        return True
    except ValueError:
        return False


body = [x for x in rows[2:] if len(x) == len(hh) and _isint(x[iS]) and _isint(x[iE])]
tot = sum(int(x[iS]) for x in body)
print("stall samples", tot, "instructions", sum(int(x[iE]) for x in body))
for x in sorted(body, key=lambda x: -int(x[iS]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(" ", x[iS], x[iE], x[1].strip()[:90])
