"""Print the key numbers of an ncu --set full report: SOL, issue, stalls, opcode mix."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
keys = ["Duration", "SM Frequency", "Memory Throughput", "DRAM Throughput", "L2 Cache Throughput",
        "L1/TEX Cache Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "L2 Hit Rate", "Registers Per Thread", "Achieved Occupancy",
        "Issued Instructions"]
for line in det.splitlines():
    t = line.strip()
    for k in keys:
        if t.startswith(k + " "):
            print("  " + " ".join(t.split()))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
ie = h.index("Instructions Executed")
names = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
ops, stalls, tot = Counter(), Counter(), 0
for r in rows[2:]:
    try:
        n = float(r[ie] or 0)
    except (ValueError, IndexError):
        continue
    text = r[1].strip()
    parts = text.split()
    if not parts:
        continue
    op = parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]
    ops[op.split(".")[0]] += n
    tot += n
    for k in names:
        try:
            stalls[k] += float(r[h.index(k)] or 0)
        except ValueError:
            pass
print(f"  instructions {tot:.4g}")
print("  top ops: " + ", ".join(f"{o} {100*n/tot:.1f}%" for o, n in ops.most_common(10)))
st = sum(stalls.values()) or 1
print("  stalls: " + ", ".join(f"{k[6:]} {100*v/st:.0f}%" for k, v in stalls.most_common(6)))
