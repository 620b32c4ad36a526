"""Summarise an ncu --csv launch list: per kernel name, mean duration / DRAM / L2 bytes."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    try:
        per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    names[r[idi]] = r[ki]
agg = defaultdict(lambda: defaultdict(list))
for i, m in per.items():
    n = names[i]
    if "sparton" not in n:
        continue
    short = n.split("(")[0].replace("void ", "")
    for k, v in m.items():
        agg[short][k].append(v)
for n, m in agg.items():
    cnt = len(m["gpu__time_duration.sum"])
    out = [f"{n[:70]:70s} x{cnt}"]
    for k in sorted(m):
        v = sum(m[k]) / len(m[k])
        out.append(f"{k.split('.')[0]}={v/1e6:.3f}{'ms' if 'time' in k else 'MB'}")
    print("  ".join(out))
