"""List hot SASS lines of an ncu source-page CSV (--page source --csv --print-source sass):
stall samples per instruction, plus every tcgen05/TMA/mbarrier instruction."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
for r in rows[hi + 1:]:
    try:
        data.append((r[0], r[1].strip(), float(r[ss] or 0), float(r[ie] or 0),
                     {k: float(r[h.index(k)] or 0) for k in stall_cols}))
    except (ValueError, IndexError):
        pass
tot = sum(d[2] for d in data) or 1
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
print(f"total samples {tot:.0f}")
for i, (a, src, smp, n, st) in enumerate(data):
    key = any(t in src for t in ("UTCHMMA", "UTCBAR", "UTMALDG", "LDTM", "SYNCS"))
    if key or smp > tot * thr:
        top = sorted(st.items(), key=lambda kv: -kv[1])[:2]
        tops = " ".join(f"{k[6:]}={v:.0f}" for k, v in top if v > 0)
        print(f"{i:5d} {100 * smp / tot:5.1f}% n={n:<10.0f} {src[:64]:64s} {tops}")
