"""Turn gpurun_out/ captures into the tracked profiles/ summaries.

Writes profiles/<tag>_launches_cfg3.csv (the ncu launch list of the bench
command), profiles/<tag>_ncu_<kernel>.txt (key metrics of each full capture)
and profiles/ncu_summary.json (per-launch DRAM bytes that bench.py reports as
roofline.traffic).
"""
import json
import shutil
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
OUT = REPO / "gpurun_out"
PROF = REPO / "profiles"
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
PROF.mkdir(exist_ok=True)

shutil.copy(OUT / "launches_cfg3.csv", PROF / f"{tag}_launches_cfg3.csv")
launch_txt = subprocess.run([sys.executable, str(REPO / "tools/ncu_launches.py"), str(OUT / "launches_cfg3.csv")],
                            capture_output=True, text=True).stdout
(PROF / f"{tag}_launches_cfg3_summary.txt").write_text(
    "# ncu --metrics gpu__time_duration,dram bytes,lts bytes --clock-control none; "
    "python bench.py --steps 2 --warmup 1 (cfg3); per-kernel means (cold-cache, serialised)\n" + launch_txt)

summary = {"fwd": {}, "bwd": {}}
for name in ("fwd", "de", "route", "dh"):
    rep = OUT / f"full_{name}.ncu-rep"
    if not rep.exists():
        continue
    txt = subprocess.run([sys.executable, str(REPO / "tools/ncu_summary.py"), str(rep)], capture_output=True,
                         text=True).stdout
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = raw.splitlines()
    import csv
    rows = list(csv.reader(lines))
    hdr, units, vals = rows[0], rows[1], rows[2]
    pick = {}
    for k, u, v in zip(hdr, units, vals):
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_bytes.sum",
                 "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                 "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
                 "gpc__cycles_elapsed.max"):
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(u, 1)
            pick[k] = x * scale
    (PROF / f"{tag}_ncu_{name}.txt").write_text(
        f"# ncu --set full --clock-control none, one launch of {name} at cfg3 (B=S=512, D=768, V=250002)\n"
        + txt + "\n" + "\n".join(f"  {k} = {v:.6g}" for k, v in pick.items()) + "\n")
    dram = pick.get("dram__bytes_read.sum", 0) + pick.get("dram__bytes_write.sum", 0)
    entry = {"dram_bytes": dram, "lts_bytes": pick.get("lts__t_bytes.sum"),
             "duration_s": pick.get("gpu__time_duration.sum"),
             "tensor_pipe_pct": pick.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")}
    if name == "fwd":
        summary["fwd"]["cfg3"] = entry
    else:
        summary["bwd"][name] = entry
(PROF / "ncu_summary.json").write_text(json.dumps(summary, indent=1) + "\n")
for f in ("bench_cfg3_full.txt", "bench_cfg2_full.txt", "bench_ref.txt"):
    if (OUT / f).exists():
        line = (OUT / f).read_text().strip().splitlines()[-1]
        (PROF / f"{tag}_{f.replace('.txt', '.json')}").write_text(line + "\n")
print(sorted(p.name for p in PROF.iterdir()))
