#!/usr/bin/env python
"""Benchmark of the B200 Sparton head: fused LM-head fwd+bwd at B=S=512, |V|=250002.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0.  A step = one forward (K1) + one backward (K2, K3a, K3b)
of the head over one synthetic batch (H ~ N(0,1), E ~ N(0, 0.02²), bias 0,
all-ones mask, dY ~ N(0,1) — every (b, v) pair active, the backward's worst
case).  Inputs (H 403 MB, E 384 MB, dY 512 MB) are larger than the 126 MB L2,
so no explicit flush is needed between steps.

* ``value``  — algorithmic TFLOP/s = (2·B·S·V·D + 4·B·V·D) / step time, whole job.
* ``e2e``    — same metric through the public torch API with pinned HOST
               buffers: H2D of the step's inputs and D2H of its outputs
               (Y, I, dH, dE, db) inside the timed region.
* ``roofline`` — the forward kernel (dominant): achieved TFLOP/s per launch
               from CUDA events around each launch vs MEASURED_PEAKS.json.
* ``cpu_baseline`` — the oracle port (oracle/, numpy + BLAS, all host threads)
               on a bounded B-slice of the same workload (N=1, rank 0 only).

``--impl reference`` times the reference's CPU algorithm (the oracle port — the
reference is pure Python/numpy and cannot travel to the GPU box) on the same
metric/unit, one bounded B-slice per step.

N > 1: the vocabulary is sharded over ranks (column-parallel head, strong
scaling of the same cfg3 workload): each rank runs K1 on its E/bias shard,
Y/I are all-gathered over NCCL, and the per-rank partial dH is all-reduced.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
CONFIGS = {
    "cfg2": dict(B=512, S=512, D=768, V=30522),
    "cfg3": dict(B=512, S=512, D=768, V=250002),
    "cfg4": dict(B=2048, S=512, D=1024, V=250002),
}
METRIC = "LM-head fwd+bwd ms, TFLOP/s vs bf16 peak, peak HBM at B=S=512, |V|=30522/250002"


def flops(c):
    return 2 * c["B"] * c["S"] * c["V"] * c["D"], 4 * c["B"] * c["V"] * c["D"]


DH_CHUNK_MB = 52   # csrc/sparton_bwd.cu DH_CHUNK_BYTES (tests/test_host.py keeps them equal)


def launches_per_step(c, v_local):
    """Kernels the library launches per step (fwd + bwd) on one rank:
    K1 + route + staged dE + db column sum + one dH launch per L2-sized
    vocabulary chunk (csrc/sparton_bwd.cu: RT_WIN = 8192 rows per route
    window, DH_CHUNK_BYTES of E per chunk)."""
    D = c["D"]
    nwin = -(-v_local // 8192)
    wpc = max(1, min(nwin, 32, (DH_CHUNK_MB << 20) // (8192 * D * 2)))
    return 1 + 1 + 1 + 1 + -(-nwin // wpc)


def measured_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"bf16_tflops": float(d["bf16_tflops"]), "bf16_tflops_sustained": float(d["bf16_tflops_sustained"]),
                "hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "source": "fallback"}


def ncu_traffic(config_name):
    """DRAM bytes per forward launch from the committed ncu capture, if any."""
    p = REPO / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get("fwd", {}).get(config_name, {}).get("dram_bytes")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/sparton_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        loaded = [x for x in sm if smax and x > 0.3 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU arms (oracle port)

def cpu_sample(c, seconds_hint=True):
    """Time the oracle port (fwd + bwd) on a bounded B-slice of the workload.

    Returns (TFLOP/s, sample description, threads).  Separable in b, so the
    slice's work is exactly B'/B of the full step."""
    import numpy as np
    sys.path.insert(0, str(REPO))
    from oracle import sparton_oracle as orc

    threads = os.cpu_count() or 1
    Bp = 1
    S, D, V = c["S"], c["D"], c["V"]
    rng = np.random.default_rng(0)
    H = orc.bf16_round(rng.standard_normal((Bp, S, D), dtype=np.float32))
    E = orc.bf16_round((rng.standard_normal((V, D), dtype=np.float32) * 0.02).astype(np.float32))
    b = np.zeros(V, np.float32)
    m = np.ones((Bp, S), np.uint8)
    dY = rng.standard_normal((Bp, V), dtype=np.float32)
    t0 = time.perf_counter()
    Y, I = orc.forward(H, E, b, m, vocab_tile=8192, threads=threads)
    orc.backward(H, E, b, Y, I, dY)
    dt = time.perf_counter() - t0
    ff, fb = flops(dict(B=Bp, S=S, D=D, V=V))
    return (ff + fb) / dt / 1e12, f"B'={Bp} of {c['B']} batch rows, S={S}, D={D}, V={V}, fwd+bwd", threads, dt


def run_reference_arm(args, c, cname):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_sample(c)
    vals = []
    t_all = []
    for _ in range(args.steps):
        v, sample, threads, dt = cpu_sample(c)
        vals.append(v)
        t_all.append(dt)
    value = statistics.median(vals)
    ff, fb = flops(c)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": (ff + fb) / (value * 1e12) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": cname, **c},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "sample_seconds_median": statistics.median(t_all),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm

def make_inputs(c, dev, rank, world):
    import torch
    gen = torch.Generator(device=dev).manual_seed(0)
    B, S, D, V = c["B"], c["S"], c["D"], c["V"]
    Vp = (V + world - 1) // world
    v0, v1 = rank * Vp, min(V, (rank + 1) * Vp)
    H = torch.randn((B, S, D), generator=gen, device=dev).to(torch.bfloat16)
    E_full_rows = torch.empty((v1 - v0, D), device=dev, dtype=torch.bfloat16)
    # Same E for every world size: rows are generated per global row block.
    g2 = torch.Generator(device=dev).manual_seed(1)
    blk = 8192
    for r0 in range(0, V, blk):
        r1 = min(V, r0 + blk)
        x = (torch.randn((r1 - r0, D), generator=g2, device=dev) * 0.02).to(torch.bfloat16)
        lo, hi = max(r0, v0), min(r1, v1)
        if lo < hi:
            E_full_rows[lo - v0:hi - v0] = x[lo - r0:hi - r0]
    bias = torch.zeros(v1 - v0, device=dev)
    mask = torch.ones((B, S), dtype=torch.uint8, device=dev)
    g3 = torch.Generator(device=dev).manual_seed(2)
    dY = torch.randn((B, V), generator=g3, device=dev)
    return H, E_full_rows, bias, mask, dY, (v0, v1, Vp)


def run_gpu_arm(args, c, cname):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(REPO))
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    from paper_2603_25011_b200 import sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    B, S, D, V = c["B"], c["S"], c["D"], c["V"]
    H, E, bias, mask, dY, (v0, v1, Vp) = make_inputs(c, dev, rank, world)
    stream = torch.cuda.current_stream()

    fwd_ev = []

    def step(timed=False):
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        if world == 1:
            Y, I = sparton_forward(H, E, bias, mask)
        else:
            Y, I = sharded.local_forward(H, E, bias, mask)
        if timed:
            e1.record(stream)
            fwd_ev.append((e0, e1))
        if world == 1:
            dH, dE, db = sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
        else:
            Yg, Ig = sharded.gather_vocab(Y, I, V, Vp)
            dH, dE, db = sharded.local_backward(H, E, Y, I, dY[:, v0:v1], grad_dtype=torch.bfloat16)
        return Y, I, dH, dE, db

    for _ in range(args.warmup):
        out = step()
        del out
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    base_alloc = torch.cuda.memory_allocated(dev)
    clk = ClockSampler(local)
    clk.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        out = step(timed=True)
        del out
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = t0.elapsed_time(t1) / args.steps
    peak_bytes = torch.cuda.max_memory_allocated(dev)
    fwd_ms = statistics.mean(a.elapsed_time(b) for a, b in fwd_ev)
    if world > 1:
        t = torch.tensor([ms, fwd_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, fwd_ms = float(t[0]), float(t[1])
    ff, fb = flops(c)
    value = (ff + fb) / (ms * 1e-3) / 1e12

    # ---- end-to-end through the public API with pinned host buffers (N=1 only).
    e2e = None
    if world == 1:
        e2e = run_e2e(args, c, H, E, bias, mask, dY)

    peaks = measured_peaks()
    fwd_flops_rank = 2 * B * S * (v1 - v0) * D
    achieved = fwd_flops_rank / (fwd_ms * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (H~N(0,1), E~N(0,0.02^2), bias 0, all-ones mask, dY~N(0,1))",
        "config": {"workload": cname, **c, "parallelism": f"vocab-shard{world}" if world > 1 else "single",
                   "l2_flush": "inputs larger than L2 (H 403 MB, E 384 MB, dY 512 MB)"},
        "fwd_ms": fwd_ms, "bwd_ms": ms - fwd_ms,
        "pct_of_bf16_peak": value / peaks["bf16_tflops"],
        "pct_of_bf16_peak_sustained": value / peaks["bf16_tflops_sustained"],
        "peak_hbm_bytes": peak_bytes, "head_owned_peak_bytes": peak_bytes - base_alloc,
        "roofline": {"kernel": "sparton_fwd_kernel<2>", "bound": "tensor", "achieved": achieved,
                     "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                     "frac": achieved / peaks["bf16_tflops_sustained"],
                     "frac_of_burst": achieved / peaks["bf16_tflops"],
                     "traffic": ncu_traffic(cname), "algorithmic_flops_per_launch": fwd_flops_rank,
                     "peak_source": peaks["source"] + " (sustained: K1 runs inside a long step; burst in "
                                    "frac_of_burst. frac > 1 means the step's lighter backward phase lets the "
                                    "forward hold higher clocks than a back-to-back cuBLAS loop at the power cap)"},
        "gpu_launches": launches_per_step(c, v1 - v0) * args.steps,
        "clocks": clocks,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu:
        v, sample, threads, dt = cpu_sample(c)
        line["cpu_baseline"] = {"value": v, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                                "sample": sample + f" ({dt:.1f} s)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(args, c, H, E, bias, mask, dY):
    """Public API end to end: pinned host inputs -> H2D -> fwd+bwd -> D2H outputs.

    Every step copies its inputs (H, E, bias, mask, dY) from pinned host memory
    and copies all outputs (Y, I, dH, dE, db) back.  As a training input
    pipeline would, copies run on side streams: step i+1's inputs stream in
    (double-buffered device buffers) while step i computes, dY arrives during
    the forward and (Y, I) stream out during the backward."""
    import torch
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    dev = H.device
    hH = H.cpu().pin_memory()
    hE = E.cpu().pin_memory()
    hb = bias.cpu().pin_memory()
    hm = mask.cpu().pin_memory()
    hdY = dY.cpu().pin_memory()
    B, S, D, V = c["B"], c["S"], c["D"], c["V"]
    oY = torch.empty((B, V), dtype=torch.float32).pin_memory()
    oI = torch.empty((B, V), dtype=torch.int32).pin_memory()
    odH = torch.empty((B, S, D), dtype=torch.bfloat16).pin_memory()
    odE = torch.empty((V, D), dtype=torch.bfloat16).pin_memory()
    odb = torch.empty((V,), dtype=torch.float32).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in (hH, hE, hb, hm, hdY))
    d2h = sum(t.numel() * t.element_size() for t in (oY, oI, odH, odE, odb))
    bufs = [[torch.empty_like(t, device=dev) for t in (hH, hE, hb, hm, hdY)] for _ in range(2)]
    comp = torch.cuda.current_stream()
    s_in = torch.cuda.Stream(device=dev)
    s_out = torch.cuda.Stream(device=dev)
    freed = [None, None]

    def step(i):
        k = i % 2
        dH_, dE_, db_, dm_, ddY = bufs[k]
        with torch.cuda.stream(s_in):
            if freed[k] is not None:
                s_in.wait_event(freed[k])
            for dst, src in ((dH_, hH), (dE_, hE), (db_, hb), (dm_, hm)):
                dst.copy_(src, non_blocking=True)
            ev_x = torch.cuda.Event()
            ev_x.record(s_in)
            ddY.copy_(hdY, non_blocking=True)
            ev_dy = torch.cuda.Event()
            ev_dy.record(s_in)
        comp.wait_event(ev_x)
        Y, I = sparton_forward(dH_, dE_, db_, dm_)
        ev_f = torch.cuda.Event()
        ev_f.record(comp)
        comp.wait_event(ev_dy)
        gH, gE, gb = sparton_backward(dH_, dE_, Y, I, ddY, grad_dtype=torch.bfloat16)
        ev_b = torch.cuda.Event()
        ev_b.record(comp)
        freed[k] = ev_b
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_f)
            oY.copy_(Y, non_blocking=True)
            oI.copy_(I, non_blocking=True)
            s_out.wait_event(ev_b)
            odH.copy_(gH, non_blocking=True)
            odE.copy_(gE, non_blocking=True)
            odb.copy_(gb, non_blocking=True)
            for t in (Y, I, gH, gE, gb):
                t.record_stream(s_out)

    for i in range(max(1, min(args.warmup, 2))):
        step(i)
    torch.cuda.synchronize()
    n = max(2, min(args.steps, 6))
    t0 = time.perf_counter()
    for i in range(n):
        step(i)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / n
    ff, fb = flops(c)
    return {"value": (ff + fb) / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": n,
            "note": "pinned host buffers; H2D/D2H on side streams overlapped with compute, "
                    "double-buffered device inputs; timed by host wall clock across all streams"}


def main() -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg3")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, c, args.config)
    return run_gpu_arm(args, c, args.config)


if __name__ == "__main__":
    raise SystemExit(main())
