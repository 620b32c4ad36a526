#!/usr/bin/env python
"""Benchmark of the B200 Sparton head: fused LM-head fwd+bwd at B=S=512, |V|=250002.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints ONE
JSON line on rank 0.  A step = one forward (K1) + one backward (K3a route, K2s
staged dE + db, K3b dH passes) of the head over one synthetic batch (H ~ N(0,1),
E ~ N(0, 0.02²), bias 0, all-ones mask, dY ~ N(0,1) — every (b, v) pair
active, the backward's worst case).  Inputs (H 403 MB, E 384 MB, dY 512 MB)
are larger than the 126 MB L2, so no explicit flush is needed between steps.

* ``value``  — algorithmic TFLOP/s = (2·B·S·V·D + 4·B·V·D) / step time, whole job.
* ``e2e``    — same metric through the public torch API with pinned HOST
               buffers: H2D of the step's inputs and D2H of its outputs
               (Y, I, dH, dE, db) inside the timed region, K steps.
* ``e2e_plugin`` — the reference-facing numpy drop-in
               (``fusedhead.forward_fully_fused`` + ``backward_fused``, numpy in
               and out, synchronous) on the same workload.
* ``roofline`` — the forward kernel (dominant): achieved TFLOP/s per launch
               from CUDA events around each launch vs MEASURED_PEAKS.json.
* ``cpu_baseline`` — the reference's own CPU path on a bounded B-slice.

``--impl reference`` times the UNMODIFIED reference (installed under
baseline/_ref: ``forward_hybrid`` + ``backward_fused`` with
``TileConfig.default_for(dims, num_threads=nproc)``, OPENBLAS_NUM_THREADS=1,
SURVEY.md §8d) on one batch row of the cfg3 workload per step; the head is
separable in b, so B'=1 is exactly 1/B of a step ("extrapolated_from_rows").
Falls back to the oracle port (oracle/, kind "port") without the install.

N > 1: the vocabulary is sharded over ranks (column-parallel head, strong
scaling of the same cfg3 workload): each rank runs K1 on its E/bias shard,
Y/I are all-gathered over NCCL, and the per-rank partial dH is all-reduced on
a communication stream overlapping the shard's dE.  The line adds a ``cfg4``
record (B=2048, D=1024, V=250002 sharded; BASELINE configs[3]).
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
CONFIGS = {
    "cfg1": dict(B=8, S=128, D=768, V=30522),
    "cfg2": dict(B=512, S=512, D=768, V=30522),
    "cfg3": dict(B=512, S=512, D=768, V=250002),
    "cfg4": dict(B=2048, S=512, D=1024, V=250002),
}
METRIC = "LM-head fwd+bwd ms, TFLOP/s vs bf16 peak, peak HBM at B=S=512, |V|=30522/250002"
DATA = "synthetic (H~N(0,1), E~N(0,0.02^2), bias 0, all-ones mask, dY~N(0,1))"


def flops(c):
    return 2 * c["B"] * c["S"] * c["V"] * c["D"], 4 * c["B"] * c["V"] * c["D"]


def config_dict(cname, c, world):
    h, e, dy = c["B"] * c["S"] * c["D"] * 2, c["V"] * c["D"] * 2, c["B"] * c["V"] * 4
    sizes = "H %d MiB, E %d MiB, dY %d MiB" % (h >> 20, e >> 20, dy >> 20)
    l2 = ("inputs larger than L2 (%s)" % sizes if h + e + dy > (126 << 20)
          else "no flush: inputs fit in L2 (%s), warm-cache steps" % sizes)
    return {"workload": cname, **c, "parallelism": f"vocab-shard{world}" if world > 1 else "single",
            "l2_flush": l2}


SPARSE_BIAS = -2.0   # SURVEY §8d "SPLADE-sparse" variant
DH_CHUNK_MB = 52   # csrc/sparton_bwd.cu DH_CHUNK_BYTES (tests/test_host.py keeps them equal)


def launches_per_step(c, v_local):
    """Kernels the library launches per step (fwd + bwd) on one rank:
    K1 + route + staged dE + db column sum + sparse dE + single-pass dH + one
    dH launch per L2-sized vocabulary chunk (csrc/sparton_bwd.cu: RT_WIN =
    8192 rows per route window, DH_CHUNK_BYTES of E per chunk).  The
    sparse-regime pair (and, in that regime, the staged dE, db and dense dH
    launches) exit on their first instruction after reading the route's
    active-pair count; all are launched."""
    D = c["D"]
    nwin = -(-v_local // 8192)
    wpc = max(1, min(nwin, 32, (DH_CHUNK_MB << 20) // (8192 * D * 2)))
    return 1 + 1 + 1 + 1 + 2 + -(-nwin // wpc)


def measured_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"bf16_tflops": float(d["bf16_tflops"]), "bf16_tflops_sustained": float(d["bf16_tflops_sustained"]),
                "hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "source": "fallback"}


def ncu_fwd(config_name, key="dram_bytes"):
    """A per-launch figure of the forward from the committed ncu capture
    (profiles/ncu_summary.json, tools/make_profiles.py), if any."""
    p = REPO / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get("fwd", {}).get(config_name, {}).get(key)
    except Exception:
        return None


def host_cpu() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


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
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
                power.append(float(parts[3]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        loaded = [x for x in sm if smax and x > 0.3 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(power) if power else None}


# ---------------------------------------------------------------- CPU arms

def _slice_inputs(c, Bp, seed=0):
    """One bounded B-slice of the workload with the GPU arm's distributions (fp32)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    S, D, V = c["S"], c["D"], c["V"]
    H = rng.standard_normal((Bp, S, D), dtype=np.float32)
    E = (rng.standard_normal((V, D), dtype=np.float32) * np.float32(0.02)).astype(np.float32)
    b = np.zeros(V, np.float32)
    m = np.ones((Bp, S), np.uint8)
    dY = rng.standard_normal((Bp, V), dtype=np.float32)
    return H, E, b, m, dY


def _reference_module():
    ref_dir = REPO / "baseline" / "_ref"
    if ref_dir.is_dir() and str(ref_dir) not in sys.path:
        sys.path.append(str(ref_dir))
    try:
        import fusedhead
        return fusedhead
    except ImportError:
        return None


class CpuArm:
    """The reference's CPU path on one batch row (B'=1) of the workload.

    kind "reference": the stock reference from baseline/_ref —
    ``forward_hybrid(inputs, TileConfig.default_for(dims, num_threads=nproc))``
    then ``backward_fused`` (its fastest strategy), BLAS
    single-threaded so the tile pool owns the cores.  kind "port": the oracle
    restatement (oracle/) when the install is absent."""

    def __init__(self, c):
        self.c = c
        self.Bp = 1
        self.threads = os.cpu_count() or 1
        self.ref = _reference_module()
        self.kind = "reference" if self.ref is not None else "port"
        H, E, b, m, dY = _slice_inputs(c, self.Bp)
        if self.ref is not None:
            fh = self.ref
            dims = fh.Dims(self.Bp, c["S"], c["D"], c["V"])
            self.inputs = fh.HeadInputs(dims=dims, H=H, E=E, b=b, mask=m)
            self.cfg = fh.TileConfig.default_for(dims, num_threads=self.threads)
        else:
            self.arrays = (H, E, b, m)
        self.dY = dY

    def sample(self) -> float:
        """Seconds for one fwd+bwd of the B'-row slice."""
        t0 = time.perf_counter()
        if self.ref is not None:
            fh = self.ref
            out = fh.forward_hybrid(self.inputs, self.cfg)
            fh.backward_fused(self.inputs, fh.SavedSparseState.from_output(out), self.dY, self.cfg)
        else:
            sys.path.insert(0, str(REPO))
            from oracle import sparton_oracle as orc
            H, E, b, m = self.arrays
            Y, I = orc.forward(H, E, b, m, vocab_tile=8192, threads=self.threads)
            orc.backward(H, E, b, Y, I, self.dY)
        return time.perf_counter() - t0

    def tflops(self, seconds: float) -> float:
        ff, fb = flops(dict(self.c, B=self.Bp))
        return (ff + fb) / seconds / 1e12

    def describe(self, seconds: float) -> dict:
        what = ("stock reference forward_hybrid + backward_fused (baseline/_ref), "
                f"TileConfig.default_for(num_threads={self.threads}), OPENBLAS_NUM_THREADS="
                f"{os.environ.get('OPENBLAS_NUM_THREADS', 'default')}"
                if self.kind == "reference" else "oracle port (oracle/sparton_oracle.py) forward + backward")
        return {"value": self.tflops(seconds), "unit": "TFLOP/s", "cores": self.threads, "kind": self.kind,
                "sample": f"B'={self.Bp} of {self.c['B']} batch rows, S={self.c['S']}, D={self.c['D']}, "
                          f"V={self.c['V']}, fwd+bwd ({seconds:.1f} s): {what}",
                "extrapolated_from_rows": self.Bp, "host_cpu": host_cpu()}


def run_reference_arm(args, c, cname):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    arm = CpuArm(c)
    for _ in range(min(args.warmup, 1)):
        arm.sample()
    ts = [arm.sample() for _ in range(args.steps)]
    t = statistics.median(ts)
    value = arm.tflops(t)
    ff, fb = flops(c)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": (ff + fb) / (value * 1e12) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": DATA.replace("synthetic", "synthetic, numpy"), "config": config_dict(cname, c, args.gpus),
        "extrapolated_from_rows": arm.Bp,
        "note": (f"each step times one batch row (B'={arm.Bp}) of the {cname} workload on the host CPU; "
                 f"ms_per_step = that time x {c['B']} rows (the head is separable in b: per-row work is "
                 "independent, fused.py:91-95,257,267-277)"),
        "cpu_baseline": arm.describe(t),
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "sample_seconds_median": t,
    }
    if cname != "cfg1" and not args.no_cfg1 and arm.kind == "reference":
        line["cfg1"] = reference_cfg1(arm.threads)
    print(json.dumps(line), flush=True)
    return 0


def reference_cfg1(threads, steps=2):
    """BASELINE configs[0], the reference's own CPU case, timed in FULL (no
    extrapolation): the stock forward_hybrid + backward_fused on the
    reference's exact cfg1 inputs (HeadInputs.seeded(Dims(8,128,768,30522),
    0, mask_keep=0.85), dY = seeded_tensor((B, V), 9))."""
    fh = _reference_module()
    dims = fh.Dims(8, 128, 768, 30522)
    inputs = fh.HeadInputs.seeded(dims, 0, mask_keep=0.85)
    dY = fh.seeded_tensor((dims.B, dims.V), 9)
    cfg = fh.TileConfig.default_for(dims, num_threads=threads)
    ts = []
    for _ in range(steps + 1):
        t0 = time.perf_counter()
        out = fh.forward_hybrid(inputs, cfg)
        fh.backward_fused(inputs, fh.SavedSparseState.from_output(out), dY, cfg)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts[1:])
    ff, fb = flops(CONFIGS["cfg1"])
    return {"config": config_dict("cfg1", CONFIGS["cfg1"], 1), "ms_per_step": t * 1e3,
            "value": (ff + fb) / t / 1e12, "unit": "TFLOP/s", "steps": steps, "cores": threads,
            "note": "stock reference forward_hybrid + backward_fused at cfg1 in full (f32), no extrapolation"}


# ---------------------------------------------------------------- GPU arm

def make_inputs(c, dev, rank, world, bias_value=0.0):
    import torch
    gen = torch.Generator(device=dev).manual_seed(0)
    B, S, D, V = c["B"], c["S"], c["D"], c["V"]
    Vp = (V + world - 1) // world
    v0, v1 = min(V, rank * Vp), min(V, (rank + 1) * Vp)
    H = torch.randn((B, S, D), generator=gen, device=dev).to(torch.bfloat16)
    E_rows = torch.empty((v1 - v0, D), device=dev, dtype=torch.bfloat16)
    # Same E for every world size: rows are generated per global row block.
    g2 = torch.Generator(device=dev).manual_seed(1)
    blk = 8192
    for r0 in range(0, V, blk):
        r1 = min(V, r0 + blk)
        x = (torch.randn((r1 - r0, D), generator=g2, device=dev) * 0.02).to(torch.bfloat16)
        lo, hi = max(r0, v0), min(r1, v1)
        if lo < hi:
            E_rows[lo - v0:hi - v0] = x[lo - r0:hi - r0]
    bias = torch.full((v1 - v0,), float(bias_value), device=dev)
    mask = torch.ones((B, S), dtype=torch.uint8, device=dev)
    g3 = torch.Generator(device=dev).manual_seed(2)
    dY = torch.randn((B, V), generator=g3, device=dev)
    return H, E_rows, bias, mask, dY, (v0, v1, Vp)


def _max_over_ranks(vals, world, dev):
    import torch
    import torch.distributed as dist
    if world == 1:
        return vals
    on = dev if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, device=on, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t]


def timed_steps(c, dev, rank, world, steps, warmup, fwd_ev=None, fused=False, bias_value=0.0):
    """Warm up, then time `steps` fwd+bwd steps between barriers; returns
    (ms per step, mean forward ms, peak bytes, head-owned peak bytes, inputs).
    ``fused``: N > 1 with the (Y, I) all-gather fused into K1's epilogue
    (sharded.FusedVocabGather) instead of NCCL all-gather + permute copy:
    "p2p" stores to every peer's buffer, "nvls" one multimem store per result
    through the multicast mapping; the partial dH is then summed by one kernel
    over peer memory (sharded.PeerDHReduce: P2P loads/stores, or multimem)."""
    import torch
    import torch.distributed as dist
    from paper_2603_25011_b200 import sharded, sparton_backward, sparton_forward

    V = c["V"]
    H, E, bias, mask, dY, (v0, v1, Vp) = make_inputs(c, dev, rank, world, bias_value)
    stream = torch.cuda.current_stream()
    fwd_ev = [] if fwd_ev is None else fwd_ev
    fg = sharded.FusedVocabGather.symmetric(c["B"], V, dev, multicast=(fused == "nvls")) if fused else None
    # The fused runs also reduce dH in one kernel over peer memory (P2P loads
    # and stores, or multimem.ld_reduce / multimem.st) instead of NCCL.
    dr = (sharded.PeerDHReduce.symmetric((c["B"], c["S"], c["D"]), torch.bfloat16, dev,
                                         multicast=(fused == "nvls")) if fused else None)

    def step(timed=False):
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        if fg is not None:
            Yg, Ig = fg.forward(H, E, bias, mask, v0)
            Y, I = Yg[:, v0:v1], Ig[:, v0:v1]
        else:
            Y, I = sparton_forward(H, E, bias, mask)
        if timed:
            e1.record(stream)
            fwd_ev.append((e0, e1))
        if world == 1:
            g = sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
        else:
            if fg is None:
                Yg, Ig = sharded.gather_vocab(Y, I, V, Vp)
            g = sharded.local_backward(H, E, Y, I, dY[:, v0:v1], grad_dtype=torch.bfloat16, dh_reduce=dr)
        return Y, I, g

    for _ in range(warmup):
        out = step()
        del out
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    base_alloc = torch.cuda.memory_allocated(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        out = step(timed=True)
        del out
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1) / steps
    fwd_ms = statistics.mean(a.elapsed_time(b) for a, b in fwd_ev)
    peak = torch.cuda.max_memory_allocated(dev)
    ms, fwd_ms = _max_over_ranks([ms, fwd_ms], world, dev)
    inputs = (H, E, bias, mask, dY, (v0, v1, Vp))
    return ms, fwd_ms, peak, peak - base_alloc, inputs


def run_gpu_arm(args, c, cname):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, str(REPO))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Test-only overrides (tests/test_gpu_bench_multi.py runs the N=2 path on
    # one GPU): every rank on one device, gloo instead of NCCL.
    if os.environ.get("SPARTON_BENCH_DEVICE") is not None:
        local = int(os.environ["SPARTON_BENCH_DEVICE"])
    backend = os.environ.get("SPARTON_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    B, S, D, V = c["B"], c["S"], c["D"], c["V"]

    clk = ClockSampler(local)
    clk.start()
    fwd_ev = []
    ms, fwd_ms, peak_bytes, head_peak, inputs = timed_steps(c, dev, rank, world, args.steps, args.warmup, fwd_ev)
    clocks = clk.stop()
    H, E, bias, mask, dY, (v0, v1, Vp) = inputs
    ff, fb = flops(c)
    value = (ff + fb) / (ms * 1e-3) / 1e12

    peaks = measured_peaks()
    fwd_flops_rank = 2 * B * S * (v1 - v0) * D
    achieved = fwd_flops_rank / (fwd_ms * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": DATA,
        "config": config_dict(cname, c, world),
        "fwd_ms": fwd_ms, "bwd_ms": ms - fwd_ms,
        "pct_of_bf16_peak": value / peaks["bf16_tflops"],
        "pct_of_bf16_peak_sustained": value / peaks["bf16_tflops_sustained"],
        "peak_hbm_bytes": peak_bytes, "head_owned_peak_bytes": head_peak,
        "roofline": {"kernel": "sparton_fwd_kernel<2>", "bound": "tensor", "achieved": achieved,
                     "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                     "frac": achieved / peaks["bf16_tflops_sustained"],
                     "frac_of_burst": achieved / peaks["bf16_tflops"],
                     "traffic": ncu_fwd(cname), "algorithmic_flops_per_launch": fwd_flops_rank,
                     "ncu_tensor_pipe_pct": ncu_fwd(cname, "tensor_pipe_pct"),
                     "peak_source": peaks["source"] + " (sustained: K1 runs inside a long step; burst in "
                                    "frac_of_burst. frac > 1 means the step's lighter backward phase lets the "
                                    "forward hold higher clocks than a back-to-back cuBLAS loop at the power cap)"},
        "gpu_launches": launches_per_step(c, v1 - v0) * args.steps * world,
        "clocks": clocks,
    }
    del H, E, bias, mask, dY, inputs
    torch.cuda.empty_cache()

    # ---- end-to-end through the public API with pinned host buffers.
    e2e = run_e2e(args, c, dev, rank, world)
    if e2e is not None:
        line["e2e"] = e2e
    if world == 1 and not args.no_plugin:
        line["e2e_plugin"] = run_plugin_e2e(c, dev)
    if world > 1 and not args.no_fused_ab:
        # A/B of the NVLink-fused (Y, I) all-gather on the
        # same workload; the headline keeps the NCCL path.
        try:
            msf, fwdf, _, _, inpf = timed_steps(c, dev, rank, world, args.steps, args.warmup, fused="p2p")
            del inpf
            line["fused_gather"] = {"ms_per_step": msf, "fwd_ms": fwdf, "value": (ff + fb) / (msf * 1e-3) / 1e12,
                                    "unit": "TFLOP/s", "note": "K1 epilogue stores into every rank's symmetric "
                                    "[B, V] buffers (sparton_fwd_multi) instead of NCCL all-gather; dH "
                                    "summed by sparton_allreduce_peers (P2P) instead of NCCL"}
        except Exception as exc:
            line["fused_gather"] = {"unavailable": repr(exc)[:300]}
        torch.cuda.empty_cache()
        try:
            msn, fwdn, _, _, inpn = timed_steps(c, dev, rank, world, args.steps, args.warmup, fused="nvls")
            del inpn
            line["nvls_gather"] = {"ms_per_step": msn, "fwd_ms": fwdn, "value": (ff + fb) / (msn * 1e-3) / 1e12,
                                   "unit": "TFLOP/s", "note": "K1 epilogue stores each result once with "
                                   "multimem.st to the symmetric buffers' NVLS multicast mapping "
                                   "(sparton_fwd_multicast); dH summed by multimem.ld_reduce + "
                                   "multimem.st (sparton_allreduce_multimem)"}
        except Exception as exc:
            line["nvls_gather"] = {"unavailable": repr(exc)[:300]}
        torch.cuda.empty_cache()
    if world == 1 and not args.no_sparse:
        # SURVEY §8d secondary run: the SPLADE-sparse variant (bias -2: a few %
        # of the (b, v) pairs active, as in trained SPLADE heads), where the
        # backward takes its sparse-regime kernels.
        sev = []
        mss, fws, _, _, inps = timed_steps(c, dev, rank, world, args.steps, args.warmup, sev, bias_value=SPARSE_BIAS)
        Hs, Es, bs, ms_, _, _ = inps
        from paper_2603_25011_b200 import sparton_forward
        Ys, _ = sparton_forward(Hs, Es, bs, ms_)
        act = float((Ys > 0).float().mean())
        del inps, Hs, Es, bs, ms_, Ys
        torch.cuda.empty_cache()
        line["splade_sparse"] = {"bias": SPARSE_BIAS, "active_pair_fraction": act, "ms_per_step": mss,
                                 "fwd_ms": fws, "bwd_ms": mss - fws, "steps": args.steps,
                                 "value": (ff + fb) / (mss * 1e-3) / 1e12, "unit": "TFLOP/s",
                                 "note": "same workload with bias -2 (few % active pairs): the backward "
                                         "runs its sparse-regime kernels (per-pair dE gathers, single-pass dH)"}
    if world > 1 and not args.no_cfg4:
        c4 = CONFIGS["cfg4"]
        ms4, fwd4, peak4, _, inp4 = timed_steps(c4, dev, rank, world, args.steps, args.warmup)
        del inp4
        torch.cuda.empty_cache()
        f4, b4 = flops(c4)
        line["cfg4"] = {"config": config_dict("cfg4", c4, world), "ms_per_step": ms4, "fwd_ms": fwd4,
                        "value": (f4 + b4) / (ms4 * 1e-3) / 1e12, "unit": "TFLOP/s", "steps": args.steps,
                        "peak_hbm_bytes": peak4,
                        "gpu_launches": launches_per_step(c4, -(-c4["V"] // world)) * args.steps * world}
    if world == 1 and cname != "cfg1" and not args.no_cfg1:
        line["cfg1"] = gpu_cfg1(dev, args.steps, args.warmup)
    if world == 1 and not args.no_naive:
        line["naive_pytorch"] = naive_pytorch(c, dev)
    if rank == 0 and world == 1 and not args.no_cpu:
        arm = CpuArm(c)
        line["cpu_baseline"] = arm.describe(arm.sample())
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def naive_pytorch(c, dev, steps=2):
    """The naive PyTorch GPU head on the same box (north_star):
    ``((H @ E.T + b) * M).relu().log1p().max(dim=1)`` with autograd, bf16,
    fwd + bwd per step, CUDA events.  It materialises the B×S×V logits, so at
    cfg3 it runs out of the 180 GB: the record keeps the OOM and times the
    largest batch (halving B) that fits, with the same algorithmic-FLOP
    accounting as the fused head."""
    import torch

    def step(H, E, b, m, dY):
        Hq, Eq, bq = (t.detach().requires_grad_(True) for t in (H, E, b))
        L = (torch.einsum("bsd,vd->bsv", Hq, Eq) + bq.to(Hq.dtype)) * m[..., None].to(Hq.dtype)
        Y = L.relu().log1p().max(dim=1).values.float()
        Y.backward(dY)

    rec = {"formula": "((H@E.T + b) * M).relu().log1p().max(dim=1), torch autograd, bf16", "oom_at_B": []}
    B = c["B"]
    while B >= 1:
        cb = dict(c, B=B)
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats(dev)
        base = torch.cuda.memory_allocated(dev)
        try:
            H, E, b, m, dY, _ = make_inputs(cb, dev, 0, 1)
            step(H, E, b, m, dY)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                step(H, E, b, m, dY)
            e1.record()
            torch.cuda.synchronize()
        except torch.OutOfMemoryError:
            rec["oom_at_B"].append(B)
            H = E = b = m = dY = None
            B //= 2
            continue
        ms = e0.elapsed_time(e1) / steps
        ff, fb = flops(cb)
        rec.update({"B": B, "ms_per_step": ms, "value": (ff + fb) / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                    "steps": steps, "peak_hbm_bytes": torch.cuda.max_memory_allocated(dev) - base})
        del H, E, b, m, dY
        break
    torch.cuda.empty_cache()
    return rec


def gpu_cfg1(dev, steps, warmup):
    """BASELINE configs[0] (B=8, S=128, D=768, V=30522) on the GPU beside the
    reference arm's full cfg1 record: the bf16 path and the fp32-accuracy path
    (the reference's dtype contract), fwd + bwd per step, CUDA events."""
    import torch
    from paper_2603_25011_b200 import (sparton_backward, sparton_backward_fp32, sparton_forward,
                                       sparton_forward_fp32)
    c = CONFIGS["cfg1"]
    B, S, D, V = c["B"], c["S"], c["D"], c["V"]
    g = torch.Generator(device=dev).manual_seed(0)
    H = torch.rand((B, S, D), generator=g, device=dev) * 2 - 1
    E = torch.rand((V, D), generator=g, device=dev) * 2 - 1
    b = torch.rand(V, generator=g, device=dev) * 2 - 1
    m = (torch.rand((B, S), generator=g, device=dev) < 0.85).to(torch.uint8)
    dY = torch.rand((B, V), generator=g, device=dev) * 2 - 1
    Hb, Eb = H.to(torch.bfloat16), E.to(torch.bfloat16)
    runs = {"bf16": lambda: sparton_backward(Hb, Eb, *sparton_forward(Hb, Eb, b, m), dY),
            "fp32_accuracy": lambda: sparton_backward_fp32(H, E, *sparton_forward_fp32(H, E, b, m), dY)}
    ff, fb = flops(c)
    rec = {"config": config_dict("cfg1", c, 1), "steps": steps, "unit": "TFLOP/s"}
    for name, fn in runs.items():
        for _ in range(max(3, warmup)):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        rec[name] = {"ms_per_step": ms, "value": (ff + fb) / (ms * 1e-3) / 1e12}
    # The bf16 step captured once in a CUDA graph and replayed: at this size the
    # step is launch-bound, and graph replay removes the per-launch host work.
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        runs["bf16"]()
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        runs["bf16"]()
    for _ in range(max(3, warmup)):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    rec["bf16_cuda_graph"] = {"ms_per_step": ms, "value": (ff + fb) / (ms * 1e-3) / 1e12}
    return rec


def run_e2e(args, c, dev, rank, world):
    """Public API end to end: pinned host inputs -> H2D -> fwd+bwd -> D2H outputs.

    Every step copies its inputs (H, E shard, bias shard, mask, dY) from pinned
    host memory and copies its outputs back (Y, I — the full gathered [B, V]
    on rank 0 of a sharded run —, dH, and this rank's dE, db).  As a training
    input pipeline would, copies run on side streams: step i+1's inputs stream
    in (double-buffered device buffers) while step i computes, dY arrives
    during the forward and (Y, I) stream out during the backward.  Timed by
    host wall clock across all streams over K steps (max over ranks)."""
    import torch
    import torch.distributed as dist
    from paper_2603_25011_b200 import sharded, sparton_backward, sparton_forward
    H, E, bias, mask, dY, (v0, v1, Vp) = make_inputs(c, dev, rank, world)
    B, S, D, V = c["B"], c["S"], c["D"], c["V"]
    hH, hE, hb, hm, hdY = (t.cpu().pin_memory() for t in (H, E, bias, mask, dY))
    del H, E, bias, mask, dY
    out_Y = rank == 0 or world == 1
    oY = torch.empty((B, V), dtype=torch.float32).pin_memory() if out_Y else None
    oI = torch.empty((B, V), dtype=torch.int32).pin_memory() if out_Y else None
    odH = torch.empty((B, S, D), dtype=torch.bfloat16).pin_memory()
    odE = torch.empty((v1 - v0, D), dtype=torch.bfloat16).pin_memory()
    odb = torch.empty((v1 - v0,), dtype=torch.float32).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in (hH, hE, hb, hm, hdY))
    d2h = sum(t.numel() * t.element_size() for t in (oY, oI, odH, odE, odb) if t is not None)
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
        if world > 1:
            Yo, Io = sharded.gather_vocab(Y, I, V, Vp)
        else:
            Yo, Io = Y, I
        ev_f = torch.cuda.Event()
        ev_f.record(comp)
        comp.wait_event(ev_dy)
        if world == 1:
            gH, gE, gb = sparton_backward(dH_, dE_, Y, I, ddY, grad_dtype=torch.bfloat16)
        else:
            gH, gE, gb = sharded.local_backward(dH_, dE_, Y, I, ddY[:, v0:v1], grad_dtype=torch.bfloat16)
        ev_b = torch.cuda.Event()
        ev_b.record(comp)
        freed[k] = ev_b
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_f)
            if out_Y:
                oY.copy_(Yo, non_blocking=True)
                oI.copy_(Io, non_blocking=True)
            s_out.wait_event(ev_b)
            odH.copy_(gH, non_blocking=True)
            odE.copy_(gE, non_blocking=True)
            odb.copy_(gb, non_blocking=True)
            for t in (Yo, Io, gH, gE, gb):
                t.record_stream(s_out)

    for i in range(max(1, min(args.warmup, 2))):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n = max(2, args.steps)
    t0 = time.perf_counter()
    for i in range(n):
        step(i)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / n
    ms = _max_over_ranks([ms], world, dev)[0]
    ff, fb = flops(c)
    return {"value": (ff + fb) / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": n,
            "note": "pinned host buffers; H2D/D2H on side streams overlapped with compute, double-buffered "
                    "device inputs; timed by host wall clock across all streams (max over ranks); bytes are "
                    "rank 0's"}


def run_plugin_e2e(c, dev, steps=3):
    """The reference-facing numpy drop-in, synchronous, numpy in and out:
    ``fusedhead.forward_fully_fused(inputs)`` then ``backward_fused(inputs,
    saved, dY)`` with PRECISION "bf16" (the arithmetic the headline times)."""
    try:
        from paper_2603_25011_b200 import fusedhead as fh
    except ImportError as exc:
        return {"unavailable": f"reference package not installed ({exc})"}
    H, E, b, m, dY = _slice_inputs(c, c["B"], seed=1)
    dims = fh.Dims(c["B"], c["S"], c["D"], c["V"])
    inputs = fh.HeadInputs(dims=dims, H=H, E=E, b=b, mask=m)
    prev = fh.PRECISION
    fh.PRECISION = "bf16"
    try:
        out = fh.forward_fully_fused(inputs)
        fh.backward_fused(inputs, fh.SavedSparseState.from_output(out), dY)
        ts = []
        for _ in range(steps):
            t0 = time.perf_counter()
            out = fh.forward_fully_fused(inputs)
            g = fh.backward_fused(inputs, fh.SavedSparseState.from_output(out), dY)
            ts.append(time.perf_counter() - t0)
    finally:
        fh.PRECISION = prev
    t = statistics.median(ts)
    ff, fb = flops(c)
    h2d = 2 * (H.nbytes + E.nbytes) + b.nbytes + m.nbytes + out.Y.nbytes + out.I.nbytes + dY.nbytes
    d2h = out.Y.nbytes + out.I.nbytes + g.dH.nbytes + g.dE.nbytes + g.db.nbytes
    return {"value": (ff + fb) / t / 1e12, "unit": "TFLOP/s", "ms_per_step": t * 1e3, "steps": steps,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "note": "fusedhead.forward_fully_fused + backward_fused (numpy fp32 in/out, PRECISION='bf16'); "
                    "synchronous copies through pinned staging (inputs memcpy'd into torch's cached pinned "
                    "buffers, outputs returned in pinned host memory), fp32->bf16 conversion on the device; "
                    "the backward "
                    "re-uploads H and E (the reference API passes them again)"}


def main() -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg3")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-plugin", action="store_true", help="skip the numpy drop-in e2e record")
    ap.add_argument("--no-cfg4", action="store_true", help="N>1: skip the cfg4 record")
    ap.add_argument("--no-fused-ab", action="store_true", help="N>1: skip the fused all-gather A/B record")
    ap.add_argument("--no-sparse", action="store_true", help="N=1: skip the SPLADE-sparse (bias -2) record")
    ap.add_argument("--no-cfg1", action="store_true", help="N=1: skip the cfg1 (reference CPU case) record")
    ap.add_argument("--no-naive", action="store_true", help="N=1: skip the naive PyTorch head record")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, c, args.config)
    return run_gpu_arm(args, c, args.config)


if __name__ == "__main__":
    # The reference's tile pool owns the cores; single-threaded BLAS avoids
    # oversubscription (15.5 s vs 6.3 s forward at B=8).  Set
    # before numpy is imported.
    if "--impl" in sys.argv and "reference" in sys.argv:
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    if "--no-cpu" not in sys.argv:
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    raise SystemExit(main())
