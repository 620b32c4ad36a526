"""GPU sweep with the reference harness's CSV schema.

Mirrors ``fusedhead.bench.run_sweep`` (/root/reference/pkg/src/fusedhead/bench.py:
193-223) and its CSV row (``BENCH_CSV_HEADER``, bench.py:32-35; ``BenchRecord``
bench.py:142-180; ``y_checksum`` bench.py:61-62) for the ``"b200"`` strategy:
one row per axis value, timed on the device, OOM rows kept with ``OOM``
sentinels.  The reference columns keep their meaning — ``peak_bytes`` is the
torch allocator's peak over the timed calls, ``saved_bytes`` the (Y, I) state
kept for backward, ``y_checksum`` the CRC32 of Y — and GPU columns are
appended: the forward and fwd+bwd medians, the algorithmic TFLOP/s, and the
cost model's compulsory bytes of the b200 plan (``costmodel.b200_traffic``:
forward, backward) with the forward's model bytes over its median time.

    python -m paper_2603_25011_b200.sweep --base 512,512,768,30522 --axis V \
        --values 30522,250002 --out sweep.csv
"""

from __future__ import annotations

import argparse
import statistics
import sys
import zlib

import numpy as np
import torch

from .head import sparton_backward, sparton_forward

REFERENCE_HEADER = ("strategy,B,S,D,V,vocab_tile,batch_tile,threads,"
                    "time_ms_med,time_ms_p10,time_ms_p90,peak_bytes,saved_bytes,y_checksum")
GPU_COLUMNS = "fwd_ms_med,fwdbwd_ms_med,fwdbwd_tflops,fwd_model_bytes,bwd_model_bytes,fwd_model_gbs"
HEADER = REFERENCE_HEADER + "," + GPU_COLUMNS
AXES = ("B", "S", "D", "V")


def y_checksum(Y: np.ndarray) -> str:
    """bench.py:61-62: CRC32 of the float32 Y bytes."""
    return f"{zlib.crc32(np.ascontiguousarray(Y, dtype=np.float32).tobytes()) & 0xFFFFFFFF:08x}"


def _pct(xs, q):
    return float(np.percentile(np.asarray(xs), q))


def sweep_point(B: int, S: int, D: int, V: int, *, repeats: int = 5, warmup: int = 2, seed: int = 0,
                device: str = "cuda") -> str:
    """One CSV row for the b200 strategy at (B, S, D, V) — the forward is the
    timed runner (as in run_sweep); fwd+bwd is timed alongside."""
    dev = torch.device(device)
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats(dev)
    try:
        g = torch.Generator(device=dev).manual_seed(seed)
        H = (torch.rand((B, S, D), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
        E = (torch.rand((V, D), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
        b = torch.rand(V, generator=g, device=dev) * 2 - 1
        m = torch.ones((B, S), dtype=torch.uint8, device=dev)
        dY = torch.rand((B, V), generator=g, device=dev)
        for _ in range(warmup):
            Y, I = sparton_forward(H, E, b, m)
            sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
        fwd, both = [], []
        for _ in range(repeats):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            Y, I = sparton_forward(H, E, b, m)
            e[1].record()
            sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
            e[2].record()
            torch.cuda.synchronize()
            fwd.append(e[0].elapsed_time(e[1]))
            both.append(e[0].elapsed_time(e[2]))
        peak = torch.cuda.max_memory_allocated(dev)
        saved = Y.numel() * 4 + I.numel() * 4
        ck = y_checksum(Y.cpu().numpy())
        flops = 2 * B * S * V * D + 4 * B * V * D
        med = statistics.median(fwd)
        fb, bb = _model_bytes(B, S, D, V)
        return (f"b200,{B},{S},{D},{V},{128 * 2},{1},{1},{med:.6g},{_pct(fwd, 10):.6g},{_pct(fwd, 90):.6g},"
                f"{peak},{saved},{ck},{med:.6g},{statistics.median(both):.6g},"
                f"{flops / (statistics.median(both) * 1e-3) / 1e12:.6g},{fb},{bb},{fb / (med * 1e-3) / 1e9:.6g}")
    except torch.OutOfMemoryError:
        fb, bb = _model_bytes(B, S, D, V)
        return f"b200,{B},{S},{D},{V},256,1,1,OOM,OOM,OOM,OOM,OOM,OOM,OOM,OOM,OOM,{fb},{bb},OOM"


def _model_bytes(B, S, D, V):
    """(forward, backward) compulsory bytes of the b200 plan (costmodel.py)."""
    from . import costmodel
    from .fusedhead import Dims
    rep = costmodel.b200_traffic(Dims(B, S, D, V))
    st = rep.stages
    return st[0].bytes_read + st[0].bytes_written, sum(x.bytes_read + x.bytes_written for x in st[1:])


def run_sweep(base: tuple[int, int, int, int], axis: str, values, **kw) -> list[str]:
    """Every axis value in order, never dropping one (bench.py:193-223)."""
    if axis not in AXES:
        raise ValueError(f"axis must be one of {AXES}, got {axis!r}")
    if not values:
        raise ValueError("values must be non-empty")
    rows = []
    for v in values:
        dims = dict(zip(AXES, base))
        dims[axis] = int(v)
        rows.append(sweep_point(dims["B"], dims["S"], dims["D"], dims["V"], **kw))
    return rows


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="b200 Sparton head sweep (reference CSV schema + GPU columns)")
    ap.add_argument("--base", default="512,512,768,30522", help="B,S,D,V")
    ap.add_argument("--axis", default="V", choices=AXES)
    ap.add_argument("--values", default="30522,250002")
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--out", default="-")
    a = ap.parse_args(argv)
    base = tuple(int(x) for x in a.base.split(","))
    if len(base) != 4 or min(base) < 1:
        print("--base must be four positive integers B,S,D,V", file=sys.stderr)
        return 2
    rows = run_sweep(base, a.axis, [int(x) for x in a.values.split(",")], repeats=a.repeats, warmup=a.warmup)
    text = HEADER + "\n" + "\n".join(rows) + "\n"
    if a.out == "-":
        sys.stdout.write(text)
    else:
        with open(a.out, "w") as f:
            f.write(text)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
