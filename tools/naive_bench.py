"""Naive PyTorch GPU head: ((H@E.T + b) * M).relu().log1p().max(dim=1)
with autograd, bf16, same inputs as bench.py.  Records OOM where the B*S*V logits
do not fit, plus the largest B that fits.  Prints one JSON line per config."""
import json
import sys

import torch

sys.path.insert(0, ".")
from bench import CONFIGS, flops, make_inputs  # noqa: E402


def naive_step(H, E, b, m, dY):
    Hq = H.detach().requires_grad_(True)
    Eq = E.detach().requires_grad_(True)
    bq = b.detach().requires_grad_(True)
    L = (torch.einsum("bsd,vd->bsv", Hq, Eq) + bq.to(Hq.dtype)) * m[..., None].to(Hq.dtype)
    Y = L.relu().log1p().max(dim=1).values.float()
    Y.backward(dY)
    return Y


def time_cfg(name, c, B=None):
    c = dict(c)
    if B is not None:
        c["B"] = B
    dev = torch.device("cuda", 0)
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    try:
        H, E, bias, mask, dY, _ = make_inputs(c, dev, 0, 1)
        naive_step(H, E, bias, mask, dY)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 3
        e0.record()
        for _ in range(n):
            naive_step(H, E, bias, mask, dY)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        ff, fb = flops(c)
        return {"path": "naive-pytorch", "config": name, "B": c["B"], "ms_per_step": ms,
                "tflops_algorithmic": (ff + fb) / ms / 1e9, "peak_hbm_bytes": torch.cuda.max_memory_allocated()}
    except torch.OutOfMemoryError:
        return {"path": "naive-pytorch", "config": name, "B": c["B"], "result": "OOM"}


for name in ("cfg2", "cfg3"):
    r = time_cfg(name, CONFIGS[name])
    print(json.dumps(r), flush=True)
    if r.get("result") == "OOM":
        for B in (256, 128, 64, 32, 16, 8):
            r2 = time_cfg(name, CONFIGS[name], B)
            if r2.get("result") != "OOM":
                print(json.dumps(r2), flush=True)
                break
