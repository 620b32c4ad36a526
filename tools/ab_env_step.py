"""A/B experiment switches on the cfg3 fwd+bwd step in ONE process: each
config is a set of SPARTON_* variables (honoured under SPARTON_DEV=1, read by
the library at every call); configs alternate round by round to cancel clock
drift.  Prints per-round and median step / forward / backward times.

    python tools/ab_env_step.py 'SPARTON_FWD_GROUP_KB=49152' 'SPARTON_FWD_GROUP_KB=32768' [--rounds 6 --steps 10]
"""
import argparse
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ["SPARTON_DEV"] = "1"
from paper_2603_25011_b200 import bwd_workspace_bytes, sparton_backward, sparton_forward  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="+")
ap.add_argument("--rounds", type=int, default=6)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--shape", default="512,512,768,250002")
ap.add_argument("--no-check", action="store_true", help="configs may change outputs (timing-only variants)")
a = ap.parse_args()
B, S, D, V = (int(x) for x in a.shape.split(","))
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
H = torch.randn((B, S, D), generator=g, device=dev).to(torch.bfloat16)
E = (torch.randn((V, D), generator=g, device=dev) * 0.02).to(torch.bfloat16)
b = torch.zeros(V, device=dev)
m = torch.ones((B, S), dtype=torch.uint8, device=dev)
dY = torch.randn((B, V), generator=g, device=dev)
Y = torch.empty((B, V), device=dev)
I = torch.empty((B, V), dtype=torch.int32, device=dev)


def apply(cfg):
    for k in [k for k in os.environ if k.startswith("SPARTON_") and k != "SPARTON_DEV"]:
        del os.environ[k]
    for kv in cfg.split(","):
        if "=" in kv:
            k, v = kv.split("=", 1)
            os.environ[k.strip()] = v.strip()


def step(fe):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sparton_forward(H, E, b, m, out=(Y, I))
    e1.record()
    fe.append((e0, e1))
    sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)


ref = None
res = {c: [] for c in a.configs}
for r in range(a.rounds):
    for c in a.configs:
        apply(c)
        fe = []
        for _ in range(3):
            step(fe)
        torch.cuda.synchronize()
        if r == 0 and not a.no_check:   # outputs must not depend on the switch
            key = (Y.clone(), I.clone())
            if ref is None:
                ref = key
            else:
                assert torch.equal(ref[0], key[0]) and torch.equal(ref[1], key[1]), f"{c}: Y/I differ"
        fe.clear()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(a.steps):
            step(fe)
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / a.steps
        fwd = statistics.mean(x.elapsed_time(y) for x, y in fe)
        res[c].append((ms, fwd))
        print(f"round {r} [{c}]: step {ms:.2f} ms  fwd {fwd:.2f}  bwd {ms - fwd:.2f}", flush=True)
for c in a.configs:
    ms = statistics.median(x[0] for x in res[c])
    fwd = statistics.median(x[1] for x in res[c])
    print(f"MEDIAN [{c}]: step {ms:.2f} fwd {fwd:.2f} bwd {ms - fwd:.2f}")
