"""A/B two or more builds of libsparton_b200.so on the cfg3 fwd+bwd step, in
ONE process on one box (alternating A B ... A B ... to cancel clock drift).
Uses only the entry points every build exports (sparton_fwd, sparton_bwd,
workspace query) through ctypes, so builds from earlier rounds can be compared;
checks that every build produces the same Y, I, dH, dE and db.

    python tools/ab_step.py build/ab/r01.so build/ab/cur.so [more.so ...] [--rounds 4] [--steps 10]
"""
import ctypes
import statistics
import sys

import torch

import argparse
ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--shape", default="512,512,768,250002", help="B,S,D,V")
args = ap.parse_args()
names = args.libs
libs = [ctypes.CDLL(p) for p in names]
rounds, steps = args.rounds, args.steps
vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
for lib in libs:
    lib.sparton_fwd.argtypes = [vp] * 6 + [i64] * 5 + [ci, vp]
    lib.sparton_bwd_workspace_bytes.argtypes = [i64] * 4 + [ci]
    lib.sparton_bwd_workspace_bytes.restype = ctypes.c_size_t
    lib.sparton_bwd.argtypes = [vp] * 8 + [i64] * 6 + [ci, ci, vp, ctypes.c_size_t, vp]

B, S, D, V = (int(x) for x in args.shape.split(","))
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
H = torch.randn((B, S, D), generator=g, device=dev).to(torch.bfloat16)
E = (torch.randn((V, D), generator=g, device=dev) * 0.02).to(torch.bfloat16)
b = torch.zeros(V, device=dev)
m = torch.ones((B, S), dtype=torch.uint8, device=dev)
dY = torch.randn((B, V), generator=g, device=dev)
Y = torch.empty((B, V), device=dev)
I = torch.empty((B, V), dtype=torch.int32, device=dev)
dH = torch.empty((B, S, D), dtype=torch.bfloat16, device=dev)
dE = torch.empty((V, D), dtype=torch.bfloat16, device=dev)
db = torch.empty(V, device=dev)
ws_n = max(int(lib.sparton_bwd_workspace_bytes(B, S, D, V, 1)) for lib in libs)
ws = torch.empty(ws_n, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream


def step(lib, fwd_ev):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    assert lib.sparton_fwd(H.data_ptr(), E.data_ptr(), b.data_ptr(), m.data_ptr(), Y.data_ptr(), I.data_ptr(),
                           B, S, D, V, V, 0, st) == 0
    e1.record()
    fwd_ev.append((e0, e1))
    assert lib.sparton_bwd(H.data_ptr(), E.data_ptr(), Y.data_ptr(), I.data_ptr(), dY.data_ptr(), dH.data_ptr(),
                           dE.data_ptr(), db.data_ptr(), B, S, D, V, V, V, 1, 1, ws.data_ptr(), ws_n, st) == 0


res = {k: [] for k in range(len(libs))}
ref = None
for r in range(rounds):
    for k, lib in enumerate(libs):
        fe = []
        for _ in range(3):
            step(lib, fe)
        torch.cuda.synchronize()
        if r == 0:   # every build must compute the same outputs
            out = [t.clone() for t in (Y, I, dH, dE, db)]
            if ref is None:
                ref = out
            else:
                same = [torch.equal(a, c) for a, c in zip(ref, out)]
                print(f"{names[k]}: outputs equal to {names[0]} (Y, I, dH, dE, db): {same}", flush=True)
        fe.clear()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(steps):
            step(lib, fe)
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / steps
        fwd = statistics.mean(a.elapsed_time(c) for a, c in fe)
        res[k].append((ms, fwd))
        print(f"round {r} {names[k]}: step {ms:.2f} ms  fwd {fwd:.2f}  bwd {ms - fwd:.2f}", flush=True)
for k in range(len(libs)):
    ms = statistics.median(x[0] for x in res[k])
    fwd = statistics.median(x[1] for x in res[k])
    print(f"MEDIAN {names[k]}: step {ms:.2f} fwd {fwd:.2f} bwd {ms - fwd:.2f}")
