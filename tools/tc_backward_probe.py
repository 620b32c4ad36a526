"""Tensor-core formulation of the backward: measured lower bound.

north_star words dH and dE/db as "gather-GEMMs, also on tensor cores".  Each
(b, v) pair has exactly one argmax row, so as matrices the routing operands are
one-hot: a tcgen05/cuBLAS tile of M rows computes M multiply-adds for every
useful one.  The cheapest tensor-core variant compacts K to the rows a tile
actually touches:

* dE: per (b, 128-row vocab tile) the A operand is 128 x K with K = distinct
  argmax positions s of the tile (one nonzero g per row), B = the K gathered
  H[b, s, :] rows (K x D);
* dH: per (b, 128-position s-tile) A = 128 x K with K = the vocabulary rows
  whose argmax falls in the tile, B = the K gathered E rows (K x D).

This probe takes (Y, I) from a real cfg3 forward, counts the compacted K of
every tile (rounded up to the MMA's K granularity of 16), and times cuBLAS
bf16 batched GEMMs of exactly those shapes on representative batches — the
GEMMs alone, without the gathers that would feed them — then extrapolates to
the whole backward.  Compare with the CUDA-core kernels' measured times.

    python tools/tc_backward_probe.py > profiles/r02_tc_backward_probe.json
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_25011_b200 import sparton_forward  # noqa: E402


def time_bmm(batch, M, K, N, dev, reps=5):
    a = torch.randn((batch, M, K), device=dev, dtype=torch.bfloat16)
    b = torch.randn((batch, K, N), device=dev, dtype=torch.bfloat16)
    for _ in range(2):
        torch.bmm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.bmm(a, b)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = torch.device("cuda", 0)
    B, S, D, V = 512, 512, 768, 250002
    g = torch.Generator(device=dev).manual_seed(0)
    H = torch.randn((B, S, D), generator=g, device=dev).to(torch.bfloat16)
    E = (torch.randn((V, D), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    Y, I = sparton_forward(H, E, torch.zeros(V, device=dev), torch.ones((B, S), dtype=torch.uint8, device=dev))
    del H, E
    act = (Y > 0)
    # ---- dE: distinct s per (b, 128-v tile)
    nvt = (V + 127) // 128
    Ip = torch.full((B, nvt * 128), -1, dtype=torch.int64, device=dev)
    Ip[:, :V] = torch.where(act, I.long(), torch.full_like(I.long(), -1))
    tiles = Ip.view(B, nvt, 128)
    onehot_cnt = torch.zeros((B, nvt, S + 1), dtype=torch.int32, device=dev)
    onehot_cnt.scatter_add_(2, tiles + 1, torch.ones_like(tiles, dtype=torch.int32))
    distinct = (onehot_cnt[:, :, 1:] > 0).sum(2)                      # (B, nvt)
    kde = ((distinct + 15) // 16 * 16).clamp(min=16)
    # ---- dH: vocabulary rows per (b, 128-position s tile)
    nst = (S + 127) // 128
    st = torch.where(act, I.long() // 128, torch.full_like(I.long(), nst))
    cnt = torch.zeros((B, nst + 1), dtype=torch.int64, device=dev)
    cnt.scatter_add_(1, st, torch.ones_like(st))
    kdh = ((cnt[:, :nst] + 15) // 16 * 16)
    out = {"config": {"B": B, "S": S, "D": D, "V": V}, "pairs_active": int(act.sum())}
    # Representative timing: the median compacted K, batch of 4096 tiles.
    kde_med = int(kde.float().median())
    n_de = B * nvt
    t = time_bmm(4096, 128, kde_med, D, dev)
    de_flops = 2.0 * 128 * D * float(kde.sum())
    de_ms = t * n_de / 4096
    out["dE"] = {"tiles": n_de, "median_K": kde_med, "mean_K": float(kde.float().mean()),
                 "gemm_tflop": de_flops / 1e12, "redundancy_vs_useful": de_flops / (2.0 * D * float(act.sum())),
                 "bmm_ms_per_4096_tiles": t, "extrapolated_gemm_ms": de_ms,
                 "achieved_tflops": 2.0 * 128 * D * kde_med * 4096 / (t * 1e-3) / 1e12}
    # dH: K per (b, s-tile) ~ V/4; time a few batch rows' worth at the median K.
    kdh_med = int(kdh.float().median())
    t2 = time_bmm(64, 128, kdh_med, D, dev, reps=3)
    n_dh = B * nst
    dh_flops = 2.0 * 128 * D * float(kdh.sum())
    out["dH"] = {"tiles": n_dh, "median_K": kdh_med, "gemm_tflop": dh_flops / 1e12,
                 "redundancy_vs_useful": dh_flops / (2.0 * D * float(act.sum())),
                 "bmm_ms_per_64_tiles": t2, "extrapolated_gemm_ms": t2 * n_dh / 64,
                 "achieved_tflops": 2.0 * 128 * D * kdh_med * 64 / (t2 * 1e-3) / 1e12}
    out["note"] = ("GEMM time only (cuBLAS bf16 bmm of the compacted one-hot shapes), no gathers, no g "
                   "precision split; the CUDA-core kernels it would replace run staged dE 9.4 ms and "
                   "dH 8 x 1.42 ms at 1.96 GHz (profiles/r02_launches_cfg3_summary.txt)")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
