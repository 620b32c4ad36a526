"""CPU oracle for the Sparton hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's algorithm
(/root/reference/pkg/src/fusedhead, pure Python/numpy — restated, not
imported, because /root/reference does not exist on the GPU box).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this module, and only as the checker or the timed
CPU baseline — never on the product path.

Pinned against the reference: ``tests/golden/*.npz`` were produced by running
the reference itself (``tests/golden/make_golden.py``) and
``tests/test_oracle.py`` checks this module against them bit-for-bit (I, and
Y/grads in deterministic mode) or within the reference's own tolerances.

Each function cites the reference lines it restates.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_SM64_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_SM64_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_SM64_MIX2 = np.uint64(0x94D049BB133111EB)


# ---------------------------------------------------------------- inputs (tensor.py:58-115)

def splitmix64(seed: int, count: int) -> np.ndarray:
    """tensor.py:58-69: word i = mix(seed + (i+1)·γ), wrapping uint64."""
    state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    idx = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = state + idx * _SM64_GAMMA
        z = (z ^ (z >> np.uint64(30))) * _SM64_MIX1
        z = (z ^ (z >> np.uint64(27))) * _SM64_MIX2
    return z ^ (z >> np.uint64(31))


def unit_floats(seed: int, count: int) -> np.ndarray:
    """tensor.py:72-74: top 53 bits -> float64 in [0, 1)."""
    return (splitmix64(seed, count) >> np.uint64(11)).astype(np.float64) * (2.0**-53)


def seeded_uniform(shape, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """tensor.py:91-105 (Uniform branch)."""
    n = int(np.prod(shape))
    return (lo + (hi - lo) * unit_floats(seed, n)).astype(np.float32).reshape(shape)


def seeded_mask(batch: int, seq: int, seed: int, keep: float = 1.0) -> np.ndarray:
    """tensor.py:108-115."""
    if keep >= 1.0:
        return np.ones((batch, seq), np.uint8)
    return (unit_floats(seed, batch * seq) < keep).astype(np.uint8).reshape(batch, seq)


def seeded_inputs(B, S, D, V, seed, mask_keep=1.0, lo=-1.0, hi=1.0):
    """HeadInputs.seeded (reference.py:48-69): H=seed, E=seed+1, b=seed+2, mask=seed+3."""
    H = seeded_uniform((B, S, D), seed, lo, hi)
    E = seeded_uniform((V, D), seed + 1, lo, hi)
    b = seeded_uniform((V,), seed + 2, lo, hi)
    mask = seeded_mask(B, S, seed + 3, mask_keep)
    return H, E, b, mask


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even) -> fp32; the GPU's input rounding."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32).reshape(np.shape(x))


# ---------------------------------------------------------------- forward

def _reduce(L: np.ndarray):
    """reference.py:96-100 / fused.py:146-151: first-index argmax over s, then
    log1p∘ReLU of the reduced maxima."""
    idx = np.argmax(L, axis=1).astype(np.int32)
    raw = np.take_along_axis(L, idx[:, None, :], axis=1)[:, 0, :]
    return np.log1p(np.maximum(raw, np.float32(0))), idx


def forward(H, E, b, mask, *, deterministic: bool = False, vocab_tile: int = 4096, threads: int = 1):
    """forward_hybrid (fused.py:115-157) / forward_eager (reference.py:103-125).

    Per (batch row, vocab tile): logits = H[b]·E_tileᵀ + bias (fp32; BLAS, or a
    fixed-order k loop when deterministic, tensor.py:173-179), masked by
    multiplication (masked positions are exactly ±0 and still compete,
    reference.py:121-122), then first-index max/argmax and log1p∘ReLU.
    Returns (Y f32 [B,V], I i32 [B,V]).
    """
    B, S, D = H.shape
    V = E.shape[0]
    Y = np.empty((B, V), np.float32)
    I = np.empty((B, V), np.int32)
    m = mask.astype(np.float32)

    def tile(job):
        bi, v0 = job
        v1 = min(v0 + vocab_tile, V)
        e = E[v0:v1]
        if deterministic:
            L = np.zeros((S, v1 - v0), np.float32)
            for k in range(D):
                L += H[bi, :, k, None] * e[None, :, k]
        else:
            L = H[bi] @ e.T
        L += b[v0:v1]
        L *= m[bi, :, None]
        y, i = _reduce(L[None])
        Y[bi, v0:v1] = y[0]
        I[bi, v0:v1] = i[0]

    jobs = [(bi, v0) for bi in range(B) for v0 in range(0, V, vocab_tile)]
    if threads > 1:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(tile, jobs))
    else:
        for j in jobs:
            tile(j)
    return Y, I


def logits_f64(H, E, b, mask, rows=None):
    """eval_head_f64's logits (reference.py:186-198), optionally for a subset of
    batch rows: float64 (B', S, V) masked logits."""
    Hs = H if rows is None else H[rows]
    ms = mask if rows is None else mask[rows]
    L = np.einsum("bsd,vd->bsv", Hs.astype(np.float64), E.astype(np.float64))
    L += b.astype(np.float64)[None, None, :]
    L *= ms[:, :, None]
    return L


def forward_f64(H, E, b, mask):
    """eval_head_f64 (reference.py:186-198)."""
    L = logits_f64(H, E, b, mask)
    idx = np.argmax(L, axis=1)
    raw = np.take_along_axis(L, idx[:, None, :], axis=1)[:, 0, :]
    return np.log1p(np.maximum(raw, 0.0)), idx.astype(np.int32)


# ---------------------------------------------------------------- backward

def backward(H, E, b, Y, I, dY, *, include_bias_grad: bool = True):
    """backward_fused (fused.py:215-278) from the saved (Y, I).

    g = dY·exp(−Y) on pairs with Y > 0 (fused.py:247-249).  dE/db accumulate
    over b ascending (embed_block, fused.py:255-265); dH[b] accumulates via
    np.add.at in ascending v order (hidden_row, fused.py:267-273).
    """
    B, S, D = H.shape
    V = E.shape[0]
    pos = Y > 0
    g = np.zeros((B, V), np.float32)
    g[pos] = dY[pos] * np.exp(-Y[pos])
    dH = np.zeros_like(H, dtype=np.float32)
    dE = np.zeros((V, D), np.float32)
    db = np.zeros((V,), np.float32)
    for bi in range(B):
        vs = np.nonzero(pos[bi])[0]
        if vs.size == 0:
            continue
        gv = g[bi, vs]
        dE[vs] += gv[:, None] * H[bi, I[bi, vs], :]
        if include_bias_grad:
            db[vs] += gv
        np.add.at(dH[bi], I[bi, vs], gv[:, None] * E[vs, :])
    return dH, dE, db


def backward_rows(H, E, Y, I, dY, rows):
    """dH for a subset of batch rows only (hidden_row, fused.py:267-273) — the
    head is separable in b, so a B-slice reproduces those rows exactly."""
    out = np.zeros((len(rows), H.shape[1], H.shape[2]), np.float32)
    for j, bi in enumerate(rows):
        pos = Y[bi] > 0
        vs = np.nonzero(pos)[0]
        if vs.size == 0:
            continue
        gv = (dY[bi, vs] * np.exp(-Y[bi, vs])).astype(np.float32)
        np.add.at(out[j], I[bi, vs], gv[:, None] * E[vs, :])
    return out


def backward_cols(H, Y, I, dY, cols):
    """dE/db for a subset of vocab columns (embed_block, fused.py:255-265) —
    separable in v, so a V-slice reproduces those rows exactly."""
    B, S, D = H.shape
    dE = np.zeros((len(cols), D), np.float32)
    db = np.zeros((len(cols),), np.float32)
    cols = np.asarray(cols)
    for bi in range(B):
        y = Y[bi, cols]
        pos = y > 0
        if not pos.any():
            continue
        j = np.nonzero(pos)[0]
        gv = (dY[bi, cols[j]] * np.exp(-y[j])).astype(np.float32)
        dE[j] += gv[:, None] * H[bi, I[bi, cols[j]], :]
        db[j] += gv
    return dE, db


# ---------------------------------------------------------------- parity helpers

def near_tie_ok(H, E, b, mask, bi, v, s_a, s_b) -> bool:
    """Two candidate argmax positions s_a, s_b of pair (bi, v) are a documented
    near-tie when |L64[s_a] − L64[s_b]| <= 4·D·2^-24·max(A_a, A_b), with
    A_s = Σ_k |H[bi,s,k]·E[v,k]| + |b[v]| (the fp32 accumulation-order bound),
    everything in float64."""
    D = H.shape[2]
    h = H[bi].astype(np.float64)
    e = E[v].astype(np.float64)
    bv = float(b[v])

    def logit(s):
        return (float(h[s] @ e) + bv) * float(mask[bi, s])

    def mag(s):
        return (float(np.abs(h[s] * e).sum()) + abs(bv)) * float(mask[bi, s])

    gap = abs(logit(s_a) - logit(s_b))
    bound = 4.0 * D * 2.0**-24 * max(mag(s_a), mag(s_b), 1e-30)
    return gap <= bound


def check_forward(H, E, b, mask, Y_gpu, I_gpu, Y_ref, I_ref, *, rtol=1e-2, atol=1e-3, rows=None):
    """Compare a device forward with the oracle: Y within (rtol, atol); I exact
    except at certified near-ties.  Returns (ok, report dict)."""
    rows = np.arange(Y_ref.shape[0]) if rows is None else np.asarray(rows)
    dy = np.abs(Y_gpu.astype(np.float64) - Y_ref.astype(np.float64))
    tol = atol + rtol * np.abs(Y_ref.astype(np.float64))
    y_bad = int((dy > tol).sum())
    mism = np.argwhere(I_gpu != I_ref)
    ties = 0
    hard = 0
    for (r, v) in mism:
        bi = int(rows[r])
        if near_tie_ok(H, E, b, mask, bi, int(v), int(I_gpu[r, v]), int(I_ref[r, v])):
            ties += 1
        else:
            hard += 1
    rep = {"max_abs_dY": float(dy.max()) if dy.size else 0.0, "y_bad": y_bad,
           "idx_mismatch": int(len(mism)), "near_ties": ties, "hard_mismatch": hard}
    return (y_bad == 0 and hard == 0), rep


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


def flops(B, S, D, V) -> tuple[int, int]:
    """Algorithmic work: fwd 2·B·S·V·D, bwd 4·B·V·D."""
    return 2 * B * S * V * D, 4 * B * V * D

