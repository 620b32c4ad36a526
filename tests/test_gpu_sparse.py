"""The backward's sparse regime (SURVEY.md §8d "SPLADE-sparse" variant).

SPLADE representations are mostly zeros: few (b, v) pairs are active
(Y > 0, fused.py:247-249).  The route counts them on the device; at most
40 % active pairs run the sparse dE (per-pair gathers of the active rows
only, the staged dE + db kernels exit), at most 12 % the single-pass dH
(whole vocabulary, no fp32 carry).  Checks: parity with the oracle at a few
percent activity (including > 32 route windows, the dH window groups), the
all-inactive batch, and bit-equality of the sparse and dense kernels on the
same inputs (the dev-gated thresholds force either path), for fp32 and bf16
gradients.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import sparton_oracle as orc

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-2, 1e-3


def _dev():
    return torch.device("cuda", 0)


def _sparse_inputs(B, S, D, V, seed, active):
    """Reference-style inputs with a per-vocab bias that leaves about
    `active` of the (b, v) pairs positive (the largest raw maxima)."""
    H, E, _, m = orc.seeded_inputs(B, S, D, V, seed, mask_keep=0.85)
    H, E = orc.bf16_round(H), orc.bf16_round(E)
    from paper_2603_25011_b200 import sparton_forward
    Ht = torch.from_numpy(H).to(_dev()).to(torch.bfloat16)
    Et = torch.from_numpy(E).to(_dev()).to(torch.bfloat16)
    mt = torch.from_numpy(m).to(_dev())
    Y0, _ = sparton_forward(Ht, Et, torch.zeros(V, device=_dev()), mt)
    raw = torch.expm1(Y0).flatten().float()
    thr = float(torch.quantile(raw[torch.randperm(raw.numel(), device=_dev())[:1 << 20]], 1.0 - active))
    b = np.full(V, -thr, np.float32)
    bt = torch.from_numpy(b).to(_dev())
    Y, I = sparton_forward(Ht, Et, bt, mt)
    torch.cuda.synchronize()
    dY = orc.seeded_uniform((B, V), seed + 7)
    return H, E, b, Y, I, dY, Ht, Et


def _bwd(Ht, Et, Y, I, dY, grad_dtype=torch.float32):
    from paper_2603_25011_b200 import sparton_backward
    dH, dE, db = sparton_backward(Ht, Et, Y, I, torch.from_numpy(dY).to(_dev()), grad_dtype=grad_dtype)
    torch.cuda.synchronize()
    return dH, dE, db


def _close(a, b):
    a = a.float().cpu().numpy().astype(np.float64) if isinstance(a, torch.Tensor) else a
    return np.all(np.abs(a - b) <= ATOL + RTOL * np.abs(b)), float(np.max(np.abs(a - b)))


@pytest.mark.parametrize("dims,active", [
    ((4, 128, 768, 5000), 0.05),
    ((3, 300, 256, 20000), 0.02),
    ((2, 64, 1024, 70000), 0.08),
    ((2, 40, 520, 3000), 0.10),      # D not a multiple of 256: partial lane chunks
    ((2, 64, 64, 300000), 0.03),     # 37 route windows: the single-pass dH walks two window groups
])
def test_sparse_regime_vs_oracle(cuda_device, dims, active):
    B, S, D, V = dims
    H, E, b, Y, I, dY, Ht, Et = _sparse_inputs(B, S, D, V, 500 + V, active)
    frac = float((Y > 0).float().mean())
    assert 0 < frac < 0.12, frac
    Yn, In = Y.cpu().numpy(), I.cpu().numpy()
    dH_r, dE_r, db_r = orc.backward(H, E, b, Yn, In, dY)
    dH, dE, db = _bwd(Ht, Et, Y, I, dY)
    for name, got, ref in (("dH", dH, dH_r), ("dE", dE, dE_r), ("db", db, db_r)):
        ok, err = _close(got, ref)
        assert ok, (name, err)


def test_all_pairs_inactive(cuda_device):
    B, S, D, V = 3, 64, 256, 9000
    H, E, _, m = orc.seeded_inputs(B, S, D, V, 11)
    from paper_2603_25011_b200 import sparton_forward
    Ht = torch.from_numpy(orc.bf16_round(H)).to(_dev()).to(torch.bfloat16)
    Et = torch.from_numpy(orc.bf16_round(E)).to(_dev()).to(torch.bfloat16)
    Y, I = sparton_forward(Ht, Et, torch.full((V,), -1e4, device=_dev()), torch.from_numpy(m).to(_dev()))
    assert not bool((Y > 0).any())
    for gd in (torch.float32, torch.bfloat16):
        dH, dE, db = _bwd(Ht, Et, Y, I, orc.seeded_uniform((B, V), 3), gd)
        assert not dH.any() and not dE.any() and not db.any()


@pytest.mark.parametrize("grad_dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("active", [0.04, 0.5])
def test_sparse_and_dense_kernels_bitwise_equal(cuda_device, monkeypatch, grad_dtype, active):
    """Same inputs through the sparse kernels (thresholds 100 %) and the dense
    ones (thresholds disabled): identical bits — one fp32 FMA chain per output
    in the reference's order either way.  V = 100000 gives the dense dH four
    vocabulary passes with the fp32 carry."""
    B, S, D, V = 4, 256, 768, 100000
    H, E, b, Y, I, dY, Ht, Et = _sparse_inputs(B, S, D, V, 77, active)
    monkeypatch.setenv("SPARTON_DEV", "1")
    out = {}
    for mode, pct in (("sparse", "100"), ("dense", "-1")):
        monkeypatch.setenv("SPARTON_DE_SPARSE_PCT", pct)
        monkeypatch.setenv("SPARTON_DH_SPARSE_PCT", pct)
        out[mode] = [t.clone() for t in _bwd(Ht, Et, Y, I, dY, grad_dtype)]
    for name, a, c in zip(("dH", "dE", "db"), out["sparse"], out["dense"]):
        assert torch.equal(a.view(torch.int16 if a.dtype == torch.bfloat16 else torch.int32),
                           c.view(torch.int16 if c.dtype == torch.bfloat16 else torch.int32)), name


def test_default_thresholds_pick_per_kernel(cuda_device, monkeypatch):
    """Between the two thresholds (12 % < active <= 40 %) dE runs sparse and
    dH dense; results equal the all-dense run bit for bit."""
    B, S, D, V = 4, 128, 256, 40000
    H, E, b, Y, I, dY, Ht, Et = _sparse_inputs(B, S, D, V, 91, 0.18)
    frac = float((Y > 0).float().mean())
    assert 0.12 < frac <= 0.4, frac
    default = [t.clone() for t in _bwd(Ht, Et, Y, I, dY)]
    monkeypatch.setenv("SPARTON_DEV", "1")
    monkeypatch.setenv("SPARTON_DE_SPARSE_PCT", "-1")
    monkeypatch.setenv("SPARTON_DH_SPARSE_PCT", "-1")
    dense = _bwd(Ht, Et, Y, I, dY)
    for a, c in zip(default, dense):
        assert torch.equal(a, c)
