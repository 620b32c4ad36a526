"""GPU parity of the argmax-routed backward (K2 dE/db, K3 route + dH).

Ports of test_fused.py:164-248 and test_reference.py:143-183.  Gradients are
driven by the GPU's own (Y, I) so parity is independent of argmax near-ties
(SURVEY.md §7.1).  Tolerance: rtol 1e-2 / atol 1e-3 (north star); observed
agreement is ~1e-6 since both sides accumulate fp32 in the same order.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden_names, load_golden
from oracle import sparton_oracle as orc

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-2, 1e-3


def _dev():
    return torch.device("cuda", 0)


def t_bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(_dev()).to(torch.bfloat16)


def t_f32(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(_dev())


def run_bwd(H, E, Y, I, dY, include_bias_grad=True, grad_dtype=torch.float32):
    from paper_2603_25011_b200 import sparton_backward
    It = torch.from_numpy(np.ascontiguousarray(I, np.int32)).to(_dev())
    dH, dE, db = sparton_backward(t_bf16(H), t_bf16(E), t_f32(Y), It, t_f32(dY),
                                  include_bias_grad=include_bias_grad, grad_dtype=grad_dtype)
    torch.cuda.synchronize()
    return dH.float().cpu().numpy(), dE.float().cpu().numpy(), db.cpu().numpy()


def run_fwd(H, E, b, m):
    from paper_2603_25011_b200 import sparton_forward
    Y, I = sparton_forward(t_bf16(H), t_bf16(E), t_f32(b),
                           torch.from_numpy(np.ascontiguousarray(m, np.uint8)).to(_dev()))
    return Y.cpu().numpy(), I.cpu().numpy()


def close(a, b, rtol=RTOL, atol=ATOL):
    return np.all(np.abs(a.astype(np.float64) - b.astype(np.float64)) <= atol + rtol * np.abs(b))


@pytest.mark.parametrize("name", golden_names())
def test_golden_backward(cuda_device, name):
    g = load_golden(name)
    H, E = g["H"], g["E"]
    if not bool(g["bf16"]):
        H, E = orc.bf16_round(H), orc.bf16_round(E)
        dH_r, dE_r, db_r = orc.backward(H, E, g["b"], g["Y"], g["I"], g["dY"])
    else:
        dH_r, dE_r, db_r = g["dH"], g["dE"], g["db"]   # the reference's own gradients
    dH, dE, db = run_bwd(H, E, g["Y"], g["I"], g["dY"])
    assert close(dH, dH_r) and close(dE, dE_r) and close(db, db_r)
    assert np.max(np.abs(dE - dE_r)) < 1e-4 and np.max(np.abs(dH - dH_r)) < 1e-4


GRID = [(1, 1, 16, 1), (2, 3, 16, 5), (4, 8, 16, 16), (2, 64, 64, 300), (3, 130, 256, 389),
        (2, 512, 768, 2000), (4, 33, 1024, 777), (2, 40, 520, 100), (3, 7, 8, 1000),
        # S beyond the staged dE's two-stage smem limit: the gathered dE path.
        (2, 1000, 128, 700), (5, 856, 64, 1501),
        # S > 2125: fewer than 16 route segments fit in smem (two-pass route)
        (1, 2200, 16, 3000)]


@pytest.mark.parametrize("dims", GRID)
def test_grid_vs_oracle_with_gpu_state(cuda_device, dims):
    B, S, D, V = dims
    H, E, b, m = orc.seeded_inputs(B, S, D, V, 300 + S + V, mask_keep=0.85)
    H, E = orc.bf16_round(H), orc.bf16_round(E)
    dY = orc.seeded_uniform((B, V), 99)
    Y, I = run_fwd(H, E, b, m)
    dH_r, dE_r, db_r = orc.backward(H, E, b, Y, I, dY)
    dH, dE, db = run_bwd(H, E, Y, I, dY)
    assert close(dH, dH_r), np.max(np.abs(dH - dH_r))
    assert close(dE, dE_r), np.max(np.abs(dE - dE_r))
    assert close(db, db_r), np.max(np.abs(db - db_r))


def test_zero_upstream_gradient(cuda_device):
    H, E, b, m = orc.seeded_inputs(2, 3, 8, 5, 42)
    Y, I = run_fwd(H, E, b, m)
    dH, dE, db = run_bwd(H, E, Y, I, np.zeros((2, 5), np.float32))
    assert not dH.any() and not dE.any() and not db.any()


def test_scalar_closed_form(cuda_device):
    x, w = 0.75, 0.875           # exact in bf16
    H = np.full((1, 1, 1), x, np.float32)
    E = np.full((1, 1), w, np.float32)
    b = np.zeros(1, np.float32)
    Y, I = run_fwd(H, E, b, np.ones((1, 1), np.uint8))
    dH, dE, db = run_bwd(H, E, Y, I, np.ones((1, 1), np.float32))
    assert dH[0, 0, 0] == pytest.approx(w / (1 + x * w), rel=1e-6)
    assert dE[0, 0] == pytest.approx(x / (1 + x * w), rel=1e-6)
    assert db[0] == pytest.approx(1 / (1 + x * w), rel=1e-6)


def test_bias_grad_can_be_disabled(cuda_device):
    H, E, b, m = orc.seeded_inputs(2, 3, 8, 5, 42)
    Y, I = run_fwd(H, E, b, m)
    dY = orc.seeded_uniform((2, 5), 9)
    dH, dE, db = run_bwd(H, E, Y, I, dY, include_bias_grad=False)
    assert not db.any() and dE.any()


def test_dead_relu_zero_grads(cuda_device):
    H, E, _, m = orc.seeded_inputs(2, 4, 8, 6, 1)
    b = np.full(6, -50.0, np.float32)
    Y, I = run_fwd(H, E, b, m)
    dH, dE, db = run_bwd(H, E, Y, I, orc.seeded_uniform((2, 6), 2))
    assert not dH.any() and not dE.any() and not db.any()


def test_reads_only_active_argmax_rows(cuda_device):
    # test_fused.py:197-226: poison every H row that is not an active argmax row.
    B, S, D, V = 2, 6, 16, 8
    H, E, b, m = orc.seeded_inputs(B, S, D, V, 31, mask_keep=0.7)
    H, E = orc.bf16_round(H), orc.bf16_round(E)
    dY = orc.seeded_uniform((B, V), 32)
    Y, I = run_fwd(H, E, b, m)
    clean = run_bwd(H, E, Y, I, dY)
    needed = {(bi, int(I[bi, v])) for bi in range(B) for v in np.nonzero(Y[bi] > 0)[0]}
    Hp = H.copy()
    for bi in range(B):
        for s in range(S):
            if (bi, s) not in needed:
                Hp[bi, s, :] = np.nan
    dirty = run_bwd(Hp, E, Y, I, dY)
    assert np.array_equal(clean[1], dirty[1]) and np.array_equal(clean[2], dirty[2])
    for bi in range(B):
        for s in range(S):
            if (bi, s) not in needed:
                assert not dirty[0][bi, s].any()


def test_bf16_gradients(cuda_device):
    B, S, D, V = 2, 64, 128, 300
    H, E, b, m = orc.seeded_inputs(B, S, D, V, 8)
    H, E = orc.bf16_round(H), orc.bf16_round(E)
    dY = orc.seeded_uniform((B, V), 4)
    Y, I = run_fwd(H, E, b, m)
    f32 = run_bwd(H, E, Y, I, dY)
    bf = run_bwd(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
    assert close(bf[0], f32[0], rtol=1e-2, atol=1e-2) and close(bf[1], f32[1], rtol=1e-2, atol=1e-2)


def test_backward_deterministic(cuda_device):
    B, S, D, V = 4, 128, 256, 3000
    H, E, b, m = orc.seeded_inputs(B, S, D, V, 12, mask_keep=0.9)
    dY = orc.seeded_uniform((B, V), 13)
    Y, I = run_fwd(H, E, b, m)
    a = run_bwd(H, E, Y, I, dY)
    c = run_bwd(H, E, Y, I, dY)
    for x, y in zip(a, c):
        assert x.tobytes() == y.tobytes()


def test_shape_mismatch_rejected(cuda_device):
    from paper_2603_25011_b200 import sparton_backward
    H = t_bf16(np.zeros((2, 3, 8)))
    E = t_bf16(np.zeros((5, 8)))
    Y = torch.zeros((2, 3), device=_dev())
    I = torch.zeros((2, 3), dtype=torch.int32, device=_dev())
    with pytest.raises(ValueError):
        sparton_backward(H, E, Y, I, torch.zeros((2, 5), device=_dev()))


@pytest.mark.parametrize("B,S,D,V", [(512, 512, 768, 30522), (512, 512, 768, 250002), (96, 512, 1024, 250002),
                                     (48, 1024, 768, 30522)])
def test_fullsize_slices_vs_oracle(cuda_device, B, S, D, V):
    """cfg2/cfg3 (and the cfg4 hidden size D=1024; S=1024 takes the gathered
    dE) backward: dH for sampled batch rows and dE/db for sampled vocab
    columns are reproduced exactly by the oracle's separable slices."""
    dev = _dev()
    gen = torch.Generator(device="cuda").manual_seed(1)
    H = torch.randn((B, S, D), generator=gen, device=dev).to(torch.bfloat16)
    E = (torch.randn((V, D), generator=gen, device=dev) * 0.02).to(torch.bfloat16)
    b = torch.zeros(V, device=dev)
    m = torch.ones((B, S), dtype=torch.uint8, device=dev)
    dY = torch.randn((B, V), generator=gen, device=dev)
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    Y, I = sparton_forward(H, E, b, m)
    dH, dE, db = sparton_backward(H, E, Y, I, dY)
    torch.cuda.synchronize()
    Hn, En = H.float().cpu().numpy(), E.float().cpu().numpy()
    Yn, In, dYn = Y.cpu().numpy(), I.cpu().numpy(), dY.cpu().numpy()
    rows = [3, min(400, B - 1)]
    dH_r = orc.backward_rows(Hn, En, Yn, In, dYn, rows)
    assert close(dH[rows].cpu().numpy(), dH_r)
    cols = np.random.default_rng(0).choice(V, 256, replace=False)
    dE_r, db_r = orc.backward_cols(Hn, Yn, In, dYn, cols)
    assert close(dE[cols].cpu().numpy(), dE_r)
    assert close(db[cols].cpu().numpy(), db_r)


@pytest.mark.parametrize("dims", [(3, 300, 256, 3001), (2, 512, 200, 1600), (6, 17, 72, 5000)])
@pytest.mark.parametrize("grad_dtype", [torch.float32, torch.bfloat16])
def test_de_paths_agree(cuda_device, monkeypatch, dims, grad_dtype):
    """The staged dE (H tiles in shared memory) and the gathered dE (per-pair
    bulk copies) accumulate the same fp32 FMAs in the same b order: equal
    results (up to the sign of zero), including db."""
    B, S, D, V = dims
    H, E, b, m = orc.seeded_inputs(B, S, D, V, 77 + S, mask_keep=0.8)
    H, E = orc.bf16_round(H), orc.bf16_round(E)
    dY = orc.seeded_uniform((B, V), 78)
    Y, I = run_fwd(H, E, b, m)
    monkeypatch.setenv("SPARTON_DEV", "1")
    monkeypatch.setenv("SPARTON_DE_STAGED", "1")
    st = run_bwd(H, E, Y, I, dY, grad_dtype=grad_dtype)
    monkeypatch.setenv("SPARTON_DE_STAGED", "0")
    ga = run_bwd(H, E, Y, I, dY, grad_dtype=grad_dtype)
    for x, y in zip(st, ga):
        assert np.array_equal(x, y)


def test_persistent_de_grid_bitwise_equal(cuda_device, monkeypatch):
    """The staged dE with a persistent grid (clusters walking several work items,
    SPARTON_DE_CLUSTERS) produces exactly the one-item-per-cluster result."""
    B, S, D, V = 3, 100, 192, 4000
    H, E, b, m = orc.seeded_inputs(B, S, D, V, 61, mask_keep=0.9)
    H, E = orc.bf16_round(H), orc.bf16_round(E)
    dY = orc.seeded_uniform((B, V), 62)
    Y, I = run_fwd(H, E, b, m)
    ref = run_bwd(H, E, Y, I, dY)
    monkeypatch.setenv("SPARTON_DEV", "1")
    monkeypatch.setenv("SPARTON_DE_CLUSTERS", "2")
    got = run_bwd(H, E, Y, I, dY)
    for x, y in zip(ref, got):
        assert np.array_equal(x, y)
