"""GPU parity on the exact paths the bench credits, plus the reference's
remaining edge behaviours and its concurrency contract.

* bf16 gradients at cfg2/cfg3 (at V=250002 the dH runs 8 vocabulary passes
  through the fp32 ``acc32`` carry) — the path bench.py and the autograd op use;
* the autograd op ``sparton_head(...).backward`` at cfg2/cfg3;
* the forward at cfg4's shape (B=2048, S=512, D=1024, V=250002);
* cfg1's exact reference inputs (``HeadInputs.seeded(Dims(8,128,768,30522), 0,
  mask_keep=0.85)``, dY = seeded_tensor(seed 9), bench.py:293-294), on bf16
  and on the fp32-accuracy path at the reference's own tolerances;
* ±0 ties resolve to the smallest index (fused.py:200; numpy argmax), and
  ``log1p(denormal) > 0`` keeps the pair active (no FTZ, reference.py:96-100);
* the staged/gathered dE boundary (S = 832 / 833) and out-of-range saved
  indices (treated as inactive, never addressed);
* head-owned peak memory flat across S (test_acceptance.py:186-202) and saved
  state independent of S (test_fused.py:154-161);
* concurrent calls from 4 host threads on distinct streams and inputs equal
  the serial results bit for bit (test_fused.py:289-302).

Tolerances: rtol 1e-2 / atol 1e-3 against the oracle on bf16-rounded inputs
(north star); the fp32 path uses the reference's Y rel 1e-5 / abs 1e-7 and
backward 1e-5 (bench.py:41-46).  Argmax exact outside certified near-ties.
"""

from __future__ import annotations

import threading

import numpy as np
import pytest
import torch

from oracle import sparton_oracle as orc

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-2, 1e-3


def _dev():
    return torch.device("cuda", 0)


def close(a, b, rtol=RTOL, atol=ATOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return bool(np.all(np.abs(a - b) <= atol + rtol * np.abs(b)))


def perf_inputs(B, S, D, V, seed=1):
    """bench.py's synthetic distribution (H ~ N(0,1), E ~ N(0, 0.02²), bias 0,
    all-ones mask, dY ~ N(0,1)): every pair active, the backward's worst case."""
    dev = _dev()
    gen = torch.Generator(device="cuda").manual_seed(seed)
    H = torch.randn((B, S, D), generator=gen, device=dev).to(torch.bfloat16)
    E = (torch.randn((V, D), generator=gen, device=dev) * 0.02).to(torch.bfloat16)
    b = torch.zeros(V, device=dev)
    m = torch.ones((B, S), dtype=torch.uint8, device=dev)
    dY = torch.randn((B, V), generator=gen, device=dev)
    return H, E, b, m, dY


def check_grads_sampled(H, E, Y, I, dY, dH, dE, db, rows, ncols=256):
    Hn, En = H.float().cpu().numpy(), E.float().cpu().numpy()
    Yn, In, dYn = Y.detach().cpu().numpy(), I.cpu().numpy(), dY.cpu().numpy()
    dH_r = orc.backward_rows(Hn, En, Yn, In, dYn, rows)
    assert close(dH[rows].float().cpu().numpy(), dH_r), "dH rows"
    cols = np.random.default_rng(0).choice(En.shape[0], ncols, replace=False)
    dE_r, db_r = orc.backward_cols(Hn, Yn, In, dYn, cols)
    assert close(dE[cols].float().cpu().numpy(), dE_r), "dE cols"
    assert close(db[cols].float().cpu().numpy(), db_r), "db cols"


@pytest.mark.parametrize("V", [30522, 250002])
def test_bf16_gradients_fullsize_vs_oracle(cuda_device, V):
    """The bench's backward (grad_dtype=bf16): at V=250002 dH runs in 8 vocab
    passes with partial sums carried in the fp32 workspace (acc32)."""
    from paper_2603_25011_b200 import bwd_workspace_bytes, sparton_backward, sparton_forward
    B, S, D = 512, 512, 768
    H, E, b, m, dY = perf_inputs(B, S, D, V)
    carry = bwd_workspace_bytes(B, S, D, V, torch.bfloat16) - bwd_workspace_bytes(B, S, D, V, torch.float32)
    assert carry == (B * S * D * 4 if V == 250002 else 0)        # the acc32 carry exists only multi-pass
    Y, I = sparton_forward(H, E, b, m)
    dH, dE, db = sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    assert dH.dtype == torch.bfloat16 and dE.dtype == torch.bfloat16
    check_grads_sampled(H, E, Y, I, dY, dH, dE, db, rows=[0, 257, 511])


@pytest.mark.parametrize("V", [30522, 250002])
def test_autograd_head_fullsize_vs_oracle(cuda_device, V):
    """SpartonHeadFn end to end: Y = sparton_head(H, E, b, M); Y.backward(dY)."""
    from paper_2603_25011_b200 import sparton_head
    B, S, D = 512, 512, 768
    H, E, b, m, dY = perf_inputs(B, S, D, V, seed=3)
    H.requires_grad_(True)
    E.requires_grad_(True)
    b.requires_grad_(True)
    Y, I = sparton_head(H, E, b, m, return_indices=True)
    Y.backward(dY)
    torch.cuda.synchronize()
    assert H.grad.dtype == torch.bfloat16 and E.grad.dtype == torch.bfloat16 and b.grad.dtype == torch.float32
    # Forward rows vs oracle as well (the autograd op is the same K1 launch).
    rows = [5, 300]
    Hn = H.detach()[rows].float().cpu().numpy()
    En = E.detach().float().cpu().numpy()
    bn, mn = b.detach().cpu().numpy(), m[rows].cpu().numpy()
    Yr, Ir = orc.forward(Hn, En, bn, mn, vocab_tile=8192, threads=orc.default_threads())
    ok, rep = orc.check_forward(Hn, En, bn, mn, Y.detach()[rows].cpu().numpy(), I[rows].cpu().numpy(), Yr, Ir)
    assert ok, rep
    check_grads_sampled(H.detach(), E.detach(), Y, I, dY, H.grad, E.grad, b.grad, rows=[5, 300])


def test_forward_cfg4_shape_rows_vs_oracle(cuda_device):
    """BASELINE configs[3]'s shape on one GPU: B=2048, S=512, D=1024 (16 K
    steps of 64), V=250002; Y/I of sampled batch rows vs the oracle."""
    from paper_2603_25011_b200 import sparton_forward
    B, S, D, V = 2048, 512, 1024, 250002
    H, E, b, m, _ = perf_inputs(B, S, D, V, seed=4)
    b = (torch.rand(V, device=_dev()) - 0.5) * 0.1       # a nonzero bias on this one
    Y, I = sparton_forward(H, E, b, m)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(Y).all()) and bool((Y >= 0).all())
    assert int(I.min()) >= 0 and int(I.max()) < S
    rows = [0, 1337, 2047]
    Hn = H[rows].float().cpu().numpy()
    En = E.float().cpu().numpy()
    bn, mn = b.cpu().numpy(), m[rows].cpu().numpy()
    Yr, Ir = orc.forward(Hn, En, bn, mn, vocab_tile=8192, threads=orc.default_threads())
    ok, rep = orc.check_forward(Hn, En, bn, mn, Y[rows].cpu().numpy(), I[rows].cpu().numpy(), Yr, Ir)
    assert ok, rep


def _cfg1():
    B, S, D, V = 8, 128, 768, 30522
    H, E, b, m = orc.seeded_inputs(B, S, D, V, 0, mask_keep=0.85)
    dY = orc.seeded_uniform((B, V), 9)
    return H, E, b, m, dY


def test_cfg1_reference_inputs_bf16(cuda_device):
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    H, E, b, m, dY = _cfg1()
    Hb, Eb = orc.bf16_round(H), orc.bf16_round(E)
    dev = _dev()
    Ht = torch.from_numpy(Hb).to(dev).to(torch.bfloat16)
    Et = torch.from_numpy(Eb).to(dev).to(torch.bfloat16)
    Y, I = sparton_forward(Ht, Et, torch.from_numpy(b).to(dev), torch.from_numpy(m).to(dev))
    Yg, Ig = Y.cpu().numpy(), I.cpu().numpy()
    Yr, Ir = orc.forward(Hb, Eb, b, m)
    ok, rep = orc.check_forward(Hb, Eb, b, m, Yg, Ig, Yr, Ir)
    assert ok, rep
    for gd in (torch.float32, torch.bfloat16):
        dH, dE, db = sparton_backward(Ht, Et, Y, I, torch.from_numpy(dY).to(dev), grad_dtype=gd)
        dH_r, dE_r, db_r = orc.backward(Hb, Eb, b, Yg, Ig, dY)
        assert close(dH.float().cpu().numpy(), dH_r) and close(dE.float().cpu().numpy(), dE_r)
        assert close(db.cpu().numpy(), db_r)


def test_cfg1_reference_inputs_fp32_path_at_reference_tolerance(cuda_device):
    """The fp32-accuracy path (exact bf16x3 split) on cfg1's fp32 inputs meets
    the reference's own tolerances against its deterministic oracle."""
    from paper_2603_25011_b200 import sparton_backward_fp32, sparton_forward_fp32
    H, E, b, m, dY = _cfg1()
    dev = _dev()
    Ht, Et = torch.from_numpy(H).to(dev), torch.from_numpy(E).to(dev)
    Y, I = sparton_forward_fp32(Ht, Et, torch.from_numpy(b).to(dev), torch.from_numpy(m).to(dev))
    Yg, Ig = Y.cpu().numpy(), I.cpu().numpy()
    Yr, Ir = orc.forward(H, E, b, m)
    ok, rep = orc.check_forward(H, E, b, m, Yg, Ig, Yr, Ir, rtol=1e-5, atol=1e-7)
    assert ok, rep
    dH, dE, db = sparton_backward_fp32(Ht, Et, Y, I, torch.from_numpy(dY).to(dev))
    dH_r, dE_r, db_r = orc.backward(H, E, b, Yg, Ig, dY)
    # BACKWARD_PAIR_TOL (1e-5 absolute at the reference's desk scale); at cfg1
    # a dH row sums ~240 terms of magnitude ~0.5, so the bound is scaled by |ref|.
    for got, want in ((dH, dH_r), (dE, dE_r), (db, db_r)):
        err = np.abs(got.cpu().numpy().astype(np.float64) - want) - 1e-5 * (1 + np.abs(want))
        assert err.max() <= 0


def _run(H, E, b, m):
    from paper_2603_25011_b200 import sparton_forward
    dev = _dev()
    Y, I = sparton_forward(torch.from_numpy(H).to(dev).to(torch.bfloat16),
                           torch.from_numpy(E).to(dev).to(torch.bfloat16),
                           torch.from_numpy(b).to(dev), torch.from_numpy(m).to(dev))
    return Y.cpu().numpy(), I.cpu().numpy()


def test_signed_zero_ties_take_smallest_index(cuda_device):
    """-0.0 and +0.0 tie (fused.py:200 strict '>', numpy first-occurrence argmax):
    masked positions give (raw)·0 = ±0 by the sign of the raw logit, and an
    unmasked logit can be exactly +0 (x + b with x = -b)."""
    B, S, D, V = 1, 4, 8, 4
    H = np.zeros((B, S, D), np.float32)
    E = np.zeros((V, D), np.float32)
    E[:, 0] = 1.0
    H[0, :, 0] = [-0.5, 1.0, -1.0, -2.0]        # raw dots x_s for every v
    b = np.array([0.0, -1.0, 0.5, -1.0], np.float32)
    m = np.array([[1, 0, 0, 1]], np.uint8)
    # v0: L = [-0.5, +0 (masked +), -0 (masked -), -2]       -> I = 1
    # v1: L = [-1.5, -0 (masked 0·(1-1)=0), -0, -3]           -> I = 1
    # v2: L = [0 (x=-0.5, b=0.5 -> +0), +0, -0, -1.5]         -> I = 0
    # v3: L = [-1.5, +0, -0, -3]                              -> I = 1
    m2 = m.copy()
    Yg, Ig = _run(H, E, b, m2)
    Yr, Ir = orc.forward(H, E, b, m2)
    assert np.array_equal(Ir, [[1, 1, 0, 1]]) and np.array_equal(Ig, Ir)
    assert np.all(Yg == 0) and np.all(Yr == 0)
    # Exact unmasked +0 ahead of masked ±0 and behind it.
    H[0, :, 0] = [3.0, 1.0, -4.0, 1.0]
    b = np.full(V, -1.0, np.float32)
    m3 = np.array([[0, 1, 0, 1]], np.uint8)          # s0 masked (+0), s1 x+b = +0, s3 x+b = +0
    Yg, Ig = _run(H, E, b, m3)
    Yr, Ir = orc.forward(H, E, b, m3)
    assert np.array_equal(Ig, Ir) and np.all(Ir == 0)


def test_denormal_logit_counts_as_active(cuda_device):
    """log1p(denormal) > 0 (reference.py:96-100): no flush-to-zero, so a
    denormal maximum gives Y > 0 and the pair sends gradient (db = Σ dY)."""
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    B, S, D, V = 3, 5, 8, 7
    dev = _dev()
    den = np.float32(1e-40)
    assert 0 < den < np.finfo(np.float32).tiny
    H = torch.zeros((B, S, D), dtype=torch.bfloat16, device=dev)
    E = torch.ones((V, D), dtype=torch.bfloat16, device=dev)
    b = torch.full((V,), float(den), device=dev)
    m = torch.ones((B, S), dtype=torch.uint8, device=dev)
    Y, I = sparton_forward(H, E, b, m)
    Yr, Ir = orc.forward(np.zeros((B, S, D), np.float32), np.ones((V, D), np.float32),
                         np.full(V, den, np.float32), np.ones((B, S), np.uint8))
    assert np.all(Yr > 0)
    Yg = Y.cpu().numpy()
    assert np.all(Yg > 0) and np.allclose(Yg, Yr, rtol=1e-3, atol=0) and np.array_equal(I.cpu().numpy(), Ir)
    dY = torch.rand((B, V), device=dev) + 0.5
    dH, dE, db = sparton_backward(H, E, Y, I, dY)
    dYn = dY.cpu().numpy()
    _, _, db_r = orc.backward(np.zeros((B, S, D), np.float32), np.ones((V, D), np.float32),
                              np.full(V, den, np.float32), Yr, Ir, dYn)
    assert np.allclose(db.cpu().numpy(), db_r, rtol=1e-6) and np.all(db_r > 0)
    # dH[b, 0, :] = Σ_v g·E[v] = Σ_v dY[b, v] (E = 1, exp(-Y) = 1)
    assert np.allclose(dH[:, 0, 0].cpu().numpy(), dYn.sum(1), rtol=1e-5)


@pytest.mark.parametrize("S", [832, 833])
def test_staged_de_boundary_vs_oracle(cuda_device, S):
    """S = 832 is the staged dE's largest sequence (two 4-CTA stages of R=208
    rows fit 227 KB); S = 833 takes the gathered dE."""
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    B, D, V = 3, 64, 2500
    H, E, b, m = orc.seeded_inputs(B, S, D, V, 40 + S, mask_keep=0.9)
    H, E = orc.bf16_round(H), orc.bf16_round(E)
    dY = orc.seeded_uniform((B, V), 41)
    dev = _dev()
    Ht = torch.from_numpy(H).to(dev).to(torch.bfloat16)
    Et = torch.from_numpy(E).to(dev).to(torch.bfloat16)
    Y, I = sparton_forward(Ht, Et, torch.from_numpy(b).to(dev), torch.from_numpy(m).to(dev))
    for gd in (torch.float32, torch.bfloat16):
        dH, dE, db = sparton_backward(Ht, Et, Y, I, torch.from_numpy(dY).to(dev), grad_dtype=gd)
        dH_r, dE_r, db_r = orc.backward(H, E, b, Y.cpu().numpy(), I.cpu().numpy(), dY)
        assert close(dH.float().cpu().numpy(), dH_r) and close(dE.float().cpu().numpy(), dE_r)
        assert close(db.cpu().numpy(), db_r)


@pytest.mark.parametrize("S", [300, 1000])
def test_out_of_range_indices_are_inactive(cuda_device, S):
    """Saved indices outside [0, S) (state from another forward) never address
    memory: those pairs contribute nothing, exactly as if Y were 0."""
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    B, D, V = 4, 128, 3000
    H, E, b, m = orc.seeded_inputs(B, S, D, V, 17, mask_keep=0.9)
    H, E = orc.bf16_round(H), orc.bf16_round(E)
    dY = orc.seeded_uniform((B, V), 18)
    dev = _dev()
    Ht = torch.from_numpy(H).to(dev).to(torch.bfloat16)
    Et = torch.from_numpy(E).to(dev).to(torch.bfloat16)
    Y, I = sparton_forward(Ht, Et, torch.from_numpy(b).to(dev), torch.from_numpy(m).to(dev))
    Yn, In = Y.cpu().numpy(), I.cpu().numpy()
    rng = np.random.default_rng(3)
    bad = rng.random((B, V)) < 0.05
    In_bad = In.copy()
    In_bad[bad] = np.where(rng.random(bad.sum()) < 0.5, S + 7, -3)
    Y0 = Yn.copy()
    Y0[bad] = 0.0
    dYt = torch.from_numpy(dY).to(dev)
    got = sparton_backward(Ht, Et, Y, torch.from_numpy(In_bad).to(dev), dYt)
    want = sparton_backward(Ht, Et, torch.from_numpy(Y0).to(dev), I, dYt)
    for x, y in zip(got, want):
        assert torch.equal(x, y)


def test_peak_memory_flat_across_S(cuda_device):
    """GPU analogue of test_acceptance.py:186-202 and test_fused.py:154-161:
    the forward's head-owned allocation (only Y and I; the kernel never
    allocates) and the saved state are identical for every S; the backward's
    head-owned peak is its outputs plus the documented workspace."""
    from paper_2603_25011_b200 import bwd_workspace_bytes, sparton_backward, sparton_forward
    B, D, V = 64, 768, 30522
    dev = _dev()
    fwd_peaks, saved = {}, {}
    for S in (128, 256, 512, 1024):
        H, E, b, m, dY = perf_inputs(B, S, D, V, seed=S)
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated(dev)
        torch.cuda.reset_peak_memory_stats(dev)
        Y, I = sparton_forward(H, E, b, m)
        torch.cuda.synchronize()
        fwd_peaks[S] = torch.cuda.max_memory_allocated(dev) - base
        saved[S] = Y.numel() * Y.element_size() + I.numel() * I.element_size()
        base = torch.cuda.memory_allocated(dev)
        torch.cuda.reset_peak_memory_stats(dev)
        dH, dE, db = sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
        torch.cuda.synchronize()
        bwd_peak = torch.cuda.max_memory_allocated(dev) - base
        outputs = dH.numel() * 2 + dE.numel() * 2 + db.numel() * 4
        ws = bwd_workspace_bytes(B, S, D, V, torch.bfloat16)
        assert bwd_peak <= outputs + ws + 4 * (2 << 20), (S, bwd_peak, outputs, ws)
        del H, E, b, m, dY, Y, I, dH, dE, db
    assert len(set(fwd_peaks.values())) == 1, fwd_peaks
    assert set(saved.values()) == {B * V * 8}
    assert fwd_peaks[128] <= B * V * 8 + (4 << 20)


def test_concurrent_threads_match_serial_bitwise(cuda_device):
    """test_fused.py:289-302 on the GPU: 4 host threads, each on its own CUDA
    stream with distinct inputs, run forward + backward (the staged dE's
    side stream included) concurrently; every result equals the serial run."""
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    dev = _dev()
    jobs = []
    for i in range(8):
        H, E, b, m = orc.seeded_inputs(3, 200 + 37 * i, 256, 4000 + 500 * i, 900 + i, mask_keep=0.8)
        dY = orc.seeded_uniform((3, 4000 + 500 * i), 950 + i)
        jobs.append(tuple(torch.from_numpy(x).to(dev) for x in (H, E, b, m, dY)))

    def run(job):
        H, E, b, m, dY = job
        Y, I = sparton_forward(H.to(torch.bfloat16), E.to(torch.bfloat16), b, m)
        g = sparton_backward(H.to(torch.bfloat16), E.to(torch.bfloat16), Y, I, dY, grad_dtype=torch.bfloat16)
        return [t.cpu() for t in (Y, I, *g)]

    serial = [run(j) for j in jobs]
    torch.cuda.synchronize()
    results = [None] * len(jobs)
    errors = []

    def worker(tid):
        try:
            s = torch.cuda.Stream(device=dev)
            with torch.cuda.stream(s):
                for rep in range(3):
                    for k in range(tid, len(jobs), 4):
                        out = run(jobs[k])
                        if rep == 2:
                            results[k] = out
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for a, c in zip(serial, results):
        for x, y in zip(a, c):
            assert torch.equal(x, y)


def test_concurrent_calls_with_different_smem_sizes(cuda_device):
    """Concurrent backwards whose staged dE / route launches need different
    dynamic shared memory (S = 64 ... 832): the per-function smem limit is a
    constant, so no thread can lower it between another thread's set and
    launch (a failed launch would raise; results equal the serial run)."""
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    dev = _dev()
    jobs = []
    for i, S in enumerate((64, 832, 128, 700, 257, 512, 96, 800)):
        H, E, b, m = orc.seeded_inputs(2, S, 128, 3000, 70 + i, mask_keep=0.9)
        dY = orc.seeded_uniform((2, 3000), 170 + i)
        jobs.append(tuple(torch.from_numpy(x).to(dev) for x in (H, E, b, m, dY)))
    fwd = [sparton_forward(j[0].to(torch.bfloat16), j[1].to(torch.bfloat16), j[2], j[3]) for j in jobs]

    def run(k):
        H, E, b, m, dY = jobs[k]
        Y, I = fwd[k]
        return [t.cpu() for t in sparton_backward(H.to(torch.bfloat16), E.to(torch.bfloat16), Y, I, dY)]

    serial = [run(k) for k in range(len(jobs))]
    errors, mism = [], []

    def worker(tid):
        try:
            s = torch.cuda.Stream(device=dev)
            with torch.cuda.stream(s):
                for rep in range(12):
                    k = (tid + rep) % len(jobs)
                    out = run(k)
                    if not all(torch.equal(x, y) for x, y in zip(out, serial[k])):
                        mism.append((tid, rep, k))
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert not mism, mism
