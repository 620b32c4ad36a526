"""MXFP8 forward — SURVEY.md §8f rank 4: tcgen05 block-scaled MXFP8.

e4m3 operands with one ue8m0 scale per 32 K elements of every row (OCP MX),
the scales applied inside the MMA (kind::mxf8f6f4.block_scale).  Checked
exactly where it can be: (1) the quantiser matches a torch restatement bit
for bit (the scale exponent rule, torch's e4m3 rounding, the tcgen05.cp scale
layout); (2) the kernel on quantised operands matches the oracle run on the
*dequantised* operands (products of scaled e4m3 values are exact in fp32, so
only the accumulation order differs): Y within rtol 1e-2 / atol 1e-3 and I
exact outside certified near-ties, across full / narrow / packed sequence
chunks (240 positions each).  Against bf16 the gap is reported.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import sparton_oracle as orc

pytestmark = pytest.mark.gpu


def _mx_reference(x: torch.Tensor):
    """Restated MX quantisation: per 32-element block, e = the smallest
    integer with amax / 2^e <= 448; q = e4m3_rn(x / 2^e) (torch's
    float8_e4m3fn conversion); returns (q bytes, e) with e shaped (rows, nblk)."""
    D = x.shape[-1]
    xf = x.float().reshape(-1, D)
    nblk = -(-D // 32)
    pad = torch.zeros((xf.shape[0], nblk * 32), device=x.device)
    pad[:, :D] = xf
    amax = pad.reshape(xf.shape[0], nblk, 32).abs().amax(dim=2)
    m, ex = torch.frexp(amax)
    e = ex - 9 + (torch.ldexp(amax, 9 - ex) > 448.0).to(torch.int32)
    e = torch.where(amax > 0, e, torch.full_like(e, -127)).clamp(-127, 127)
    scale = torch.exp2(-e.float()).repeat_interleave(32, dim=1)[:, :D]
    q = (xf * scale).to(torch.float8_e4m3fn).view(torch.uint8).reshape(x.shape)
    return q, e


@pytest.mark.parametrize("shape,op", [((3, 300, 768), "H"), ((8, 32, 64), "H"), ((5, 48, 80), "H"),
                                      ((2, 512, 1024), "H"), ((1000, 768), "E"), ((129, 80), "E")])
def test_mx_quantizer_matches_restatement(cuda_device, shape, op):
    from paper_2603_25011_b200 import quantize_mx
    from paper_2603_25011_b200.head import mx_scale_index
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(shape, generator=g, device="cuda")
    # heterogeneous block magnitudes: what block scaling is for
    x = x * torch.exp2(torch.randint(-6, 7, shape[:-1] + (1,), generator=g, device="cuda").float())
    x = x.to(torch.bfloat16)
    q, sf = quantize_mx(x, op)
    q_ref, e_ref = _mx_reference(x)
    assert torch.equal(q, q_ref)
    idx = mx_scale_index(shape, op).cuda()
    assert torch.equal(sf.to(torch.int64)[idx], (e_ref + 127).to(torch.int64))


def _inputs(B, S, D, V, seed, mask_keep=0.85):
    H, E, b, m = orc.seeded_inputs(B, S, D, V, seed, mask_keep=mask_keep)
    b = (b * 0.5).astype(np.float32)
    return H, E, b, m


@pytest.mark.parametrize("dims", [
    (2, 512, 768, 3001),     # chunks of 240, 240, 32 (narrow last chunk)
    (3, 240, 256, 1000),     # one full chunk
    (4, 300, 128, 700),      # 240 + 60
    (8, 32, 64, 500),        # packed: 7 batch rows per chunk
    (5, 48, 256, 600),       # packed: 5 rows, 32-column groups straddle rows
    (16, 100, 1024, 2000),   # packed: 2 rows
    (2, 200, 80, 300),       # D = 80: a 16-element tail block, zero-filled K stage
    (3, 1000, 256, 900),     # long sequence: 5 chunks
])
def test_mx_forward_vs_oracle_on_dequantised_inputs(cuda_device, dims):
    from paper_2603_25011_b200 import dequantize_mx, sparton_forward_mx
    B, S, D, V = dims
    H, E, b, m = _inputs(B, S, D, V, 17 + S + D)
    Ht = torch.from_numpy(H).cuda().to(torch.bfloat16)
    Et = torch.from_numpy(E).cuda().to(torch.bfloat16)
    bt = torch.from_numpy(b).cuda()
    mt = torch.from_numpy(m).cuda()
    (Y, I), (qH, sH, qE, sE) = sparton_forward_mx(Ht, Et, bt, mt, return_quantized=True)
    torch.cuda.synchronize()
    Hd = dequantize_mx(qH, sH, "H").cpu().numpy()
    Ed = dequantize_mx(qE, sE, "E").cpu().numpy()
    Yr, Ir = orc.forward(Hd, Ed, b, m)
    ok, rep = orc.check_forward(Hd, Ed, b, m, Y.cpu().numpy(), I.cpu().numpy(), Yr, Ir, rtol=1e-2, atol=1e-3)
    assert ok, rep


def test_mx_forward_full_size_rows_vs_oracle(cuda_device):
    """cfg3-shaped forward (V = 250002, B = 4 rows): sampled vocab columns of
    every row against the oracle on the dequantised operands."""
    from paper_2603_25011_b200 import dequantize_mx, sparton_forward_mx
    g = torch.Generator(device="cuda").manual_seed(5)
    B, S, D, V = 4, 512, 768, 250002
    H = torch.randn((B, S, D), generator=g, device="cuda").to(torch.bfloat16)
    E = (torch.randn((V, D), generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    b = torch.zeros(V, device="cuda")
    m = torch.ones((B, S), dtype=torch.uint8, device="cuda")
    (Y, I), (qH, sH, qE, sE) = sparton_forward_mx(H, E, b, m, return_quantized=True)
    cols = torch.randperm(V, generator=torch.Generator().manual_seed(1))[:2048].sort().values
    Hd = dequantize_mx(qH, sH, "H").cpu().numpy()
    Ed = dequantize_mx(qE, sE, "E")[cols.cuda()].cpu().numpy()
    bn, mn = b[cols.cuda()].cpu().numpy(), m.cpu().numpy()
    Yr, Ir = orc.forward(Hd, Ed, bn, mn)
    ok, rep = orc.check_forward(Hd, Ed, bn, mn, Y[:, cols.cuda()].cpu().numpy(), I[:, cols.cuda()].cpu().numpy(),
                                Yr, Ir, rtol=1e-2, atol=1e-3)
    assert ok, rep


def test_mx_vs_bf16_and_per_tensor_fp8(cuda_device):
    """The gap to bf16, next to the per-tensor e4m3 path's (reported)."""
    from paper_2603_25011_b200 import sparton_forward, sparton_forward_fp8, sparton_forward_mx
    g = torch.Generator(device="cuda").manual_seed(3)
    B, S, D, V = 8, 512, 768, 30522
    H = torch.randn((B, S, D), generator=g, device="cuda")
    H = (H * torch.exp2(torch.randint(-3, 4, (B, S, 1), generator=g, device="cuda").float())).to(torch.bfloat16)
    E = (torch.randn((V, D), generator=g, device="cuda") * 0.02).to(torch.bfloat16)
    b = torch.zeros(V, device="cuda")
    m = torch.ones((B, S), dtype=torch.uint8, device="cuda")
    Y16, I16 = sparton_forward(H, E, b, m)
    out = {}
    for name, fn in (("mx", sparton_forward_mx), ("fp8", sparton_forward_fp8)):
        Y8, I8 = fn(H, E, b, m)
        out[name] = (float(((Y8 - Y16).abs() / Y16.abs().clamp_min(1e-3)).median()),
                     float((I8 == I16).float().mean()))
    print("vs bf16 (median rel |dY|, argmax agreement):", out)
    assert out["mx"][0] < 0.05 and out["mx"][1] > 0.5


def test_mx_autograd_head(cuda_device):
    """SpartonHeadMxFn: MX forward, bf16 backward at the MX forward's (Y, I)."""
    from paper_2603_25011_b200 import sparton_backward, sparton_forward_mx, sparton_head_mx
    g = torch.Generator(device="cuda").manual_seed(9)
    B, S, D, V = 3, 300, 256, 4000
    H = torch.randn((B, S, D), generator=g, device="cuda").to(torch.bfloat16).requires_grad_()
    E = (torch.randn((V, D), generator=g, device="cuda") * 0.05).to(torch.bfloat16).requires_grad_()
    b = torch.zeros(V, device="cuda", requires_grad=True)
    m = torch.ones((B, S), dtype=torch.uint8, device="cuda")
    Y, I = sparton_head_mx(H, E, b, m)
    Y0, I0 = sparton_forward_mx(H.detach(), E.detach(), b.detach(), m)
    assert torch.equal(Y, Y0) and torch.equal(I, I0)
    dY = torch.randn((B, V), generator=g, device="cuda")
    Y.backward(dY)
    dH, dE, db = sparton_backward(H.detach(), E.detach(), Y0, I0, dY, grad_dtype=torch.bfloat16)
    assert torch.equal(H.grad, dH) and torch.equal(E.grad, dE.to(E.dtype)) and torch.equal(b.grad, db)
