"""Torch-facing Sparton head: functional forward/backward and the autograd.Function.

The reference has no torch API; this is the GPU-native form of
its operator pair ``forward_fully_fused`` / ``backward_fused``
(/root/reference/pkg/src/fusedhead/fused.py:160-212, :215-278).  Torch is
plumbing here: it owns device memory (caching allocator, so peak-HBM numbers
stay in torch's accounting) and streams; every byte of arithmetic runs in the
sm_100a kernels behind the C ABI (``_lib``).  There is no CPU path: non-CUDA
tensors raise.

State kept for backward is exactly (Y, I) — B·V·(4+4) bytes, independent of S —
plus references to the inputs H and E (SavedSparseState, fused.py:67-80).
"""

from __future__ import annotations

import torch

from . import _lib

__all__ = [
    "sparton_forward",
    "sparton_forward_fp8",
    "sparton_forward_mx",
    "quantize_mx",
    "dequantize_mx",
    "quantize_e4m3",
    "sparton_backward",
    "sparton_forward_fp32",
    "sparton_backward_fp32",
    "sparton_backward_fp8",
    "SpartonHeadFp8Fn",
    "sparton_head_fp8",
    "SpartonHeadMxFn",
    "sparton_head_mx",
    "split_bf16x3",
    "SpartonHeadFn",
    "sparton_head",
    "bwd_workspace_bytes",
]


def _stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def _require_cuda(name: str, t: torch.Tensor) -> None:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor, got {type(t).__name__}")
    if not t.is_cuda:
        raise RuntimeError(
            f"{name} is on {t.device}: the sparton head runs only on CUDA (sm_100a); there is no CPU fallback")


def _pad_hidden(x: torch.Tensor) -> torch.Tensor:
    """Zero-pad the hidden axis to a multiple of 8 (TMA stride rule); zero K
    columns add exactly 0 to every dot product."""
    d = x.shape[-1]
    if d % 8 == 0:
        return x
    return torch.nn.functional.pad(x, (0, 8 - d % 8))


def _check_inputs(H, E, bias, mask):
    for name, t in (("H", H), ("E", E), ("bias", bias), ("mask", mask)):
        _require_cuda(name, t)
    if H.dim() != 3:
        raise ValueError(f"H must be (B, S, D), got shape {tuple(H.shape)}")
    B, S, D = H.shape
    if E.dim() != 2 or E.shape[1] != D:
        raise ValueError(f"E must be (V, {D}), got shape {tuple(E.shape)}")
    V = E.shape[0]
    if H.dtype != torch.bfloat16 or E.dtype != torch.bfloat16:
        raise ValueError(f"H and E must be bfloat16, got {H.dtype} and {E.dtype}")
    if bias.shape != (V,) or bias.dtype != torch.float32:
        raise ValueError(f"bias must be float32 of shape ({V},), got {bias.dtype} {tuple(bias.shape)}")
    if mask.shape != (B, S) or mask.dtype not in (torch.uint8, torch.bool):
        raise ValueError(f"mask must be uint8/bool of shape ({B}, {S}), got {mask.dtype} {tuple(mask.shape)}")
    if min(B, S, D, V) < 1:
        raise ValueError(f"all dims must be positive, got B={B} S={S} D={D} V={V}")
    return B, S, D, V


@torch.no_grad()
def sparton_forward(H: torch.Tensor, E: torch.Tensor, bias: torch.Tensor, mask: torch.Tensor,
                    *, cta_group: int = 0, out: tuple[torch.Tensor, torch.Tensor] | None = None,
                    extra_out: tuple[tuple[int, int], ...] = (), multicast_out: tuple[int, int] | None = None
                    ) -> tuple[torch.Tensor, torch.Tensor]:
    """Fused head forward: returns (Y f32 [B, V], I int32 [B, V]).

    Y[b,v] = log1p(relu(max_s((H[b,s]·E[v] + bias[v]) · mask[b,s]))), I = first argmax.
    The B×S×V logits are never materialised.  ``out`` may be column views of
    wider row-major buffers (unit column stride, Y and I sharing a row
    stride).  ``extra_out`` lists up to 7 more (Y, I) device addresses (raw
    pointers, same row stride as ``out``) that receive identical stores —
    the peers' copies of a vocab-sharded head's output (``sparton_fwd_multi``).
    ``multicast_out`` = (Y, I) NVLS multicast addresses of the same columns
    (row stride of ``out``): results are stored there with multimem.st only —
    the switch writes every rank's copy, ``out`` included
    (``sparton_fwd_multicast``).
    """
    B, S, D, V = _check_inputs(H, E, bias, mask)
    Hp = _pad_hidden(H.contiguous()).reshape(B * S, -1)
    Ep = _pad_hidden(E.contiguous())
    Dp = Hp.shape[1]
    m = mask.contiguous()
    if m.dtype == torch.bool:
        m = m.view(torch.uint8)
    bias = bias.contiguous()
    if out is None:
        Y = torch.empty((B, V), dtype=torch.float32, device=H.device)
        I = torch.empty((B, V), dtype=torch.int32, device=H.device)
    else:
        Y, I = out
        if Y.shape != (B, V) or I.shape != (B, V) or Y.dtype != torch.float32 or I.dtype != torch.int32:
            raise ValueError("out must be (Y float32 [B,V], I int32 [B,V])")
    ldY = Y.stride(0)
    if Y.stride(1) != 1 or I.stride(1) != 1 or I.stride(0) != ldY:
        raise ValueError("Y and I must share a row stride with unit column stride")
    lib = _lib.load()
    if multicast_out is not None and extra_out:
        raise ValueError("multicast_out and extra_out are exclusive")
    with torch.cuda.device(H.device):
        if multicast_out is not None:
            rc = lib.sparton_fwd_multicast(Hp.data_ptr(), Ep.data_ptr(), bias.data_ptr(), m.data_ptr(),
                                           int(multicast_out[0]), int(multicast_out[1]), B, S, Dp, V, ldY,
                                           int(cta_group), _stream_ptr())
        elif extra_out:
            import ctypes
            n = 1 + len(extra_out)
            ys = (ctypes.c_void_p * n)(Y.data_ptr(), *[int(y) for y, _ in extra_out])
            is_ = (ctypes.c_void_p * n)(I.data_ptr(), *[int(i) for _, i in extra_out])
            rc = lib.sparton_fwd_multi(Hp.data_ptr(), Ep.data_ptr(), bias.data_ptr(), m.data_ptr(), n, ys, is_,
                                       B, S, Dp, V, ldY, int(cta_group), _stream_ptr())
        else:
            rc = lib.sparton_fwd(Hp.data_ptr(), Ep.data_ptr(), bias.data_ptr(), m.data_ptr(),
                                 Y.data_ptr(), I.data_ptr(), B, S, Dp, V, ldY, int(cta_group), _stream_ptr())
    _lib.check(rc)
    return Y, I


@torch.no_grad()
def quantize_e4m3(x: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Per-tensor e4m3 quantisation on the GPU: returns (q uint8 view of e4m3
    values shaped like x, amax float32 scalar tensor); x ~= q * amax / 448."""
    _require_cuda("x", x)
    if x.dtype != torch.bfloat16:
        raise ValueError(f"x must be bfloat16, got {x.dtype}")
    xc = x.contiguous()
    n = xc.numel()
    if n % 16:
        raise ValueError("numel must be a multiple of 16")
    q = torch.empty(xc.shape, dtype=torch.uint8, device=x.device)
    amax = torch.empty((), dtype=torch.float32, device=x.device)
    lib = _lib.load()
    with torch.cuda.device(x.device):
        rc = lib.sparton_quantize_e4m3(xc.data_ptr(), n, q.data_ptr(), amax.data_ptr(), _stream_ptr())
    _lib.check(rc)
    return q, amax


@torch.no_grad()
def sparton_forward_fp8(H: torch.Tensor, E: torch.Tensor, bias: torch.Tensor, mask: torch.Tensor, *,
                        E_q: tuple[torch.Tensor, torch.Tensor] | None = None, cta_group: int = 0,
                        return_quantized: bool = False):
    """FP8 (e4m3) variant of the fused forward — tcgen05 kind::f8f6f4 at twice
    the bf16 tensor rate; the paper's future-work item.

    H and E (bf16) are quantised per tensor on the GPU (``E_q`` may pass a
    cached ``quantize_e4m3(E)``).  Y/I follow the same definition as
    ``sparton_forward`` on the dequantised operands; they are approximate
    relative to bf16 (e4m3 keeps 3 mantissa bits).  ``return_quantized``
    also returns (qH, amax_h, qE, amax_e) for ``sparton_backward_fp8``."""
    B, S, D, V = _check_inputs(H, E, bias, mask)
    if D % 16:
        raise ValueError("the e4m3 forward needs D to be a multiple of 16")
    qH, aH = quantize_e4m3(H)
    qE, aE = E_q if E_q is not None else quantize_e4m3(E)
    m = mask.contiguous()
    if m.dtype == torch.bool:
        m = m.view(torch.uint8)
    bias = bias.contiguous()
    Y = torch.empty((B, V), dtype=torch.float32, device=H.device)
    I = torch.empty((B, V), dtype=torch.int32, device=H.device)
    out = _fwd_fp8_launch(qH, aH, qE, aE, bias, m, Y, I, cta_group)
    return (out, (qH, aH, qE, aE)) if return_quantized else out


def _fwd_fp8_launch(qH, aH, qE, aE, bias, m, Y, I, cta_group=0):
    B, V = Y.shape
    S, D = qH.shape[1], qH.shape[2]
    lib = _lib.load()
    with torch.cuda.device(qH.device):
        rc = lib.sparton_fwd_fp8(qH.data_ptr(), qE.data_ptr(), aH.data_ptr(), aE.data_ptr(), bias.data_ptr(),
                                 m.data_ptr(), Y.data_ptr(), I.data_ptr(), B, S, D, V, V, int(cta_group),
                                 _stream_ptr())
    _lib.check(rc)
    return Y, I


@torch.no_grad()
def quantize_mx(x: torch.Tensor, operand: str) -> tuple[torch.Tensor, torch.Tensor]:
    """MXFP8 quantisation on the GPU (OCP MX, e4m3 elements, one ue8m0 scale
    per 32 consecutive elements of a row): returns (q uint8 view of e4m3
    values shaped like x, sf uint8 scale bytes in the forward's tcgen05.cp
    layout).  ``operand`` "H" for a (B, S, D) hidden-state tensor, "E" for the
    (V, D) vocabulary matrix.  x ~= q * 2^(sf - 127) blockwise."""
    _require_cuda("x", x)
    if x.dtype != torch.bfloat16:
        raise ValueError(f"x must be bfloat16, got {x.dtype}")
    if operand == "H":
        if x.dim() != 3:
            raise ValueError("H must be (B, S, D)")
        (B, S, D), V, op = x.shape, 1, _lib.SPARTON_MX_H
    elif operand == "E":
        if x.dim() != 2:
            raise ValueError("E must be (V, D)")
        (V, D), B, S, op = x.shape, 1, 1, _lib.SPARTON_MX_E
    else:
        raise ValueError(f"operand must be 'H' or 'E', got {operand!r}")
    lib = _lib.load()
    nsf = int(lib.sparton_mx_scales_bytes(B, S, D, V, op))
    if nsf <= 0:
        raise ValueError(f"bad shape {tuple(x.shape)}")
    xc = x.contiguous()
    q = torch.empty(xc.shape, dtype=torch.uint8, device=x.device)
    sf = torch.empty(nsf, dtype=torch.uint8, device=x.device)
    with torch.cuda.device(x.device):
        rc = lib.sparton_quantize_mx(xc.data_ptr(), B, S, D, V, op, q.data_ptr(), sf.data_ptr(), nsf,
                                     _stream_ptr())
    _lib.check(rc)
    return q, sf


def mx_scale_index(shape, operand: str, S: int | None = None):
    """Host-side restatement of the scale layout (sparton_quant_mx_kernel):
    for every (row, 32-element block) of x, the byte offset of its scale in
    ``sf``.  Returns an int64 tensor of shape (rows, ceil(D / 32)).  Used by
    ``dequantize_mx`` and the tests."""
    if operand == "H":
        B, S_, D = shape
        rows = B * S_
        sn = 240
        pack = sn // S_ if (16 <= S_ <= 128 and sn // S_ > 1) else 1
        group, chunk, spg, slot_rows = pack * S_, sn, (1 if pack > 1 else -(-S_ // sn)), 256
    else:
        V, D = shape
        rows, group, chunk, spg, slot_rows = V, 128, 128, 1, 128
    nkg = -(-D // 128)
    r = torch.arange(rows, dtype=torch.int64).unsqueeze(1)
    blk = torch.arange(-(-D // 32), dtype=torch.int64).unsqueeze(0)
    g, within = r // group, r % group
    slot, i = g * spg + within // chunk, within % chunk
    return (((slot * nkg + blk // 4) * (slot_rows // 128) + i // 128) * 512 + (i % 32) * 16 +
            ((i % 128) // 32) * 4 + blk % 4)


def dequantize_mx(q: torch.Tensor, sf: torch.Tensor, operand: str) -> torch.Tensor:
    """float32 values of an MX-quantised operand: q (e4m3 bytes) x 2^(sf-127)."""
    shape = tuple(q.shape)
    D = shape[-1]
    vals = q.view(torch.float8_e4m3fn).float().reshape(-1, D)
    idx = mx_scale_index(shape, operand).to(q.device)
    e = sf.to(torch.int64)[idx].float() - 127.0                 # (rows, nblk)
    scale = torch.exp2(e).repeat_interleave(32, dim=1)[:, :D]
    return (vals * scale).reshape(shape)


@torch.no_grad()
def sparton_forward_mx(H: torch.Tensor, E: torch.Tensor, bias: torch.Tensor, mask: torch.Tensor, *,
                       E_q: tuple[torch.Tensor, torch.Tensor] | None = None, return_quantized: bool = False):
    """MXFP8 variant of the fused forward: H and E
    quantised with per-32-element ue8m0 block scales (``quantize_mx``), the
    tensor cores apply the scales (tcgen05.mma kind::mxf8f6f4.block_scale).
    Y/I follow the definition of ``sparton_forward`` on the dequantised
    operands.  ``E_q`` may pass a cached ``quantize_mx(E, "E")``;
    ``return_quantized`` also returns (qH, sfH, qE, sfE)."""
    B, S, D, V = _check_inputs(H, E, bias, mask)
    if D % 16:
        raise ValueError("the MXFP8 forward needs D to be a multiple of 16")
    qH, sH = quantize_mx(H, "H")
    qE, sE = E_q if E_q is not None else quantize_mx(E, "E")
    m = mask.contiguous()
    if m.dtype == torch.bool:
        m = m.view(torch.uint8)
    bias = bias.contiguous()
    Y = torch.empty((B, V), dtype=torch.float32, device=H.device)
    I = torch.empty((B, V), dtype=torch.int32, device=H.device)
    lib = _lib.load()
    with torch.cuda.device(H.device):
        rc = lib.sparton_fwd_mx(qH.data_ptr(), sH.data_ptr(), qE.data_ptr(), sE.data_ptr(), bias.data_ptr(),
                                m.data_ptr(), Y.data_ptr(), I.data_ptr(), B, S, D, V, V, _stream_ptr())
    _lib.check(rc)
    return ((Y, I), (qH, sH, qE, sE)) if return_quantized else (Y, I)


@torch.no_grad()
def sparton_backward_fp8(qH: torch.Tensor, amax_h: torch.Tensor, qE: torch.Tensor, amax_e: torch.Tensor,
                         Y: torch.Tensor, I: torch.Tensor, dY: torch.Tensor, *, include_bias_grad: bool = True,
                         grad_dtype: torch.dtype = torch.bfloat16
                         ) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Backward of the FP8 forward: the argmax-routed gradients with the e4m3
    operands the forward multiplied (``quantize_e4m3`` outputs: qH [B,S,D]
    and qE [V,D] bytes, amax scalars; value = q * amax / 448).  dE gathers
    staged e4m3 H rows and dH gathers e4m3 E rows — half the bytes of the
    bf16 backward — with fp32 accumulation in the reference's order, and the
    dequantisation scale applied once per output element.  This is the
    straight-through gradient of ``sparton_forward_fp8``; S <= 832."""
    for name, t in (("qH", qH), ("qE", qE), ("amax_h", amax_h), ("amax_e", amax_e), ("Y", Y), ("I", I),
                    ("dY", dY)):
        _require_cuda(name, t)
    if qH.dim() != 3 or qE.dim() != 2 or qE.shape[1] != qH.shape[2]:
        raise ValueError("qH must be (B, S, D) and qE (V, D)")
    if qH.dtype != torch.uint8 or qE.dtype != torch.uint8:
        raise ValueError("qH and qE must hold e4m3 bytes (uint8, from quantize_e4m3)")
    B, S, D = qH.shape
    V = qE.shape[0]
    if Y.shape != (B, V) or I.shape != (B, V) or dY.shape != (B, V):
        raise ValueError(f"saved state and dY must have shape {(B, V)}")
    if Y.dtype != torch.float32 or I.dtype != torch.int32 or dY.dtype != torch.float32:
        raise ValueError("Y/dY must be float32 and I int32")
    if grad_dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("grad_dtype must be torch.float32 or torch.bfloat16")
    qH, qE = qH.contiguous(), qE.contiguous()
    if Y.stride(1) != 1 or I.stride(1) != 1 or I.stride(0) != Y.stride(0) or Y.stride(0) < V:
        Y, I = Y.contiguous(), I.contiguous()
    if dY.stride(1) != 1 or dY.stride(0) < V:
        dY = dY.contiguous()
    dev = qH.device
    dH = torch.empty((B, S, D), dtype=grad_dtype, device=dev)
    dE = torch.empty((V, D), dtype=grad_dtype, device=dev)
    db = torch.empty((V,), dtype=torch.float32, device=dev)
    lib = _lib.load()
    gd = _lib.SPARTON_BF16 if grad_dtype == torch.bfloat16 else _lib.SPARTON_F32
    ws_bytes = int(lib.sparton_bwd_workspace_bytes(B, S, D, V, gd))
    ws = torch.empty((ws_bytes,), dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        rc = lib.sparton_bwd_fp8(qH.data_ptr(), qE.data_ptr(), amax_h.data_ptr(), amax_e.data_ptr(), Y.data_ptr(),
                                 I.data_ptr(), dY.data_ptr(), dH.data_ptr(), dE.data_ptr(), db.data_ptr(), B, S, D,
                                 V, Y.stride(0), dY.stride(0), int(bool(include_bias_grad)), gd, ws.data_ptr(),
                                 ws_bytes, _stream_ptr(), None)
    _lib.check(rc)
    return dH, dE, db


def bwd_workspace_bytes(B: int, S: int, D: int, V: int, grad_dtype: torch.dtype = torch.float32) -> int:
    gd = _lib.SPARTON_BF16 if grad_dtype == torch.bfloat16 else _lib.SPARTON_F32
    return int(_lib.load().sparton_bwd_workspace_bytes(B, S, D + (-D) % 8, V, gd))


@torch.no_grad()
def sparton_backward(H: torch.Tensor, E: torch.Tensor, Y: torch.Tensor, I: torch.Tensor,
                     dY: torch.Tensor, *, include_bias_grad: bool = True,
                     grad_dtype: torch.dtype = torch.float32,
                     dh_ready: torch.cuda.Event | None = None,
                     out_dH: torch.Tensor | None = None
                     ) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Argmax-routed backward from the saved (Y, I) only (fused.py:215-278).

    Returns (dH [B,S,D], dE [V,D], db [V] f32); dH/dE in ``grad_dtype``
    (float32 or bfloat16), accumulated in fp32 by single-owner kernels.
    Like the reference, only shapes are validated (fused.py:232-245).
    ``dY`` (and Y/I, sharing one row stride) may be column slices of wider
    row-major tensors (unit column stride; row strides passed as ldDY / ldY,
    no copy).  ``dh_ready``, if
    given, is recorded on the current stream as soon as dH is final, before
    the dE work joins (``sparton_bwd_ex``).  ``out_dH`` receives dH instead of
    a fresh tensor (contiguous [B, S, D] in ``grad_dtype``, D a multiple of 8:
    e.g. a peer-addressable buffer the sharded head reduces in place).
    """
    for name, t in (("H", H), ("E", E), ("Y", Y), ("I", I), ("dY", dY)):
        _require_cuda(name, t)
    if H.dim() != 3 or E.dim() != 2 or E.shape[1] != H.shape[2]:
        raise ValueError("input shapes disagree with dims")
    B, S, D = H.shape
    V = E.shape[0]
    if Y.shape != (B, V) or I.shape != (B, V):
        raise ValueError(f"saved state must have shape {(B, V)}")
    if dY.shape != (B, V):
        raise ValueError(f"dY must have shape {(B, V)}, got {tuple(dY.shape)}")
    if Y.dtype != torch.float32 or I.dtype != torch.int32 or dY.dtype != torch.float32:
        raise ValueError("Y/dY must be float32 and I int32")
    if grad_dtype not in (torch.float32, torch.bfloat16):
        raise ValueError("grad_dtype must be torch.float32 or torch.bfloat16")
    Hp = _pad_hidden(H.contiguous())
    Ep = _pad_hidden(E.contiguous())
    Dp = Hp.shape[2]
    if Y.stride(1) != 1 or I.stride(1) != 1 or I.stride(0) != Y.stride(0) or Y.stride(0) < V:
        Y = Y.contiguous()
        I = I.contiguous()
    if dY.stride(1) != 1 or dY.stride(0) < V:
        dY = dY.contiguous()
    dev = H.device
    if out_dH is not None:
        if (out_dH.shape != (B, S, Dp) or out_dH.dtype != grad_dtype or not out_dH.is_contiguous()
                or out_dH.device != dev):
            raise ValueError(f"out_dH must be a contiguous {grad_dtype} tensor of shape {(B, S, Dp)} on {dev}")
        dH = out_dH
    else:
        dH = torch.empty((B, S, Dp), dtype=grad_dtype, device=dev)
    dE = torch.empty((V, Dp), dtype=grad_dtype, device=dev)
    db = torch.empty((V,), dtype=torch.float32, device=dev)
    lib = _lib.load()
    gd = _lib.SPARTON_BF16 if grad_dtype == torch.bfloat16 else _lib.SPARTON_F32
    ws_bytes = int(lib.sparton_bwd_workspace_bytes(B, S, Dp, V, gd))
    ws = torch.empty((ws_bytes,), dtype=torch.uint8, device=dev)
    ev = 0
    if dh_ready is not None:
        if dh_ready.cuda_event == 0:       # torch creates the event lazily on first record
            dh_ready.record()
        ev = dh_ready.cuda_event
    with torch.cuda.device(dev):
        rc = lib.sparton_bwd_ex(Hp.data_ptr(), Ep.data_ptr(), Y.data_ptr(), I.data_ptr(), dY.data_ptr(),
                                dH.data_ptr(), dE.data_ptr(), db.data_ptr(), B, S, Dp, V, Y.stride(0),
                                dY.stride(0), int(bool(include_bias_grad)), gd, ws.data_ptr(), ws_bytes,
                                _stream_ptr(), ev)
    _lib.check(rc)
    if Dp != D:
        dH = dH[..., :D]
        dE = dE[:, :D]
    return dH, dE, db


# ---------------------------------------------------------------- fp32 inputs on bf16 tensor cores

def split_bf16x3(x: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Exact three-way split of fp32 values into bf16 parts, x = x1 + x2 + x3.

    x1 = bf16(x) keeps the top 8 significant bits; x - x1 is exact in fp32
    (Sterbenz) and has at most 16 bits, x2 = bf16(x - x1) takes the next 8 and
    the remainder (at most 8 bits) is x3 exactly.  (Values whose low parts
    underflow bf16's denormal range lose those bits, as fp32 would.)"""
    x = x.float()
    x1 = x.to(torch.bfloat16)
    r = x - x1.float()
    x2 = r.to(torch.bfloat16)
    x3 = (r - x2.float()).to(torch.bfloat16)
    return x1, x2, x3


@torch.no_grad()
def sparton_forward_fp32(H: torch.Tensor, E: torch.Tensor, bias: torch.Tensor, mask: torch.Tensor
                         ) -> tuple[torch.Tensor, torch.Tensor]:
    """Forward on fp32 H/E at fp32 accuracy, on the same bf16 tensor-core kernel.

    With H = H1 + H2 + H3 and E = E1 + E2 + E3 (``split_bf16x3``; |X2| <=
    2^-8 |X|, |X3| <= 2^-16 |X|), every partial product Hi·Ej of two 8-bit
    significands is exact in fp32.  The six terms with i + j <= 4 are one bf16
    contraction over the concatenated hidden axis (D' = 6·D,
    H' = [H1, H1, H2, H1, H2, H3], E' = [E1, E2, E1, E3, E2, E1]) accumulated
    in fp32; the three dropped terms are below 2^-23 of each product, i.e.
    within fp32 rounding.  The result is an fp32 dot
    product in a different summation order — what the reference's own fp32
    tolerances allow (Y rel 1e-5, bench.py:41-46).  Costs 6x the bf16
    forward; meant for the fp32 numpy drop-in (``fusedhead.PRECISION``)."""
    for name, t in (("H", H), ("E", E)):
        _require_cuda(name, t)
        if t.dtype != torch.float32:
            raise ValueError(f"{name} must be float32 for the fp32 forward, got {t.dtype}")
    h = split_bf16x3(H)
    e = split_bf16x3(E)
    terms = ((0, 0), (0, 1), (1, 0), (0, 2), (1, 1), (2, 0))
    Hc = torch.cat([h[i] for i, _ in terms], dim=-1)
    Ec = torch.cat([e[j] for _, j in terms], dim=-1)
    return sparton_forward(Hc, Ec, bias, mask)


@torch.no_grad()
def sparton_backward_fp32(H: torch.Tensor, E: torch.Tensor, Y: torch.Tensor, I: torch.Tensor,
                          dY: torch.Tensor, *, include_bias_grad: bool = True
                          ) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Backward on fp32 H/E: dE = Σ_b g·H[b, I] and dH = Σ_v g·E[v] are
    linear in H and E, so with the exact splits they are the fp32 sums of
    three bf16-operand backwards (each fp32-accumulated in the reference's
    order) — fp32 accuracy (the reference's BACKWARD_PAIR_TOL 1e-5)."""
    for name, t in (("H", H), ("E", E)):
        _require_cuda(name, t)
        if t.dtype != torch.float32:
            raise ValueError(f"{name} must be float32 for the fp32 backward, got {t.dtype}")
    h = split_bf16x3(H)
    e = split_bf16x3(E)
    dH, dE, db = sparton_backward(h[0], e[0], Y, I, dY, include_bias_grad=include_bias_grad)
    for k in (1, 2):
        a, b_, _ = sparton_backward(h[k], e[k], Y, I, dY, include_bias_grad=include_bias_grad)
        dH += a
        dE += b_
    return dH, dE, db


class SpartonHeadFn(torch.autograd.Function):
    """Autograd op: Y = SpartonHead(H, E, bias, mask).

    forward saves (H, E, Y, I) — H and E are the caller's tensors, so the head
    adds only B·V·8 bytes of saved state (SavedSparseState, fused.py:67-80).
    backward returns (dH, dE, db, None) in the input dtypes.
    """

    @staticmethod
    def forward(ctx, H, E, bias, mask, include_bias_grad=True):
        Y, I = sparton_forward(H, E, bias, mask)
        ctx.save_for_backward(H, E, Y, I)
        ctx.include_bias_grad = bool(include_bias_grad)
        ctx.mark_non_differentiable(I)
        return Y, I

    @staticmethod
    def backward(ctx, dY, dI_unused):
        H, E, Y, I = ctx.saved_tensors
        if dY is None:
            return None, None, None, None, None
        dH, dE, db = sparton_backward(H, E, Y, I, dY.float(), include_bias_grad=ctx.include_bias_grad,
                                      grad_dtype=H.dtype)
        if dE.dtype != E.dtype:
            dE = dE.to(E.dtype)
        return dH, dE, db, None, None


class SpartonHeadFp8Fn(torch.autograd.Function):
    """FP8 autograd op: the e4m3 forward (``sparton_forward_fp8``) saves the
    quantised operands with (Y, I); backward is ``sparton_backward_fp8``
    (straight-through w.r.t. the quantisation).  Gradients in the inputs'
    dtypes (bf16 for H/E, f32 for bias)."""

    @staticmethod
    def forward(ctx, H, E, bias, mask, include_bias_grad=True):
        (Y, I), (qH, aH, qE, aE) = sparton_forward_fp8(H, E, bias, mask, return_quantized=True)
        ctx.save_for_backward(qH, aH, qE, aE, Y, I)
        ctx.include_bias_grad = bool(include_bias_grad)
        ctx.dtypes = (H.dtype, E.dtype)
        ctx.mark_non_differentiable(I)
        return Y, I

    @staticmethod
    def backward(ctx, dY, dI_unused):
        qH, aH, qE, aE, Y, I = ctx.saved_tensors
        if dY is None:
            return None, None, None, None, None
        dH, dE, db = sparton_backward_fp8(qH, aH, qE, aE, Y, I, dY.float(),
                                          include_bias_grad=ctx.include_bias_grad, grad_dtype=ctx.dtypes[0])
        return dH, dE.to(ctx.dtypes[1]), db, None, None


class SpartonHeadMxFn(torch.autograd.Function):
    """MXFP8 autograd op: the block-scaled e4m3 forward (``sparton_forward_mx``)
    and the bf16 argmax-routed backward on the caller's bf16 H, E at the MX
    forward's (Y, I) — the usual low-precision recipe (FP8 forward, bf16
    backward), straight-through w.r.t. the quantisation.  Saved state is the
    same B·V·8 bytes as ``SpartonHeadFn``."""

    @staticmethod
    def forward(ctx, H, E, bias, mask, include_bias_grad=True):
        Y, I = sparton_forward_mx(H, E, bias, mask)
        ctx.save_for_backward(H, E, Y, I)
        ctx.include_bias_grad = bool(include_bias_grad)
        ctx.mark_non_differentiable(I)
        return Y, I

    backward = staticmethod(SpartonHeadFn.backward)


def sparton_head_mx(H: torch.Tensor, E: torch.Tensor, bias: torch.Tensor, mask: torch.Tensor,
                    include_bias_grad: bool = True) -> tuple[torch.Tensor, torch.Tensor]:
    """Functional MXFP8 head: (Y, I) with autograd through Y (``SpartonHeadMxFn``)."""
    return SpartonHeadMxFn.apply(H, E, bias, mask, include_bias_grad)


def sparton_head_fp8(H: torch.Tensor, E: torch.Tensor, bias: torch.Tensor, mask: torch.Tensor,
                     *, return_indices: bool = False, include_bias_grad: bool = True):
    """FP8 (e4m3, per-tensor scales) forward + backward of the head."""
    Y, I = SpartonHeadFp8Fn.apply(H, E, bias, mask, include_bias_grad)
    return (Y, I) if return_indices else Y


def sparton_head(H: torch.Tensor, E: torch.Tensor, bias: torch.Tensor, mask: torch.Tensor,
                 *, return_indices: bool = False, include_bias_grad: bool = True):
    """Differentiable SPLADE max-pooled LM head (drop-in for the naive
    ``((H@E.T + b) * M[...,None]).relu().log1p().max(dim=1)``)."""
    Y, I = SpartonHeadFn.apply(H, E, bias, mask, include_bias_grad)
    return (Y, I) if return_indices else Y
