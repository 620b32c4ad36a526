"""paper_2603_25011_b200 — B200-native fused SPLADE LM head (Sparton).

The hot path of arXiv 2603.25011 built from scratch for sm_100a:
``Y = log1p(relu(max_s((H·Eᵀ + b) ⊙ M)))`` plus int32 argmax, forward in one
tcgen05/TMEM/TMA kernel, backward in deterministic argmax-routed gather
kernels, behind the C ABI of ``include/sparton.h``.

Public surface:
  * torch:  ``sparton_forward``, ``sparton_backward``, ``SpartonHeadFn``, ``sparton_head``
  * reference-API mirror (numpy in/out): ``paper_2603_25011_b200.fusedhead``
  * vocab-sharded multi-GPU head: ``paper_2603_25011_b200.sharded``
"""

from .head import (SpartonHeadFn, SpartonHeadFp8Fn, SpartonHeadMxFn, sparton_head_mx, bwd_workspace_bytes, dequantize_mx, quantize_e4m3, quantize_mx,
                   sparton_backward, sparton_backward_fp8, sparton_backward_fp32, sparton_forward,
                   sparton_forward_fp8, sparton_forward_fp32, sparton_forward_mx, sparton_head, sparton_head_fp8,
                   split_bf16x3)

__version__ = "0.1.0"

__all__ = [
    "SpartonHeadFn",
    "SpartonHeadFp8Fn",
    "sparton_backward_fp8",
    "sparton_head_fp8",
    "bwd_workspace_bytes",
    "sparton_backward",
    "sparton_backward_fp32",
    "sparton_forward",
    "sparton_forward_fp32",
    "split_bf16x3",
    "sparton_forward_fp8",
    "quantize_e4m3",
    "sparton_forward_mx",
    "SpartonHeadMxFn",
    "sparton_head_mx",
    "quantize_mx",
    "dequantize_mx",
    "sparton_head",
]
