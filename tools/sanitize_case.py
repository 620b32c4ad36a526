"""One fused forward + bf16/fp32 backward at the given (B, S, D, V) for
compute-sanitizer runs (tools/sanitize.sh).
Usage: python tools/sanitize_case.py B S D V [bias] [mx]
  bias: constant bias (e.g. -2: few active pairs, the backward's sparse regime)
  mx:   also run the MXFP8 forward (quantisers + block-scaled kernel)"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_25011_b200 import sparton_backward, sparton_forward, sparton_forward_mx  # noqa: E402

B, S, D, V = (int(x) for x in sys.argv[1:5])
bias = float(sys.argv[5]) if len(sys.argv) > 5 else 0.0
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
H = torch.randn((B, S, D), generator=g, device=dev).to(torch.bfloat16)
E = (torch.randn((V, D), generator=g, device=dev) * 0.02).to(torch.bfloat16)
b = torch.full((V,), bias, device=dev)
m = (torch.rand((B, S), generator=g, device=dev) < 0.9).to(torch.uint8)
dY = torch.randn((B, V), generator=g, device=dev)
Y, I = sparton_forward(H, E, b, m)
for gd in (torch.bfloat16, torch.float32):
    dH, dE, db = sparton_backward(H, E, Y, I, dY, grad_dtype=gd)
if "mx" in sys.argv[5:]:
    Ym, Im = sparton_forward_mx(H, E, b, m)
torch.cuda.synchronize()
print("case ok", B, S, D, V, bias, float((Y > 0).float().mean()), float(Y.sum()), float(dH.float().abs().sum()))
