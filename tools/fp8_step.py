"""FP8 vs bf16 fwd+bwd step time at cfg3 (CUDA events, 10 steps after 3
warm-ups): sparton_forward_fp8 + sparton_backward_fp8 against the bf16 pair.
Prints one JSON line per path."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_25011_b200 import (quantize_e4m3, sparton_backward, sparton_backward_fp8,  # noqa: E402
                                   sparton_forward, sparton_forward_fp8)

B, S, D, V = 512, 512, 768, 250002
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
H = torch.randn((B, S, D), generator=g, device=dev).to(torch.bfloat16)
E = (torch.randn((V, D), generator=g, device=dev) * 0.02).to(torch.bfloat16)
b = torch.zeros(V, device=dev)
m = torch.ones((B, S), dtype=torch.uint8, device=dev)
dY = torch.randn((B, V), generator=g, device=dev)
Eq = quantize_e4m3(E)


def bf16_step():
    Y, I = sparton_forward(H, E, b, m)
    return Y, I, sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)


def fp8_step():
    (Y, I), (qH, aH, qE, aE) = sparton_forward_fp8(H, E, b, m, E_q=Eq, return_quantized=True)
    return Y, I, sparton_backward_fp8(qH, aH, qE, aE, Y, I, dY)


for name, fn in (("bf16", bf16_step), ("fp8", fp8_step)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / 10
    fl = 2 * B * S * V * D + 4 * B * V * D
    print(json.dumps({"path": name, "ms_per_step": ms, "tflops": fl / ms / 1e9}), flush=True)
