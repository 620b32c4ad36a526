"""The paper's long-sequence backward table (A100, B=128,
V=30522, D=768, S = 1024..8192, Sparton backward 71.2 / 118.6 / 212.7 /
399.6 ms, 0.99 / 1.55 / 2.68 / 5.13 GB) on one B200: forward and backward
times (CUDA events, 10 iterations after 3 warm-ups) and the head-owned peak
memory of the backward (outputs + workspace), one JSON line per S."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_25011_b200 import sparton_backward, sparton_forward  # noqa: E402

B, D, V = 128, 768, 30522
dev = torch.device("cuda", 0)
for S in (1024, 2048, 4096, 8192):
    g = torch.Generator(device=dev).manual_seed(S)
    H = torch.randn((B, S, D), generator=g, device=dev).to(torch.bfloat16)
    E = (torch.randn((V, D), generator=g, device=dev) * 0.02).to(torch.bfloat16)
    b = torch.zeros(V, device=dev)
    m = torch.ones((B, S), dtype=torch.uint8, device=dev)
    dY = torch.randn((B, V), generator=g, device=dev)
    res = {}
    for name in ("fwd", "bwd"):
        Y, I = sparton_forward(H, E, b, m)
        fn = (lambda: sparton_forward(H, E, b, m)) if name == "fwd" else \
             (lambda: sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16))
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
        base = torch.cuda.memory_allocated(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            out = fn()
            del out
        e1.record()
        torch.cuda.synchronize()
        res[name + "_ms"] = e0.elapsed_time(e1) / 10
        res[name + "_head_peak_gb"] = (torch.cuda.max_memory_allocated(dev) - base) / 1e9
        del Y, I
    print(json.dumps({"B": B, "S": S, "D": D, "V": V, **res}), flush=True)
    del H, E, b, m, dY
    torch.cuda.empty_cache()
