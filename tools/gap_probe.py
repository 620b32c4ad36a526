"""How fast do SM clocks recover after the power-capped forward?  fwd -> GPU
sleep(gap) -> bwd at cfg3; reports bwd time per gap (diagnostic only)."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import CONFIGS, make_inputs  # noqa: E402
from paper_2603_25011_b200 import sparton_backward, sparton_forward  # noqa: E402

c = CONFIGS["cfg3"]
dev = torch.device("cuda", 0)
H, E, bias, mask, dY, _ = make_inputs(c, dev, 0, 1)
for gap_ms in [0, 1, 3, 10, 30, 0]:
    cyc = int(gap_ms * 1.9e6)
    res = []
    for it in range(10):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        Y, I = sparton_forward(H, E, bias, mask)
        e[1].record()
        if cyc:
            torch.cuda._sleep(cyc)
        e[2].record()
        sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
        e[3].record()
        if it >= 3:
            res.append(e)
    torch.cuda.synchronize()
    f = statistics.mean(a.elapsed_time(b) for a, b, _, _ in res)
    g = statistics.mean(b.elapsed_time(c_) for _, b, c_, _ in res)
    bw = statistics.mean(c_.elapsed_time(d) for _, _, c_, d in res)
    print(f"gap {gap_ms:3d} ms (measured {g:.2f}): fwd {f:.2f}  bwd {bw:.2f}", flush=True)
    time.sleep(2)
