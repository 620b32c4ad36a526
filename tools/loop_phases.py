"""fwd -> bwd loop at cfg3 (like bench.py's step) with CUDA events per phase,
for each SPARTON_BWD_CONCURRENT mode given on the command line."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import CONFIGS, make_inputs  # noqa: E402
from paper_2603_25011_b200 import sparton_backward, sparton_forward  # noqa: E402

os.environ["SPARTON_DEV"] = "1"
c = CONFIGS["cfg3"]
dev = torch.device("cuda", 0)
H, E, bias, mask, dY, _ = make_inputs(c, dev, 0, 1)
for mode in sys.argv[1:]:
    os.environ["SPARTON_BWD_CONCURRENT"] = mode
    evs = []
    for it in range(13):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        Y, I = sparton_forward(H, E, bias, mask)
        e[1].record()
        sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
        e[2].record()
        if it >= 3:
            evs.append(e)
    torch.cuda.synchronize()
    f = [a.elapsed_time(b) for a, b, _ in evs]
    bw = [b.elapsed_time(c_) for _, b, c_ in evs]
    print(f"mode {mode}: fwd {statistics.mean(f):.2f}  bwd {statistics.mean(bw):.2f}  total "
          f"{statistics.mean(f) + statistics.mean(bw):.2f} ms", flush=True)
    time.sleep(3)
