"""Time fwd-only, bwd-only and fwd+bwd loops in one process (cfg3) to separate
kernel speed from power-state effects; samples SM clocks per phase."""
import json
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import CONFIGS, make_inputs  # noqa: E402
from paper_2603_25011_b200 import sparton_backward, sparton_forward  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
dev = torch.device("cuda", 0)
H, E, bias, mask, dY, _ = make_inputs(c, dev, 0, 1)
Y, I = sparton_forward(H, E, bias, mask)
out = sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
torch.cuda.synchronize()


def clocks():
    r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                       capture_output=True, text=True).stdout.strip()
    return r


def loop(name, fn, n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    time.sleep(0.05)
    mid = clocks()
    torch.cuda.synchronize()
    print(json.dumps({"phase": name, "ms_per_iter": e0.elapsed_time(e1) / n, "clock_power_mid": mid}), flush=True)


for rep in range(2):
    loop("fwd", lambda: sparton_forward(H, E, bias, mask, out=(Y, I)), 10)
    time.sleep(2)
    loop("bwd", lambda: sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16), 10)
    time.sleep(2)
    loop("fwd+bwd", lambda: (sparton_forward(H, E, bias, mask, out=(Y, I)),
                             sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)), 10)
    time.sleep(2)
