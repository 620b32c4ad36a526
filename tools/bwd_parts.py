"""Power/clock/time of backward parts in isolation (experiment switch
SPARTON_BWD_CONCURRENT: 1 full, 3 route+dE only, 4 route+dH only) at cfg3."""
import os
import subprocess
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
Y, I = sparton_forward(H, E, bias, mask)
torch.cuda.synchronize()
Q = "clocks.sm,power.draw.instant"
for mode in sys.argv[1:]:
    os.environ["SPARTON_BWD_CONCURRENT"] = mode
    for _ in range(3):
        sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    p = subprocess.Popen(["nvidia-smi", f"--query-gpu={Q}", "--format=csv,noheader,nounits", "-lms", "50"],
                         stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 60
    e0.record()
    for _ in range(n):
        sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
    e1.record()
    torch.cuda.synchronize()
    p.terminate()
    rows = [r.split(", ") for r in p.communicate()[0].strip().splitlines()][6:-2]
    clk = sorted(float(r[0]) for r in rows)
    pw = sorted(float(r[1]) for r in rows)
    print(f"mode {mode}: {e0.elapsed_time(e1)/n:.2f} ms  clk {clk[len(clk)//2]:.0f}  power {pw[len(pw)//2]:.0f} W",
          flush=True)
    time.sleep(2)
