"""Sample SM clock / power while looping (a) the fused forward at cfg3, (b) the
backward, (c) a cuBLAS bf16 8192^3 matmul — tells whether a phase is power-capped."""
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import CONFIGS, make_inputs  # noqa: E402
from paper_2603_25011_b200 import sparton_backward, sparton_forward  # noqa: E402

c = CONFIGS["cfg3"]
dev = torch.device("cuda", 0)
H, E, bias, mask, dY, _ = make_inputs(c, dev, 0, 1)
Y, I = sparton_forward(H, E, bias, mask)
sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
bm = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
torch.cuda.synchronize()
Q = "clocks.sm,power.draw.instant,power.draw.average,clocks_event_reasons.active"


def phase(name, fn, n):
    p = subprocess.Popen(["nvidia-smi", f"--query-gpu={Q}", "--format=csv,noheader,nounits", "-lms", "50"],
                         stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    p.terminate()
    out = p.communicate()[0].strip().splitlines()
    rows = [x.split(", ") for x in out]
    busy = rows[6:-2] if len(rows) > 10 else rows
    clk = sorted(float(r[0]) for r in busy)
    pw = sorted(float(r[1]) for r in busy if r[1].replace('.', '').isdigit())
    reasons = sorted(set(r[3] for r in busy))
    print(f"{name}: {e0.elapsed_time(e1)/n:.2f} ms/iter; sm clk median {clk[len(clk)//2]:.0f} "
          f"[{clk[0]:.0f},{clk[-1]:.0f}]; power instant median {pw[len(pw)//2] if pw else -1:.0f} W max "
          f"{pw[-1] if pw else -1:.0f}; reasons {reasons}", flush=True)
    time.sleep(2)


phase("fwd", lambda: sparton_forward(H, E, bias, mask, out=(Y, I)), 40)
phase("bwd", lambda: sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16), 80)
phase("cublas8192", lambda: torch.matmul(a, bm), 3000)
phase("fwd+bwd", lambda: (sparton_forward(H, E, bias, mask, out=(Y, I)),
                          sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)), 30)
