"""Time the fused forward at a shape (CUDA events, 10 iters after 3 warm-ups): ms and TF/s."""
import os
import subprocess
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_2603_25011_b200 import sparton_forward

os.environ.setdefault("SPARTON_DEV", "1")   # lets SPARTON_FWD_EPI experiments through
B, S, D, V = (int(x) for x in sys.argv[1:5])
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
H = torch.randn((B, S, D), device=dev, generator=g).to(torch.bfloat16)
E = (torch.randn((V, D), device=dev, generator=g) * 0.02).to(torch.bfloat16)
b = torch.zeros(V, device=dev)
m = torch.ones((B, S), dtype=torch.uint8, device=dev)
Y, I = sparton_forward(H, E, b, m)
for _ in range(3):
    sparton_forward(H, E, b, m, out=(Y, I))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw.instant", "--format=csv,noheader,nounits",
                        "-lms", "50"], stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
e0.record()
for _ in range(n):
    sparton_forward(H, E, b, m, out=(Y, I))
e1.record()
torch.cuda.synchronize()
smi.terminate()
rows = [r.split(", ") for r in smi.communicate()[0].strip().splitlines()][6:-2]
clk = sorted(float(r[0]) for r in rows) or [0]
pw = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit()) or [0]
ms = e0.elapsed_time(e1) / n
print(f"{sys.argv[5] if len(sys.argv) > 5 else ''} fwd {ms:.2f} ms  {2*B*S*V*D/ms/1e9:.0f} TF/s  clk {clk[len(clk)//2]:.0f} MHz  {pw[len(pw)//2]:.0f} W  Ysum={float(Y.double().sum()):.6e} Isum={int(I.long().sum())}", flush=True)
