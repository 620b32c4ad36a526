"""Run the fused forward once at a given shape (for ncu DRAM-traffic probes)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2603_25011_b200 import sparton_forward

B, S, D, V = (int(x) for x in sys.argv[1:5])
dev = torch.device("cuda")
H = torch.randn((B, S, D), device=dev).to(torch.bfloat16)
E = (torch.randn((V, D), device=dev) * 0.02).to(torch.bfloat16)
b = torch.zeros(V, device=dev)
m = torch.ones((B, S), dtype=torch.uint8, device=dev)
for _ in range(int(sys.argv[5]) if len(sys.argv) > 5 else 2):
    Y, I = sparton_forward(H, E, b, m)
torch.cuda.synchronize()
print("ok", float(Y.sum()))
