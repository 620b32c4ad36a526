"""Forward at cfg3: bf16 vs e4m3 (per-tensor scales) vs MXFP8 (ue8m0 block
scales per 32 K elements; E quantised once as a weight, H quantised every
call and included in the time), plus the quantisers alone."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2603_25011_b200 import quantize_e4m3, quantize_mx, sparton_forward, sparton_forward_fp8, sparton_forward_mx

B, S, D, V = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (512, 512, 768, 250002)))
g = torch.Generator(device="cuda").manual_seed(0)
H = torch.randn((B, S, D), generator=g, device="cuda").to(torch.bfloat16)
E = (torch.randn((V, D), generator=g, device="cuda") * 0.02).to(torch.bfloat16)
b = torch.zeros(V, device="cuda")
m = torch.ones((B, S), dtype=torch.uint8, device="cuda")
Eq = quantize_e4m3(E)
Emx = quantize_mx(E, "E")
runs = (("bf16", lambda: sparton_forward(H, E, b, m)), ("fp8", lambda: sparton_forward_fp8(H, E, b, m, E_q=Eq)),
        ("mxfp8", lambda: sparton_forward_mx(H, E, b, m, E_q=Emx)), ("quant_e4m3(H)", lambda: quantize_e4m3(H)),
        ("quant_mx(H)", lambda: quantize_mx(H, "H")))
for name, fn in runs + runs[:3]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: fwd {ms:.2f} ms  {2*B*S*V*D/ms/1e9:.0f} TF/s (algorithmic)", flush=True)
