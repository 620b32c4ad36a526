import sys, torch
sys.path.insert(0, ".")
from paper_2603_25011_b200 import quantize_e4m3, sparton_forward_fp8
B, S, D, V = 512, 512, 768, 250002
g = torch.Generator(device="cuda").manual_seed(0)
H = torch.randn((B, S, D), generator=g, device="cuda").to(torch.bfloat16)
E = (torch.randn((V, D), generator=g, device="cuda") * 0.02).to(torch.bfloat16)
b = torch.zeros(V, device="cuda"); m = torch.ones((B, S), dtype=torch.uint8, device="cuda")
Eq = quantize_e4m3(E)
ref = None
for cg in (2, 4, 2, 4):
    for _ in range(3): Y, I = sparton_forward_fp8(H, E, b, m, E_q=Eq, cta_group=cg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): Y, I = sparton_forward_fp8(H, E, b, m, E_q=Eq, cta_group=cg)
    e1.record(); torch.cuda.synchronize()
    if ref is None: ref = (Y.clone(), I.clone())
    print(f"fp8 cg={cg}: {e0.elapsed_time(e1)/10:.2f} ms  same={torch.equal(Y, ref[0]) and torch.equal(I, ref[1])}", flush=True)
