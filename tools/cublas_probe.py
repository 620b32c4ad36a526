"""Time cuBLAS bf16 GEMMs at the Sparton forward shape (V x B*S x D) as a yardstick."""
import json, torch
torch.manual_seed(0)
dev = "cuda"
for (V, BS, D) in [(30522, 262144, 768), (8192, 8192, 8192), (32768, 65536, 768)]:
    a = torch.randn(V, D, device=dev, dtype=torch.bfloat16)
    b = torch.randn(BS, D, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        c = a @ b.T
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 5
    for _ in range(n):
        c = a @ b.T
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(json.dumps({"probe": "cublas_bf16", "V": V, "BS": BS, "D": D, "ms": ms,
                      "tflops": 2 * V * BS * D / ms / 1e9}))
    del a, b, c
    torch.cuda.empty_cache()
