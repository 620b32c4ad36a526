"""compute-sanitizer case for sparton_allreduce_peers (tools/sanitize.sh): three ranks on one GPU, uneven slices, fp32 and bf16 outputs."""
import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_2603_25011_b200 import _lib
lib = _lib.load()
dev = torch.device("cuda", 0)
for n, dt in ((4 * 1001, 0), (4 * 3, 1), (4 * 50000, 1)):
    parts = [torch.randn(n, device=dev) for _ in range(3)]
    outs = [torch.zeros(n, device=dev, dtype=torch.float32 if dt == 0 else torch.bfloat16) for _ in range(3)]
    pa = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in parts])
    oa = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in outs])
    for r in range(3):
        _lib.check(lib.sparton_allreduce_peers(pa, oa, 3, r, dt, n, torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("ok")
