import time, numpy as np, torch
dev = torch.device("cuda", 0)
H = np.random.default_rng(0).standard_normal((512, 512, 768), dtype=np.float32)
def t(name, fn, n=3):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(f"{name}: {min(ts)*1e3:.1f} ms  ({H.nbytes/min(ts)/1e9:.1f} GB/s)", flush=True)
t("pageable .to(dev)", lambda: torch.from_numpy(H).to(dev))
t("pin_memory()", lambda: torch.from_numpy(H).pin_memory())
P = torch.from_numpy(H).pin_memory()
t("pinned .to(dev) async", lambda: P.to(dev, non_blocking=True))
buf = torch.empty(H.shape, dtype=torch.float32).pin_memory()
t("copy_ into cached pinned", lambda: buf.copy_(torch.from_numpy(H)))
import threading
def mt_copy(nt=8):
    src = torch.from_numpy(H).view(-1); dst = buf.view(-1); n = src.numel(); step = (n + nt - 1) // nt
    th = [threading.Thread(target=lambda i=i: dst[i*step:(i+1)*step].copy_(src[i*step:(i+1)*step])) for i in range(nt)]
    [x.start() for x in th]; [x.join() for x in th]
t("copy_ into pinned, 8 threads", mt_copy)
torch.set_num_threads(16)
t("copy_ into cached pinned (16 intra-op threads)", lambda: buf.copy_(torch.from_numpy(H)))
D = torch.empty(H.shape, device=dev)
t("D2H .cpu()", lambda: D.cpu())
t("D2H into cached pinned", lambda: buf.copy_(D, non_blocking=True))
t("D2H .cpu().numpy() copy to fresh numpy", lambda: D.cpu().numpy())
