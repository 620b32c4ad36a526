import sys, torch
sys.path.insert(0, ".")
from paper_2603_25011_b200 import sparton_backward, sparton_forward
dev = torch.device("cuda", 0)
for (B, S, D, V) in ((8, 128, 768, 30522), (4, 512, 768, 100000), (3, 1000, 256, 20000)):
    g = torch.Generator(device=dev).manual_seed(0)
    H = torch.randn((B, S, D), generator=g, device=dev).to(torch.bfloat16)
    E = (torch.randn((V, D), generator=g, device=dev) * 0.05).to(torch.bfloat16)
    b = torch.randn(V, generator=g, device=dev) * 0.1
    m = (torch.rand((B, S), generator=g, device=dev) < 0.9).to(torch.uint8)
    dY = torch.randn((B, V), generator=g, device=dev)
    Y0, I0 = sparton_forward(H, E, b, m)
    g0 = sparton_backward(H, E, Y0, I0, dY, grad_dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            Y, I = sparton_forward(H, E, b, m); gg = sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        Y, I = sparton_forward(H, E, b, m)
        gg = sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    ok = torch.equal(Y, Y0) and torch.equal(I, I0) and all(torch.equal(a, c) for a, c in zip(gg, g0))
    # timing eager vs graph
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        Yx, Ix = sparton_forward(H, E, b, m); gx = sparton_backward(H, E, Yx, Ix, dY, grad_dtype=torch.bfloat16)
    e1.record(); torch.cuda.synchronize(); te = e0.elapsed_time(e1) / 20
    e0.record()
    for _ in range(20):
        graph.replay()
    e1.record(); torch.cuda.synchronize(); tg = e0.elapsed_time(e1) / 20
    print((B, S, D, V), "graph == eager:", ok, f"eager {te:.3f} ms graph {tg:.3f} ms")
