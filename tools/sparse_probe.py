"""Backward time vs pair activity (SURVEY §8d "SPLADE-sparse" variant): cfg3
with bias b in {0, -1, -2, -3} (fewer active pairs as b falls); prints the
active fraction, forward ms and backward ms (full, route+dE only, route+dH
only via the dev-gated SPARTON_BWD_CONCURRENT switch)."""
import os
import sys

import torch

sys.path.insert(0, ".")
os.environ["SPARTON_DEV"] = "1"
from bench import CONFIGS, make_inputs  # noqa: E402
from paper_2603_25011_b200 import sparton_backward, sparton_forward  # noqa: E402

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
biases = [float(x) for x in sys.argv[2:]] or [0.0, -1.0, -2.0, -3.0]
dev = torch.device("cuda", 0)
H, E, bias, mask, dY, _ = make_inputs(c, dev, 0, 1)


def timed(fn, n=10):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for bv in biases:
    bias.fill_(bv)
    Y, I = sparton_forward(H, E, bias, mask)
    torch.cuda.synchronize()
    act = float((Y > 0).float().mean())
    fwd = timed(lambda: sparton_forward(H, E, bias, mask), 3)
    out = []
    # default thresholds, all-dense kernels, all-sparse kernels
    for label, pct in (("default", None), ("dense", "-1"), ("sparse", "100")):
        for k in ("SPARTON_DE_SPARSE_PCT", "SPARTON_DH_SPARSE_PCT"):
            if pct is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = pct
        res = {}
        for mode in ("1", "3", "4"):
            os.environ["SPARTON_BWD_CONCURRENT"] = mode
            res[mode] = timed(lambda: sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16))
        os.environ["SPARTON_BWD_CONCURRENT"] = "1"
        out.append(f"{label}: {res['1']:.2f} (route+dE {res['3']:.2f}, route+dH {res['4']:.2f})")
    print(f"bias {bv:+.2f}: active {act:.4f}  fwd {fwd:.2f} ms  bwd ms " + " | ".join(out), flush=True)
