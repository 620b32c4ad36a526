"""A/B the backward scheduling modes in one process (cfg3): bwd-only loops."""
import json, os, sys, time
import torch
sys.path.insert(0, ".")
from bench import CONFIGS, make_inputs
from paper_2603_25011_b200 import sparton_backward, sparton_forward
c = CONFIGS["cfg3"]
dev = torch.device("cuda", 0)
H, E, bias, mask, dY, _ = make_inputs(c, dev, 0, 1)
Y, I = sparton_forward(H, E, bias, mask)
ref = [t.float().clone() for t in sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)]
for rep in range(3):
    for mode in ("0", "1", "2"):
        os.environ["SPARTON_BWD_CONCURRENT"] = mode
        out = sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
        torch.cuda.synchronize()
        same = all(torch.equal(a.float(), b) for a, b in zip(out, ref))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            sparton_backward(H, E, Y, I, dY, grad_dtype=torch.bfloat16)
        e1.record(); torch.cuda.synchronize()
        print(json.dumps({"mode": mode, "ms": e0.elapsed_time(e1) / 5, "bitwise_same": same}), flush=True)
        time.sleep(1)
