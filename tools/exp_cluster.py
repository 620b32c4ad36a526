"""A/B forward cluster shapes (1, 2, 4 CTAs) in one process at cfg3; checks bitwise equality."""
import json, sys, time
import torch
sys.path.insert(0, ".")
from bench import CONFIGS, make_inputs
from paper_2603_25011_b200 import sparton_forward
c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
dev = torch.device("cuda", 0)
H, E, bias, mask, dY, _ = make_inputs(c, dev, 0, 1)
ref = sparton_forward(H, E, bias, mask, cta_group=2)
torch.cuda.synchronize()
for rep in range(2):
    for cg in (2, 4):
        Y, I = sparton_forward(H, E, bias, mask, cta_group=cg)
        torch.cuda.synchronize()
        same = torch.equal(Y, ref[0]) and torch.equal(I, ref[1])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            sparton_forward(H, E, bias, mask, cta_group=cg, out=(Y, I))
        e1.record(); torch.cuda.synchronize()
        print(json.dumps({"cluster": cg, "ms": e0.elapsed_time(e1) / 4, "bitwise_same_as_pair": same}), flush=True)
        time.sleep(2)
