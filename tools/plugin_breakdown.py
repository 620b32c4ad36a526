"""Where the reference-facing numpy drop-in spends a cfg3 step: host->device
staging, the kernels, device->host, per phase (wall clock, synchronised)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import CONFIGS, _slice_inputs  # noqa: E402
from paper_2603_25011_b200 import fusedhead as fh  # noqa: E402
from paper_2603_25011_b200.fusedhead import _download, _upload  # noqa: E402
from paper_2603_25011_b200 import sparton_backward, sparton_forward  # noqa: E402

c = CONFIGS["cfg3"]
H, E, b, m, dY = _slice_inputs(c, c["B"], seed=1)
dev = torch.device("cuda", 0)
fh.PRECISION = "bf16"
dims = fh.Dims(c["B"], c["S"], c["D"], c["V"])
inputs = fh.HeadInputs(dims=dims, H=H, E=E, b=b, mask=m)


def t(label, fn, rec):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    rec.setdefault(label, []).append((time.perf_counter() - t0) * 1e3)
    return r


for it in range(4):
    rec = {}
    Hd = t("up H (fp32->bf16)", lambda: _upload(H, dev, "bf16"), rec)
    Ed = t("up E (fp32->bf16)", lambda: _upload(E, dev, "bf16"), rec)
    bd = t("up b, mask", lambda: (_upload(b, dev), _upload(m, dev, dtype=np.uint8)), rec)
    Y, I = t("forward kernel", lambda: sparton_forward(Hd, Ed, bd[0], bd[1]), rec)
    Yh, Ih = t("down Y, I", lambda: _download(Y, I), rec)
    Hd2 = t("up H again", lambda: _upload(H, dev, "bf16"), rec)
    Ed2 = t("up E again", lambda: _upload(E, dev, "bf16"), rec)
    Y2 = t("up Y, I, dY", lambda: (_upload(Yh, dev), _upload(Ih, dev, dtype=np.int32), _upload(dY, dev)), rec)
    g = t("backward kernels", lambda: sparton_backward(Hd2, Ed2, Y2[0], Y2[1], Y2[2]), rec)
    gh = t("down dH, dE, db", lambda: _download(*g), rec)
    tot = t("full drop-in step", lambda: fh.backward_fused(inputs, fh.SavedSparseState.from_output(
        fh.forward_fully_fused(inputs)), dY), rec)
    if it == 3:
        for k, v in rec.items():
            print(f"{k:24s} {v[0]:8.1f} ms")
