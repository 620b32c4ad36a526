"""GPU sweep in the reference harness's CSV schema (paper_2603_25011_b200.sweep)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_sweep_rows(cuda_device):
    from paper_2603_25011_b200 import sweep
    rows = sweep.run_sweep((2, 40, 64, 300), "V", [300, 1001], repeats=2, warmup=1)
    ncol = len(sweep.HEADER.split(","))
    assert len(rows) == 2
    for r, v in zip(rows, (300, 1001)):
        f = r.split(",")
        assert len(f) == ncol and f[0] == "b200" and int(f[4]) == v
        assert float(f[8]) > 0 and int(f[12]) == 2 * v * 8     # saved (Y, I) bytes = B*V*8
        assert len(f[13]) == 8
        assert int(f[17]) == 2 * 40 * 64 * 2 + v * 64 * 2 + v * 4 + 2 * 40 + 2 * v * 8   # model fwd bytes
        assert int(f[18]) > 0 and float(f[19]) > 0
