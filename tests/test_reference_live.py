"""CPU: when the read-only reference is present (build container only), check
the oracle against the live reference on a wider grid than the fixtures.
Skipped on the GPU box, where /root/reference does not exist."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import sparton_oracle as orc

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference not mounted")


@pytest.fixture(scope="module")
def fh():
    sys.path.insert(0, str(REF))
    import fusedhead
    return fusedhead


GRID = [(b, s, d, v) for b in (1, 2, 4) for s in (1, 3, 8, 32) for d in (2, 4, 16) for v in (1, 5, 16, 64)]


@pytest.mark.parametrize("dims", GRID[::3])
def test_oracle_equals_reference(fh, dims):
    B, S, D, V = dims
    seed = 31 * B + 7 * S + 3 * D + V
    inputs = fh.HeadInputs.seeded(fh.Dims(*dims), seed, mask_keep=0.8)
    dY = fh.seeded_tensor((B, V), seed + 9)
    ref, _ = fh.forward_eager(inputs, deterministic=True)
    Y, I = orc.forward(inputs.H, inputs.E, inputs.b, inputs.mask, deterministic=True)
    assert Y.tobytes() == ref.Y.tobytes() and np.array_equal(I, ref.I)
    gref = fh.backward_fused(inputs, fh.SavedSparseState.from_output(ref), dY)
    dH, dE, db = orc.backward(inputs.H, inputs.E, inputs.b, ref.Y, ref.I, dY)
    assert dH.tobytes() == gref.dH.tobytes() and dE.tobytes() == gref.dE.tobytes()
    assert db.tobytes() == gref.db.tobytes()
    # the oracle's input generator is the reference's
    H, E, b, m = orc.seeded_inputs(B, S, D, V, seed, mask_keep=0.8)
    assert H.tobytes() == inputs.H.tobytes() and np.array_equal(m, inputs.mask)


def test_mirror_api_types_match_reference(fh):
    """paper_2603_25011_b200.fusedhead mirrors the reference's dataclasses and
    validation (same names, same errors) without needing a GPU for this part."""
    from paper_2603_25011_b200 import fusedhead as mine
    for name in ("Dims", "HeadInputs", "HeadOutput", "HeadGradients", "SavedSparseState", "TileConfig",
                 "forward_hybrid", "forward_fully_fused", "backward_fused", "seeded_tensor", "seeded_mask",
                 "splitmix64"):
        assert hasattr(mine, name) and hasattr(fh, name), name
    d = mine.Dims(3, 4, 5, 6)
    a = mine.HeadInputs.seeded(d, 7, mask_keep=0.5)
    r = fh.HeadInputs.seeded(fh.Dims(3, 4, 5, 6), 7, mask_keep=0.5)
    assert a.H.tobytes() == r.H.tobytes() and np.array_equal(a.mask, r.mask)
    for dims in [(16, 4096, 8, 1024), (2, 3, 4, 5), (8, 512, 768, 30522)]:
        c1 = mine.TileConfig.default_for(mine.Dims(*dims))
        c2 = fh.TileConfig.default_for(fh.Dims(*dims))
        assert (c1.vocab_tile, c1.batch_tile) == (c2.vocab_tile, c2.batch_tile)


def test_sweep_csv_schema_matches_reference(fh):
    # The GPU sweep keeps the reference harness's CSV columns (bench.py:32-35)
    # and checksum (bench.py:61-62), then appends its GPU columns.
    from fusedhead import bench as ref_bench
    from paper_2603_25011_b200 import sweep
    assert sweep.REFERENCE_HEADER == ref_bench.BENCH_CSV_HEADER
    assert sweep.HEADER.startswith(ref_bench.BENCH_CSV_HEADER + ",")
    Y = np.random.default_rng(0).random((3, 7), dtype=np.float32)
    assert sweep.y_checksum(Y) == ref_bench.y_checksum(Y)
