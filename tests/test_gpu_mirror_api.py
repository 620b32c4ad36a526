"""The reference-facing drop-in (paper_2603_25011_b200.fusedhead) on the GPU.

Ports of the reference's operator tests (test_fused.py, test_reference.py)
driven through the mirror of ``forward_hybrid`` / ``forward_fully_fused`` /
``backward_fused`` with numpy in/out, exactly as the reference's own callers
use them, and checked against the oracle on the same (bf16-rounded) inputs.
Tolerance: rtol 1e-2 / atol 1e-3 (north star); argmax exact outside certified
near-ties.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sparton_oracle as orc

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-2, 1e-3


def _close(a, b):
    return np.all(np.abs(a.astype(np.float64) - b.astype(np.float64)) <= ATOL + RTOL * np.abs(b))


def _inputs(B, S, D, V, seed, keep=0.85, bf16=True):
    from paper_2603_25011_b200 import fusedhead as fh
    x = fh.HeadInputs.seeded(fh.Dims(B, S, D, V), seed, mask_keep=keep)
    if bf16:
        x.H[...] = orc.bf16_round(x.H)
        x.E[...] = orc.bf16_round(x.E)
    return x


@pytest.mark.parametrize("dims", [(2, 3, 4, 5), (4, 33, 64, 300), (3, 130, 768, 2000), (1, 600, 16, 7)])
@pytest.mark.parametrize("entry", ["forward_hybrid", "forward_fully_fused"])
def test_mirror_forward_vs_oracle(cuda_device, dims, entry):
    from paper_2603_25011_b200 import fusedhead as fh
    x = _inputs(*dims, seed=11 + sum(dims))
    out = getattr(fh, entry)(x)
    assert out.Y.dtype == np.float32 and out.I.dtype == np.int32 and out.Y.shape == (dims[0], dims[3])
    Yr, Ir = orc.forward(x.H, x.E, x.b, x.mask)
    ok, rep = orc.check_forward(x.H, x.E, x.b, x.mask, out.Y, out.I, Yr, Ir, rtol=RTOL, atol=ATOL)
    assert ok, rep


def test_mirror_backward_vs_oracle_and_saved_state(cuda_device):
    from paper_2603_25011_b200 import fusedhead as fh
    x = _inputs(3, 70, 128, 900, seed=5)
    out = fh.forward_fully_fused(x)
    saved = fh.SavedSparseState.from_output(out)
    assert saved.nbytes == 3 * 900 * 8            # O(B·V), independent of S (fused.py:67-80)
    dY = orc.seeded_uniform((3, 900), 6)
    g = fh.backward_fused(x, saved, dY)
    dH_r, dE_r, db_r = orc.backward(x.H, x.E, x.b, out.Y, out.I, dY)
    assert _close(g.dH, dH_r) and _close(g.dE, dE_r) and _close(g.db, db_r)
    g0 = fh.backward_fused(x, saved, dY, include_bias_grad=False)     # fused.py:221,264
    assert not g0.db.any() and np.array_equal(g0.dE, g.dE)


def test_mirror_strategy_runner_signature(cuda_device):
    # bench.py:98-104: runner(inputs, cfg, tracker) -> HeadOutput; tracker records the saved bytes.
    from paper_2603_25011_b200 import fusedhead as fh

    class Tracker:
        saved = 0

        def note_saved(self, n):
            self.saved += n

    runners = {}
    fh.register_strategy(runners)
    x = _inputs(2, 16, 32, 100, seed=9)
    t = Tracker()
    out = runners[fh.STRATEGY_NAME](x, fh.TileConfig.default_for(x.dims), t)
    assert t.saved == out.Y.nbytes + out.I.nbytes
    Yr, Ir = orc.forward(x.H, x.E, x.b, x.mask)
    assert orc.check_forward(x.H, x.E, x.b, x.mask, out.Y, out.I, Yr, Ir, rtol=RTOL, atol=ATOL)[0]


def test_mirror_reference_errors(cuda_device):
    # reference.py:32-46 (inputs) and fused.py:240-245 (backward shapes) -> ValueError.
    from paper_2603_25011_b200 import fusedhead as fh
    x = _inputs(2, 3, 8, 5, seed=1)
    bad = fh.HeadInputs(x.dims, x.H, x.E, x.b, (x.mask * 2).astype(np.uint8))
    with pytest.raises(ValueError):
        fh.forward_fully_fused(bad)
    nan = fh.HeadInputs(x.dims, x.H.copy(), x.E, x.b, x.mask)
    nan.H[0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        fh.forward_hybrid(nan)
    out = fh.forward_fully_fused(x)
    with pytest.raises(ValueError):
        fh.backward_fused(x, fh.SavedSparseState.from_output(out), np.zeros((2, 4), np.float32))


def test_mirror_validation_messages_match_reference_validate(cuda_device):
    """The drop-in checks layout on the host and values on the device, with
    the exact ValueError of the reference's HeadInputs.validate
    (reference.py:30-46) for every failure, in the same precedence."""
    from paper_2603_25011_b200 import fusedhead as fh
    x = _inputs(2, 3, 8, 5, seed=2)

    def variant(**kw):
        f = {"H": x.H.copy(), "E": x.E.copy(), "b": x.b.copy(), "mask": x.mask.copy()}
        f.update(kw)
        return fh.HeadInputs(x.dims, f["H"], f["E"], f["b"], f["mask"])

    def poke(a, idx, val):
        a = a.copy()
        a[idx] = val
        return a

    cases = [
        variant(H=x.H[:, :2]), variant(H=x.H.astype(np.float64)), variant(E=x.E.T.copy()),
        variant(b=x.b[:4]), variant(mask=x.mask.astype(np.int32)),
        variant(H=poke(x.H, (1, 2, 3), np.nan)), variant(E=poke(x.E, (4, 0), np.inf)),
        variant(b=poke(x.b, 2, -np.inf)), variant(mask=poke(x.mask, (0, 1), 3)),
        # several faults at once: the first in the reference's order wins
        variant(H=poke(x.H, (0, 0, 0), np.nan), E=poke(x.E, (0, 0), np.nan), mask=poke(x.mask, (0, 0), 2)),
        variant(b=poke(x.b, 0, np.nan), mask=poke(x.mask, (0, 0), 2)),
    ]
    for bad in cases:
        with pytest.raises(ValueError) as ref:
            bad.validate()
        for entry in (fh.forward_fully_fused, fh.forward_hybrid):
            with pytest.raises(ValueError) as got:
                entry(bad)
            assert str(got.value) == str(ref.value)


def test_mirror_zero_inputs_and_all_masked(cuda_device):
    # test_reference.py:33-39 (zeros -> Y = 0, I = 0) and :72-79 (all-masked row).
    from paper_2603_25011_b200 import fusedhead as fh
    d = fh.Dims(2, 4, 8, 6)
    z = fh.HeadInputs(d, np.zeros((2, 4, 8), np.float32), np.zeros((6, 8), np.float32),
                      np.zeros(6, np.float32), np.ones((2, 4), np.uint8))
    out = fh.forward_fully_fused(z)
    assert not out.Y.any() and not out.I.any()
    x = _inputs(2, 4, 8, 6, seed=3)
    x.mask[1] = 0
    out = fh.forward_fully_fused(x)
    assert not out.Y[1].any() and not out.I[1].any()
