"""The reference's own harness driving the B200 operators.

``fusedhead.drop_in()`` swaps ``forward_hybrid`` / ``forward_fully_fused`` /
``backward_fused`` in the installed reference (baseline/_ref) for the GPU
entry points and registers the ``"b200"`` runner in the reference's real
``STRATEGY_RUNNERS``; the reference's UNMODIFIED ``run_check``,
``run_gradcheck`` and ``run_sweep`` (bench.py:193-368) then run on the B200
at the reference's own tolerances (Y rel 1e-5, backward 1e-5, FD 1e-4,
bench.py:41-46) — possible because the numpy drop-in computes fp32 inputs at
fp32 accuracy (exact bf16x3 split, head.sparton_forward_fp32).  Ports of
test_bench_cli.py:44-142 and test_acceptance.py criteria 5, 6 and 9.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture()
def ref(cuda_device):
    from paper_2603_25011_b200 import fusedhead as fh
    import fusedhead
    from fusedhead import bench
    return fh, fusedhead, bench


@pytest.mark.parametrize("dims,seed", [((2, 3, 4, 5), 42), ((2, 1, 4, 5), 7), ((3, 17, 24, 40), 3),
                                       ((2, 64, 96, 300), 11)])
def test_run_check_passes_on_b200(ref, dims, seed):
    fh, fusedhead, bench = ref
    with fh.drop_in():
        assert bench.forward_hybrid is fh.forward_hybrid
        result = bench.run_check(fusedhead.Dims(*dims), seed)     # the reference's tile-config grid
    assert result.passed, "\n".join(result.lines)
    assert result.lines[-1] == "PASS"
    assert bench.forward_hybrid is not fh.forward_hybrid       # restored on exit


def test_run_check_corrupted_b200_output_fails_and_names_entry(ref):
    fh, fusedhead, bench = ref
    with fh.drop_in():
        result = bench.run_check(fusedhead.Dims(2, 3, 4, 5), 42, corrupt=(1, 3))
    text = "\n".join(result.lines)
    assert not result.passed and "(b=1, v=3)" in text and "FAIL" in text


@pytest.mark.parametrize("dims,seed", [((2, 3, 4, 5), 42), ((1, 2, 2, 2), 0)])
def test_run_gradcheck_passes_on_b200(ref, dims, seed):
    fh, fusedhead, bench = ref
    with fh.drop_in():
        result = bench.run_gradcheck(fusedhead.Dims(*dims), seed)
    assert result.passed, "\n".join(result.lines)


def test_bf16_precision_fails_reference_tolerance_but_meets_north_star(ref):
    """The bf16 mode rounds H/E to 8-bit significands: it is outside the
    reference's fp32 tolerances (so run_check reports FAIL) while within the
    north-star rtol 1e-2 / atol 1e-3 — the reason fp32 is the drop-in default."""
    fh, fusedhead, bench = ref
    from fusedhead.reference import forward_eager
    dims = fusedhead.Dims(2, 16, 64, 200)
    with fh.drop_in(precision="bf16"):
        result = bench.run_check(dims, 5, configs=[fusedhead.TileConfig(1, 1)])
        x = fusedhead.HeadInputs.seeded(dims, 5, mask_keep=0.85)
        got = fh.forward_fully_fused(x)
    assert not result.passed
    want, _ = forward_eager(x, deterministic=True)
    assert np.all(np.abs(got.Y - want.Y) <= 1e-3 + 1e-2 * np.abs(want.Y))


def test_run_sweep_b200_rows_saved_state_and_flat_peak(ref):
    """Criterion 5 (saved bytes constant in S) and criterion 6 (flat head-owned
    peak across S) through the reference's run_sweep on the "b200" runner; the
    reference's four built-in names stay untouched (criterion 9)."""
    fh, fusedhead, bench = ref
    spec = bench.SweepSpec(axis="seq", values=[8, 16, 32, 64], base=fusedhead.Dims(4, 64, 16, 256),
                           strategies=["b200"], repeats=2, warmup=1, seed=6, tile=(64, 4))
    with fh.drop_in():
        records = bench.run_sweep(spec)
        assert bench.STRATEGY_NAMES == ("eager", "compiled-sim", "hybrid", "fully_fused")
    assert "b200" not in bench.STRATEGY_RUNNERS
    b200 = [r for r in records if r.strategy == "b200"]
    assert [r.dims.S for r in b200] == [8, 16, 32, 64]
    assert all(not r.is_oom and r.saved_bytes == 4 * 256 * 8 for r in b200)
    assert len({r.peak_bytes for r in b200}) == 1 and b200[0].peak_bytes == 4 * 256 * 8
    text = bench.records_to_csv(records)
    width = len(bench.BENCH_CSV_HEADER.split(","))
    assert all(len(line.split(",")) == width for line in text.splitlines())


def test_run_sweep_b200_oom_sentinel_under_cap(ref):
    """memtrack.py:18-28,43-51 / bench.py:220-221: a tracker cap below the
    head-owned (Y, I) bytes gives the reference's OOM sentinel row."""
    fh, fusedhead, bench = ref
    spec = bench.SweepSpec(axis="vocab", values=[64, 1024], base=fusedhead.Dims(4, 8, 16, 64),
                           strategies=["b200"], repeats=1, warmup=0, mem_cap_bytes=4 * 64 * 8)
    with fh.drop_in():
        records = bench.run_sweep(spec)
    assert len(records) == 2
    assert not records[0].is_oom and records[0].peak_bytes == 4 * 64 * 8
    assert records[1].is_oom and "OOM" in records[1].to_csv_row()


def test_tracker_cap_raises_reference_exception(ref):
    fh, fusedhead, bench = ref
    x = fusedhead.HeadInputs.seeded(fusedhead.Dims(2, 4, 8, 100), 1)
    t = fusedhead.AllocTracker(cap_bytes=100)
    with pytest.raises(fusedhead.AllocationCapExceeded):
        fh.forward_fully_fused(x, None, t)
    assert t.current_bytes == 0
    t2 = fusedhead.AllocTracker()
    fh.forward_fully_fused(x, None, t2)
    assert t2.current_bytes == 0 and t2.peak_bytes == 2 * 100 * 8 and t2.saved_bytes == 2 * 100 * 8
