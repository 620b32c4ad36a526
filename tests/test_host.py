"""CPU: host-side logic of the product package — the reference-API mirror's
validation and error types, the strategy registry hook, the no-CPU-fallback
rule, and the vocab-shard arithmetic."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2603_25011_b200 import fusedhead as fh
from paper_2603_25011_b200.sharded import shard_range


def test_dims_validation_matches_reference_contract():
    with pytest.raises(ValueError):
        fh.Dims(0, 1, 1, 1)
    with pytest.raises(OverflowError):
        fh.Dims(2**40, 2**40, 2**40, 1)
    assert fh.Dims(2, 3, 4, 5).with_axis("vocab", 9).V == 9
    with pytest.raises(ValueError):
        fh.Dims(2, 3, 4, 5).with_axis("depth", 1)


def test_headinputs_validate_errors():
    inp = fh.HeadInputs.seeded(fh.Dims(2, 3, 4, 5), 1)
    bad = fh.HeadInputs(inp.dims, inp.H.astype(np.float64), inp.E, inp.b, inp.mask)
    with pytest.raises(ValueError):
        bad.validate()
    nan = fh.HeadInputs(inp.dims, inp.H.copy(), inp.E, inp.b, inp.mask)
    nan.H[0, 0, 0] = np.nan
    with pytest.raises(ValueError):
        nan.validate()
    m = inp.mask.copy()
    m[0, 0] = 2
    with pytest.raises(ValueError):
        fh.HeadInputs(inp.dims, inp.H, inp.E, inp.b, m).validate()


def test_tileconfig_validation():
    d = fh.Dims(2, 3, 4, 5)
    with pytest.raises(ValueError):
        fh.TileConfig(0, 1).validate_for(d)
    with pytest.raises(ValueError):
        fh.TileConfig(1, 3).validate_for(d)
    with pytest.raises(ValueError):
        fh.TileConfig(1, 1, num_threads=0).validate_for(d)
    c = fh.TileConfig.default_for(fh.Dims(16, 4096, 8, 1024))
    assert c.batch_tile * 4096 * c.vocab_tile * 4 <= 1 << 20


def test_register_strategy_touches_only_given_dict():
    runners = {"eager": object()}
    fh.register_strategy(runners)
    assert runners["b200"] is fh.run_b200 and len(runners) == 2


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU path")
def test_no_cpu_fallback():
    inp = fh.HeadInputs.seeded(fh.Dims(2, 3, 8, 5), 1)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fh.forward_hybrid(inp)
    from paper_2603_25011_b200 import sparton_forward
    H = torch.zeros((2, 3, 8), dtype=torch.bfloat16)
    E = torch.zeros((5, 8), dtype=torch.bfloat16)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sparton_forward(H, E, torch.zeros(5), torch.ones((2, 3), dtype=torch.uint8))
    from paper_2603_25011_b200 import quantize_e4m3, sparton_forward_fp8
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sparton_forward_fp8(H, E, torch.zeros(5), torch.ones((2, 3), dtype=torch.uint8))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        quantize_e4m3(torch.zeros(16, dtype=torch.bfloat16))


def test_backward_shape_errors_before_device_check():
    inp = fh.HeadInputs.seeded(fh.Dims(2, 3, 4, 5), 42)
    saved = fh.SavedSparseState(np.zeros((2, 3), np.float32), np.zeros((2, 3), np.int32))
    with pytest.raises(ValueError):
        fh.backward_fused(inp, saved, np.zeros((2, 5), np.float32))
    assert fh.SavedSparseState(np.zeros((2, 5), np.float32), np.zeros((2, 5), np.int32)).nbytes == 80


@pytest.mark.parametrize("V,P", [(250002, 8), (250002, 4), (250002, 2), (30522, 8), (5, 4), (1, 3)])
def test_shard_ranges_partition_vocab(V, P):
    covered = np.zeros(V, np.int32)
    Vp = None
    for r in range(P):
        v0, v1, vp = shard_range(V, P, r)
        Vp = vp if Vp is None else Vp
        assert vp == Vp and 0 <= v1 - v0 <= Vp
        covered[v0:v1] += 1
    assert np.all(covered == 1)
    assert Vp * P >= V
    with pytest.raises(ValueError):
        shard_range(V, P, P)


def test_sweep_rejects_bad_axis_and_empty_values():
    from paper_2603_25011_b200 import sweep
    with pytest.raises(ValueError):
        sweep.run_sweep((2, 3, 8, 5), "Q", [1])
    with pytest.raises(ValueError):
        sweep.run_sweep((2, 3, 8, 5), "V", [])
    assert sweep.main(["--base", "1,2,3"]) == 2


def test_bench_launch_count_matches_library_constants():
    # bench.py's gpu_launches claim is derived from the library's dH chunking.
    import re
    from pathlib import Path

    import bench

    src = (Path(__file__).resolve().parent.parent / "paper_2603_25011_b200/csrc/sparton_bwd.cu").read_text()
    chunk = int(re.search(r"constexpr long long DH_CHUNK_BYTES = (\d+)ll << 20;", src).group(1))
    win = int(re.search(r"constexpr int RT_WIN = (\d+);", src).group(1))
    assert bench.DH_CHUNK_MB == chunk and win == 8192
    cfg3 = {"D": 768}
    assert bench.launches_per_step(cfg3, 250002) == 6 + 8     # 31 windows, 4 per 52 MB pass
    assert bench.launches_per_step(cfg3, 30522) == 6 + 1


def test_cost_model_b200_plan():
    """costmodel.b200_traffic: the forward's compulsory bytes (H + E + bias +
    mask in, Y + I out; 1.812 GB at cfg3), its peak equal to
    the library's workspace query, and the reference's CSV schema."""
    import io
    import contextlib
    from paper_2603_25011_b200 import _lib, costmodel as cm
    from paper_2603_25011_b200.fusedhead import Dims
    rep = cm.b200_traffic(Dims(512, 512, 768, 250002))
    fwd = rep.stages[0]
    assert fwd.label == "k1-fwd" and abs((fwd.bytes_read + fwd.bytes_written) / 1e9 - 1.812) < 0.001
    assert rep.saved_state_bytes == 512 * 250002 * 8
    lib = _lib.load()
    for dims in [(512, 512, 768, 250002), (512, 1024, 768, 250002), (2, 3, 8, 5), (4, 300, 256, 1000),
                 (2048, 512, 1024, 250002)]:
        for gd, gb in ((_lib.SPARTON_F32, 4), (_lib.SPARTON_BF16, 2)):
            assert lib.sparton_bwd_workspace_bytes(*dims, gd) == cm.workspace_bytes(*dims, gb), dims
    rows = cm._cm.reports_to_csv_rows(cm.all_reports(Dims(8, 128, 768, 30522)))
    b200 = [r for r in rows if r.startswith("b200,")]
    assert [r.split(",")[1] for r in b200] == ["k1-fwd", "bwd-route", "bwd-dE", "bwd-dH", "total"]
    assert all(len(r.split(",")) == len(cm.COST_CSV_HEADER.split(",")) for r in rows)
    out = io.StringIO()
    with contextlib.redirect_stdout(out):
        assert cm.main(["--dims", "8x128x768x30522"]) == 0
    assert "b200" in out.getvalue() and "fully_fused" in out.getvalue()
