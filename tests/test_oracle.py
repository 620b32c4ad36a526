"""CPU: pin the oracle (oracle/sparton_oracle.py) against golden fixtures made by
running the reference itself (tests/golden/make_golden.py), plus the
reference's known-answer tests restated.  No GPU needed."""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import GOLDEN, golden_names, load_golden
from oracle import sparton_oracle as orc


def test_splitmix_golden():
    with np.load(GOLDEN / "splitmix_golden.npz") as z:
        assert orc.splitmix64(42, 16).tobytes() == z["splitmix_42_16"].tobytes()
        assert orc.seeded_uniform((2, 3, 4), 42).tobytes() == z["seeded_2x3x4_seed42"].tobytes()
        assert np.array_equal(orc.seeded_mask(4, 8, 5, keep=0.5), z["mask_4x8_seed5_keep05"])


@pytest.mark.parametrize("name", golden_names())
def test_inputs_regenerate_bit_exactly(name):
    g = load_golden(name)
    B, S, D, V = (int(x) for x in g["dims"])
    if name in ("small_instance", "all_masked_row"):
        pytest.skip("explicit mask")
    keep = 0.85 if bool(g["bf16"]) else 0.8
    if name == "bf16_partial_tiles":
        keep = 0.7
    H, E, b, m = orc.seeded_inputs(B, S, D, V, int(g["seed"]), mask_keep=keep)
    if bool(g["bf16"]):
        H, E = orc.bf16_round(H), orc.bf16_round(E)
    assert H.tobytes() == g["H"].tobytes() and E.tobytes() == g["E"].tobytes()
    assert b.tobytes() == g["b"].tobytes() and np.array_equal(m, g["mask"])
    assert orc.seeded_uniform((B, V), int(g["dY_seed"])).tobytes() == g["dY"].tobytes()


@pytest.mark.parametrize("name", golden_names())
def test_forward_deterministic_bit_exact(name):
    g = load_golden(name)
    Y, I = orc.forward(g["H"], g["E"], g["b"], g["mask"], deterministic=True)
    assert Y.tobytes() == g["Y"].tobytes()
    assert np.array_equal(I, g["I"])


@pytest.mark.parametrize("name", golden_names())
def test_forward_blas_close_and_f64(name):
    g = load_golden(name)
    Y, I = orc.forward(g["H"], g["E"], g["b"], g["mask"])
    assert np.all(np.abs(Y - g["Y"]) <= np.maximum(1e-7, 1e-5 * np.abs(g["Y"])))
    y64, _ = orc.forward_f64(g["H"], g["E"], g["b"], g["mask"])
    assert np.max(np.abs(y64 - g["Y64"])) == 0.0


@pytest.mark.parametrize("name", golden_names())
def test_backward_matches_reference(name):
    g = load_golden(name)
    dH, dE, db = orc.backward(g["H"], g["E"], g["b"], g["Y"], g["I"], g["dY"])
    # same algorithm, same fp32 order as fused.py:247-273 -> bit exact
    assert dH.tobytes() == g["dH"].tobytes()
    assert dE.tobytes() == g["dE"].tobytes()
    assert db.tobytes() == g["db"].tobytes()
    if "dH_e" in g:
        for got, ref in ((dH, g["dH_e"]), (dE, g["dE_e"]), (db, g["db_e"])):
            assert np.max(np.abs(got - ref)) < 1e-5


@pytest.mark.parametrize("name", [n for n in golden_names() if n.startswith("bf16")])
def test_slices_reproduce_full(name):
    g = load_golden(name)
    rows = [0, g["Y"].shape[0] - 1]
    dH_rows = orc.backward_rows(g["H"], g["E"], g["Y"], g["I"], g["dY"], rows)
    assert dH_rows.tobytes() == g["dH"][rows].tobytes()
    cols = np.arange(0, g["Y"].shape[1], 7)
    dE_c, db_c = orc.backward_cols(g["H"], g["Y"], g["I"], g["dY"], cols)
    assert dE_c.tobytes() == g["dE"][cols].tobytes()
    assert db_c.tobytes() == g["db"][cols].tobytes()


def test_known_answers():
    Y, I = orc.forward(np.array([[[1.0], [3.0]]], np.float32), np.array([[1.0]], np.float32),
                       np.zeros(1, np.float32), np.ones((1, 2), np.uint8))
    assert Y[0, 0] == pytest.approx(math.log(4.0), abs=1e-7) and I[0, 0] == 1
    Y, I = orc.forward(np.array([[[2.0], [2.0], [1.0]]], np.float32), np.array([[1.0]], np.float32),
                       np.zeros(1, np.float32), np.ones((1, 3), np.uint8))
    assert I[0, 0] == 0
    # masked exact zero beats a negative logit
    Y, I = orc.forward(np.array([[[-1.0], [-2.0]]], np.float32), np.array([[1.0]], np.float32),
                       np.zeros(1, np.float32), np.array([[1, 0]], np.uint8))
    assert Y[0, 0] == 0 and I[0, 0] == 1


def test_scalar_backward_closed_form():
    x, w = 0.7, 0.9
    H = np.full((1, 1, 1), x, np.float32)
    E = np.full((1, 1), w, np.float32)
    b = np.zeros(1, np.float32)
    Y, I = orc.forward(H, E, b, np.ones((1, 1), np.uint8))
    dH, dE, db = orc.backward(H, E, b, Y, I, np.ones((1, 1), np.float32))
    assert dH[0, 0, 0] == pytest.approx(w / (1 + x * w), rel=1e-6)
    assert dE[0, 0] == pytest.approx(x / (1 + x * w), rel=1e-6)
    assert db[0] == pytest.approx(1 / (1 + x * w), rel=1e-6)


def test_bf16_round_is_rne():
    x = np.array([1.0, 1.0 + 2**-8, 1.0 + 3 * 2**-8, -2.5, 3.0e-39], np.float32)
    r = orc.bf16_round(x)
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == np.float32(1.0 + 2**-6)
    assert r[3] == -2.5
    import torch
    t = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert r.tobytes() == t.tobytes()


def test_near_tie_rule():
    # identical rows -> exact tie -> always a near tie; distinct rows -> not
    H = np.array([[[1.0, 2.0], [1.0, 2.0], [0.0, 0.5]]], np.float32)
    E = np.array([[0.5, 0.25]], np.float32)
    b = np.zeros(1, np.float32)
    m = np.ones((1, 3), np.uint8)
    assert orc.near_tie_ok(H, E, b, m, 0, 0, 0, 1)
    assert not orc.near_tie_ok(H, E, b, m, 0, 0, 0, 2)


def test_check_forward_reports():
    H, E, b, m = orc.seeded_inputs(2, 5, 4, 6, 3)
    Y, I = orc.forward(H, E, b, m)
    ok, rep = orc.check_forward(H, E, b, m, Y, I, Y, I)
    assert ok and rep["idx_mismatch"] == 0
    Y2 = Y.copy()
    Y2[0, 0] += 1.0
    ok, rep = orc.check_forward(H, E, b, m, Y2, I, Y, I)
    assert not ok and rep["y_bad"] == 1
