"""Analytical traffic of the B200 plan, in the reference cost model's schema.

The reference models four CPU strategies by the bytes each plan must move by
construction (``fusedhead.costmodel``: ``eager_traffic`` / ``compiled_traffic``
/ ``fused_traffic``, /root/reference/pkg/src/fusedhead/costmodel.py:78-171,
CSV via ``reports_to_csv_rows`` :200-215 under ``COST_CSV_HEADER`` :24).
``b200_traffic`` adds the GPU plan as a fifth ``CostReport`` built from the
reference's own ``Stage`` / ``CostReport`` types, so the same table and CSV
carry it.  The counts are the compulsory HBM bytes of each kernel (every
operand read once, every result written once) — the ``algorithmic bytes``
the DESIGN.md rooflines use, and what the sweep's ``*_model_bytes`` columns
divide by the measured time:

* ``k1-fwd``   (K1): H, E, bias, mask in; Y, I out — logits never leave the SM.
* ``bwd-route`` (K3a): Y, I, dY in; (v, g) pair lists, per-(b, window, s)
  offsets and (staged regime) the per-(b, v) (s, g) records out.
* ``bwd-dE``   (K2s + db): H and the records in; dE and db out.
* ``bwd-dH``   (K3b): pair lists, offsets, E in; dH out.

``peak_activation_bytes`` is the backward's device workspace (the only
transient the head allocates: the forward keeps its tiles in shared and
tensor memory), ``saved_state_bytes`` the (Y, I) pair, B·V·8 — both as the
reference defines them (memtrack.py:31-60).  With few active pairs (the
sparse regime) the pair lists and gathers shrink; the model is the dense
upper bound, as the reference's is.

    python -m paper_2603_25011_b200.costmodel --dims 512x512x768x250002 [--csv PATH]
"""

from __future__ import annotations

import argparse
import sys

from .fusedhead import _ref

_cm = __import__(_ref.__name__ + ".costmodel", fromlist=["costmodel"])
COST_CSV_HEADER = _cm.COST_CSV_HEADER
Stage, CostReport, DtypeSpec = _cm.Stage, _cm.CostReport, _cm.DtypeSpec

RT_WIN = 8192          # csrc/sparton_bwd.cu: route window (vocab rows)
STAGED_MAX_S = 832     # csrc/sparton_bwd.cu: de_staged_rows() > 0


def workspace_bytes(B: int, S: int, D: int, V: int, grad_bytes: int = 2) -> int:
    """The backward workspace (``sparton_bwd_workspace_bytes``), restated
    (tests/test_abi.py::test_workspace_formula pins the two together)."""
    up = lambda x: (x + 255) // 256 * 256
    nwin = -(-V // RT_WIN)
    wpc = max(1, min(nwin, 32, (52 << 20) // (RT_WIN * D * 2)))
    nchunks = -(-nwin // wpc)
    staged = S <= STAGED_MAX_S
    total = up(B * V * 8) + up(B * nwin * (S + 1) * 4) + up(V * 4)
    if not staged and grad_bytes == 2:
        bc = min(B, max(32, (48 << 20) // (S * D * 2)))
        if -(-B // bc) > 1:
            total += up(V * D * 4)
    if grad_bytes == 2 and nchunks > 1:
        total += up(B * S * D * 4)
    if staged:
        total += up(B * (V + V % 2) * 8)
    return total + 256


def b200_traffic(dims, dt=None, grad_bytes: int = 2, backward: bool = True):
    """The B200 plan's compulsory HBM bytes per stage (``CostReport``)."""
    dt = dt or DtypeSpec()
    B, S, D, V = dims.B, dims.S, dims.D, dims.V
    a, ix = 2, dt.index_bytes        # H and E are bf16 on the device whatever the host dtype
    nwin = -(-V // RT_WIN)
    staged = S <= STAGED_MAX_S
    h, e, yi = B * S * D * a, V * D * a, B * V * (4 + ix)
    stages = [Stage("k1-fwd", h + e + V * 4 + B * S * 1, yi)]
    if backward:
        lists, offs = B * V * 8, B * nwin * (S + 1) * 4
        recs = B * V * 8 if staged else 0
        stages += [
            Stage("bwd-route", yi + B * V * 4, lists + offs + recs),
            Stage("bwd-dE", h + (recs if staged else lists + offs), V * D * grad_bytes + V * 4),
            Stage("bwd-dH", lists + offs + e, B * S * D * grad_bytes),
        ]
    peak = workspace_bytes(B, S, D, V, grad_bytes) if backward else 0
    rep = CostReport("b200", stages, peak_activation_bytes=peak, saved_state_bytes=B * V * (4 + ix))
    rep.validate()
    return rep


def all_reports(dims, dt=None):
    """The reference's four strategies plus the B200 plan."""
    dt = dt or DtypeSpec()
    return _cm.all_reports(dims, dt) + [b200_traffic(dims, dt)]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="analytical traffic table incl. the b200 plan")
    ap.add_argument("--dims", default="512x512x768x30522", help="BxSxDxV")
    ap.add_argument("--act-bytes", type=int, choices=(2, 4), default=2)
    ap.add_argument("--csv", metavar="PATH", default=None)
    a = ap.parse_args(argv)
    try:
        B, S, D, V = (int(x) for x in a.dims.lower().split("x"))
        dims = _ref.Dims(B, S, D, V)
    except (ValueError, TypeError) as exc:
        print(f"bad --dims: {exc}", file=sys.stderr)
        return 2
    reports = all_reports(dims, DtypeSpec(activation_bytes=a.act_bytes))
    if a.csv:
        with open(a.csv, "w") as f:
            f.write("\n".join([COST_CSV_HEADER] + _cm.reports_to_csv_rows(reports)) + "\n")
    else:
        print(_cm.format_reports(reports))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
