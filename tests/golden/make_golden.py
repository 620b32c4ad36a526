"""Generate the golden fixtures under tests/golden/ by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src and
records, per case, the reference's own outputs:

  * forward_eager(deterministic=True)            -> Y, I   (reference.py:103-125)
  * eval_head_f64                                -> Y64, I64 (reference.py:186-198)
  * backward_fused from the reference's (Y, I)   -> dH, dE, db (fused.py:215-278)
  * backward_eager                               -> dH_e, dE_e, db_e (reference.py:143-183)

Inputs are HeadInputs.seeded(dims, seed, mask_keep=...) (reference.py:48-69),
optionally rounded to bf16 before the reference sees them (the "bf16" cases
are exactly what the GPU kernels compute on), and are stored in the fixture
so GPU tests never need the generator.  The missing SplitMix64 golden of the
reference (tests/data/seeded_2x3x4_seed42.npy, test_tensor.py:12) is
regenerated here from tensor.py:58-105 and stored as splitmix_golden.npz.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def bf16_round(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)


# name, (B, S, D, V), seed, mask_keep, dY_seed, bf16, explicit mask
CASES = [
    ("small_instance", (2, 3, 4, 5), 42, None, 9, False, [[1, 1, 0], [1, 1, 1]]),
    ("grid0", (1, 1, 2, 1), 700, 0.8, 800, False, None),
    ("grid1", (2, 3, 4, 5), 701, 0.8, 801, False, None),
    ("grid2", (4, 8, 2, 16), 702, 0.8, 802, False, None),
    ("grid3", (1, 32, 16, 5), 703, 0.8, 803, False, None),
    ("grid4", (2, 8, 4, 64), 704, 0.8, 804, False, None),
    ("grid5", (4, 3, 16, 16), 705, 0.8, 805, False, None),
    ("all_masked_row", (2, 3, 4, 5), 8, None, 10, False, [[0, 0, 0], [1, 1, 1]]),
    ("bf16_s300", (4, 64, 64, 300), 7, 0.85, 16, True, None),
    ("bf16_bert_slice", (2, 128, 768, 256), 11, 0.85, 20, True, None),
    ("bf16_partial_tiles", (3, 300, 64, 389), 13, 0.7, 22, True, None),
]


def main() -> int:
    sys.path.insert(0, str(REF_SRC))
    import fusedhead as fh  # the reference, read-only

    for name, dims_t, seed, keep, dy_seed, bf16, mask in CASES:
        dims = fh.Dims(*dims_t)
        if mask is not None:
            inputs = fh.HeadInputs.seeded(dims, seed, mask=np.array(mask, np.uint8))
        else:
            inputs = fh.HeadInputs.seeded(dims, seed, mask_keep=keep)
        if bf16:
            inputs = fh.HeadInputs(dims, bf16_round(inputs.H), bf16_round(inputs.E), inputs.b, inputs.mask)
            inputs.validate()
        dY = fh.seeded_tensor((dims.B, dims.V), dy_seed)
        out, saved = fh.forward_eager(inputs, deterministic=True)
        y64, i64 = fh.eval_head_f64(inputs.H, inputs.E, inputs.b, inputs.mask)
        gf = fh.backward_fused(inputs, fh.SavedSparseState.from_output(out), dY)
        ge = fh.backward_eager(inputs, saved, out, dY)
        hyb = fh.forward_hybrid(inputs, fh.TileConfig.default_for(dims, deterministic=True))
        assert np.array_equal(hyb.I, out.I) and hyb.Y.tobytes() == out.Y.tobytes()
        extra = {} if bf16 else dict(dH_e=ge.dH, dE_e=ge.dE, db_e=ge.db)
        np.savez_compressed(
            OUT / f"{name}.npz",
            dims=np.array(dims_t, np.int64), seed=seed, dY_seed=dy_seed, bf16=bf16,
            H=inputs.H, E=inputs.E, b=inputs.b, mask=inputs.mask, dY=dY,
            Y=out.Y, I=out.I, Y64=y64, I64=i64,
            dH=gf.dH, dE=gf.dE, db=gf.db, **extra,
        )
        print(f"{name}: dims={dims_t} active={(out.Y > 0).mean():.3f}")

    t = fh.seeded_tensor((2, 3, 4), 42, fh.Uniform(-1.0, 1.0))
    words = fh.splitmix64(42, 16)
    m = fh.seeded_mask(4, 8, 5, keep=0.5)
    np.savez_compressed(OUT / "splitmix_golden.npz", seeded_2x3x4_seed42=t, splitmix_42_16=words,
                        mask_4x8_seed5_keep05=m)
    print("splitmix_golden written")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
