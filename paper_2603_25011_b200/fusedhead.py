"""Drop-in mirror of the reference's ``fusedhead`` operator API, running on B200.

Same names, signatures, dataclasses and error behaviour as
/root/reference/pkg/src/fusedhead (``__init__.py:27-46``): numpy arrays in,
numpy arrays out, so the reference's callers (its bench harness
``STRATEGY_RUNNERS`` at bench.py:98-104, its tests) can drive the GPU kernels
unchanged.  Objects of the reference's own dataclasses are accepted too
(duck typing on ``.dims/.H/.E/.b/.mask`` and ``.Y/.I``).

Numerics: H and E are rounded to bf16 (round-to-nearest-even) at the upload
boundary and products accumulate in fp32 on the tensor cores; Y and the
gradients are fp32.  Parity with the fp32 reference is therefore within the
north-star tolerance (rtol 1e-2, atol 1e-3) and argmax-exact except at
documented near-ties.  ``TileConfig`` is accepted and
validated for API compatibility; the GPU tile shapes are compile-time
constants, so vocab_tile / batch_tile / num_threads do not change results.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np
import torch

from .head import sparton_backward, sparton_forward

MAX_ADDRESSABLE = 2**63 - 1
_TILE_BUFFER_BUDGET = 1 << 20
STRATEGY_NAME = "b200"

_SM64_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_SM64_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_SM64_MIX2 = np.uint64(0x94D049BB133111EB)


# ---------------------------------------------------------------- types (tensor.py / reference.py / fused.py)

@dataclass(frozen=True)
class Dims:
    """Problem sizes B, S, D, V (tensor.py:22-44), with the same overflow guard."""

    B: int
    S: int
    D: int
    V: int

    def __post_init__(self):
        for name in ("B", "S", "D", "V"):
            value = getattr(self, name)
            if not isinstance(value, int) or value < 1:
                raise ValueError(f"dims.{name} must be a positive integer, got {value!r}")
        if self.B * self.S * self.D > MAX_ADDRESSABLE or self.B * self.V > MAX_ADDRESSABLE:
            raise OverflowError(f"dims {self} exceed the addressable size")

    def with_axis(self, axis: str, value: int) -> "Dims":
        field = {"batch": "B", "seq": "S", "vocab": "V"}.get(axis)
        if field is None:
            raise ValueError(f"unknown axis {axis!r}")
        return replace(self, **{field: value})


@dataclass(frozen=True)
class Uniform:
    lo: float = -1.0
    hi: float = 1.0


@dataclass(frozen=True)
class Constant:
    value: float = 0.0


def splitmix64(seed: int, count: int) -> np.ndarray:
    """Counter-based SplitMix64 stream, word i = mix(seed + (i+1)·γ) (tensor.py:58-69)."""
    state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    idx = np.arange(1, count + 1, dtype=np.uint64)
    z = state + idx * _SM64_GAMMA
    z = (z ^ (z >> np.uint64(30))) * _SM64_MIX1
    z = (z ^ (z >> np.uint64(27))) * _SM64_MIX2
    return z ^ (z >> np.uint64(31))


def _unit_floats(seed: int, count: int) -> np.ndarray:
    return (splitmix64(seed, count) >> np.uint64(11)).astype(np.float64) * (2.0**-53)


def seeded_tensor(shape, seed: int, dist=Uniform()) -> np.ndarray:
    """Deterministic float32 tensor (tensor.py:91-105): same bytes everywhere."""
    shape = tuple(int(n) for n in shape)
    if not shape or any(n < 1 for n in shape):
        raise ValueError(f"shape must be nonempty with positive entries, got {shape}")
    n = 1
    for d in shape:
        n *= d
        if n > MAX_ADDRESSABLE:
            raise OverflowError(f"shape {shape} overflows the addressable size")
    if isinstance(dist, Constant):
        return np.full(shape, np.float32(dist.value), dtype=np.float32)
    if not isinstance(dist, Uniform):
        raise TypeError(f"unsupported distribution {dist!r}")
    if not dist.lo < dist.hi:
        raise ValueError(f"uniform bounds must satisfy lo < hi, got {dist}")
    vals = dist.lo + (dist.hi - dist.lo) * _unit_floats(seed, n)
    return vals.astype(np.float32).reshape(shape)


def seeded_mask(batch: int, seq: int, seed: int, keep: float = 1.0) -> np.ndarray:
    """{0,1} uint8 mask, each position kept with probability ``keep`` (tensor.py:108-115)."""
    if not 0.0 <= keep <= 1.0:
        raise ValueError(f"keep must lie in [0, 1], got {keep}")
    if keep >= 1.0:
        return np.ones((batch, seq), np.uint8)
    return (_unit_floats(seed, batch * seq) < keep).astype(np.uint8).reshape(batch, seq)


def _require_finite(arr: np.ndarray, name: str) -> None:
    if not np.isfinite(arr).all():
        raise ValueError(f"{name} contains NaN or Inf")


@dataclass
class HeadInputs:
    """(H, E, b, mask) quadruple with the reference's validation (reference.py:22-69)."""

    dims: Dims
    H: np.ndarray
    E: np.ndarray
    b: np.ndarray
    mask: np.ndarray

    def validate(self) -> None:
        _validate_inputs(self)

    @classmethod
    def seeded(cls, dims: Dims, seed: int, *, mask: np.ndarray | None = None, mask_keep: float = 1.0,
               dist=Uniform(-1.0, 1.0)) -> "HeadInputs":
        if mask is None:
            mask = seeded_mask(dims.B, dims.S, seed + 3, keep=mask_keep)
        inputs = cls(dims=dims,
                     H=seeded_tensor((dims.B, dims.S, dims.D), seed, dist),
                     E=seeded_tensor((dims.V, dims.D), seed + 1, dist),
                     b=seeded_tensor((dims.V,), seed + 2, dist),
                     mask=np.ascontiguousarray(mask, dtype=np.uint8))
        inputs.validate()
        return inputs


@dataclass
class HeadOutput:
    Y: np.ndarray
    I: np.ndarray


@dataclass
class HeadGradients:
    dH: np.ndarray
    dE: np.ndarray
    db: np.ndarray


@dataclass
class SavedSparseState:
    """(Y, I): O(B·V) bytes, independent of S (fused.py:67-80)."""

    Y: np.ndarray
    I: np.ndarray

    @classmethod
    def from_output(cls, out) -> "SavedSparseState":
        return cls(Y=out.Y, I=out.I)

    @property
    def nbytes(self) -> int:
        return self.Y.nbytes + self.I.nbytes


@dataclass(frozen=True)
class TileConfig:
    """Tiling policy (fused.py:37-64).  Validated for compatibility; the GPU
    tiles are fixed (128·CG vocab rows x 256 positions x 64 K per stage)."""

    vocab_tile: int
    batch_tile: int
    deterministic: bool = False
    num_threads: int = 1

    def validate_for(self, dims) -> None:
        if not 1 <= self.vocab_tile <= dims.V:
            raise ValueError(f"vocab_tile must lie in [1, {dims.V}], got {self.vocab_tile}")
        if not 1 <= self.batch_tile <= dims.B:
            raise ValueError(f"batch_tile must lie in [1, {dims.B}], got {self.batch_tile}")
        if self.num_threads < 1:
            raise ValueError(f"num_threads must be positive, got {self.num_threads}")

    @classmethod
    def default_for(cls, dims, *, deterministic: bool = False, num_threads: int = 1) -> "TileConfig":
        c = min(64, dims.V)
        bt = min(8, dims.B)
        while bt > 1 and bt * dims.S * c * 4 > _TILE_BUFFER_BUDGET:
            bt //= 2
        while c > 1 and bt * dims.S * c * 4 > _TILE_BUFFER_BUDGET:
            c //= 2
        return cls(vocab_tile=c, batch_tile=bt, deterministic=deterministic, num_threads=num_threads)


def _validate_inputs(inputs) -> None:
    """reference.py:32-46, verbatim in behaviour: shapes, dtypes, finiteness, mask values."""
    d = inputs.dims
    if inputs.H.shape != (d.B, d.S, d.D) or inputs.H.dtype != np.float32:
        raise ValueError(f"H must be float32 {(d.B, d.S, d.D)}, got {inputs.H.dtype} {inputs.H.shape}")
    if inputs.E.shape != (d.V, d.D) or inputs.E.dtype != np.float32:
        raise ValueError(f"E must be float32 {(d.V, d.D)}, got {inputs.E.dtype} {inputs.E.shape}")
    if inputs.b.shape != (d.V,) or inputs.b.dtype != np.float32:
        raise ValueError(f"b must be float32 {(d.V,)}, got {inputs.b.dtype} {inputs.b.shape}")
    if inputs.mask.shape != (d.B, d.S) or inputs.mask.dtype != np.uint8:
        raise ValueError(f"mask must be uint8 {(d.B, d.S)}, got {inputs.mask.dtype} {inputs.mask.shape}")
    _require_finite(inputs.H, "H")
    _require_finite(inputs.E, "E")
    _require_finite(inputs.b, "b")
    if not np.all((inputs.mask == 0) | (inputs.mask == 1)):
        raise ValueError("mask values must be exactly 0 or 1")


# ---------------------------------------------------------------- device staging

def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the b200 fused head needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _upload_bf16(x: np.ndarray, dev) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(dev).to(torch.bfloat16)


def _run_forward(inputs, tracker) -> HeadOutput:
    dev = _device()
    d = inputs.dims
    H = _upload_bf16(inputs.H, dev)
    E = _upload_bf16(inputs.E, dev)
    b = torch.from_numpy(np.ascontiguousarray(inputs.b, dtype=np.float32)).to(dev)
    m = torch.from_numpy(np.ascontiguousarray(inputs.mask, dtype=np.uint8)).to(dev)
    Y, I = sparton_forward(H, E, b, m)
    out = HeadOutput(Y=Y.cpu().numpy(), I=I.cpu().numpy())
    if tracker is not None:
        tracker.note_saved(out.Y.nbytes + out.I.nbytes)
    assert out.Y.shape == (d.B, d.V)
    return out


def forward_hybrid(inputs, cfg: TileConfig | None = None, tracker=None) -> HeadOutput:
    """Drop-in for fused.forward_hybrid (fused.py:115-157) on the B200 kernel."""
    _validate_inputs(inputs)
    (cfg or TileConfig.default_for(inputs.dims)).validate_for(inputs.dims)
    return _run_forward(inputs, tracker)


def forward_fully_fused(inputs, cfg: TileConfig | None = None, tracker=None) -> HeadOutput:
    """Drop-in for fused.forward_fully_fused (fused.py:160-212): on B200 the
    streaming reduction and the hybrid are the same single fused kernel."""
    _validate_inputs(inputs)
    (cfg or TileConfig.default_for(inputs.dims)).validate_for(inputs.dims)
    return _run_forward(inputs, tracker)


def backward_fused(inputs, saved, dY: np.ndarray, cfg: TileConfig | None = None, *,
                   include_bias_grad: bool = True) -> HeadGradients:
    """Drop-in for fused.backward_fused (fused.py:215-278): shape checks only,
    gradients from (Y, I) alone, fp32 outputs."""
    d = inputs.dims
    (cfg or TileConfig.default_for(d)).validate_for(d)
    if inputs.H.shape != (d.B, d.S, d.D) or inputs.E.shape != (d.V, d.D):
        raise ValueError("input shapes disagree with dims")
    if saved.Y.shape != (d.B, d.V) or saved.I.shape != (d.B, d.V):
        raise ValueError(f"saved state must have shape {(d.B, d.V)}")
    if dY.shape != (d.B, d.V):
        raise ValueError(f"dY must have shape {(d.B, d.V)}, got {dY.shape}")
    dev = _device()
    H = _upload_bf16(inputs.H, dev)
    E = _upload_bf16(inputs.E, dev)
    Y = torch.from_numpy(np.ascontiguousarray(saved.Y, dtype=np.float32)).to(dev)
    I = torch.from_numpy(np.ascontiguousarray(saved.I, dtype=np.int32)).to(dev)
    g = torch.from_numpy(np.ascontiguousarray(dY, dtype=np.float32)).to(dev)
    dH, dE, db = sparton_backward(H, E, Y, I, g, include_bias_grad=include_bias_grad)
    return HeadGradients(dH=dH.cpu().numpy(), dE=dE.cpu().numpy(), db=db.cpu().numpy())


def run_b200(inputs, cfg: TileConfig, tracker) -> HeadOutput:
    """Strategy runner with the reference's signature ``runner(inputs, cfg, tracker)``
    (bench.py:98-104)."""
    return forward_fully_fused(inputs, cfg, tracker)


def register_strategy(runners: dict) -> None:
    """Register the ``"b200"`` runner into a reference ``STRATEGY_RUNNERS`` dict.

    Only the dict passed in is touched (the reference's acceptance test counts
    exactly its four built-in strategy names, test_acceptance.py:278-283).
    """
    runners[STRATEGY_NAME] = run_b200
