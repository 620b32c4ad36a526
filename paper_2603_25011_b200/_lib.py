"""ctypes binding of the C ABI in ``include/sparton.h`` (``libsparton_b200.so``).

This is the only place Python touches the native library.  It raises loudly
when the library is missing — there is no CPU fallback anywhere on the
product path.  Status codes map onto the reference's exception types:
``SPARTON_EINVAL`` -> ``ValueError`` (reference.py:32-46, fused.py:240-245),
anything else -> ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libsparton_b200.so"


def _lib_path() -> Path:
    """The in-tree library.  ``SPARTON_LIB`` (A/B timing of two builds) is a
    development override honoured only under ``SPARTON_DEV=1`` — the same
    single gate the native library applies to its own experiment switches."""
    if os.environ.get("SPARTON_DEV") == "1" and os.environ.get("SPARTON_LIB"):
        return Path(os.environ["SPARTON_LIB"]).resolve()
    return LIB_PATH

SPARTON_OK = 0
SPARTON_EINVAL = 1
SPARTON_ECUDA = 2
SPARTON_ENOTSUP = 3
SPARTON_F32 = 0
SPARTON_BF16 = 1
SPARTON_MX_H = 0
SPARTON_MX_E = 1

# Every entry point include/sparton.h declares (checked by tests/test_abi.py).
EXPORTED = (
    "sparton_abi_version",
    "sparton_last_error",
    "sparton_device_sm_count",
    "sparton_fwd",
    "sparton_fwd_fp8",
    "sparton_fwd_multi",
    "sparton_fwd_multicast",
    "sparton_quantize_e4m3",
    "sparton_bwd_workspace_bytes",
    "sparton_bwd",
    "sparton_bwd_ex",
    "sparton_bwd_fp8",
    "sparton_mx_scales_bytes",
    "sparton_quantize_mx",
    "sparton_fwd_mx",
    "sparton_allreduce_peers",
    "sparton_allreduce_multimem",
)

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


class SpartonLibraryMissing(RuntimeError):
    """The native library has not been built (run __graft_entry__.build())."""


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _lib_path()
        if not path.exists():
            raise SpartonLibraryMissing(
                f"{path} not found: the sparton CUDA library is required (no CPU fallback); "
                "build it with `python -m paper_2603_25011_b200.build`")
        lib = ctypes.CDLL(str(path))
        c_i64, c_vp, c_int = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        lib.sparton_abi_version.restype = c_int
        lib.sparton_abi_version.argtypes = []
        lib.sparton_last_error.restype = ctypes.c_char_p
        lib.sparton_last_error.argtypes = []
        lib.sparton_device_sm_count.restype = c_int
        lib.sparton_device_sm_count.argtypes = []
        lib.sparton_fwd.restype = c_int
        lib.sparton_fwd.argtypes = [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                    c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_vp]
        lib.sparton_fwd_multi.restype = c_int
        lib.sparton_fwd_multi.argtypes = [c_vp, c_vp, c_vp, c_vp, c_int, ctypes.POINTER(c_vp),
                                          ctypes.POINTER(c_vp), c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_vp]
        lib.sparton_fwd_multicast.restype = c_int
        lib.sparton_fwd_multicast.argtypes = [c_vp] * 6 + [c_i64] * 5 + [c_int, c_vp]
        lib.sparton_fwd_fp8.restype = c_int
        lib.sparton_fwd_fp8.argtypes = [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                        c_i64, c_i64, c_i64, c_i64, c_i64, c_int, c_vp]
        lib.sparton_quantize_e4m3.restype = c_int
        lib.sparton_quantize_e4m3.argtypes = [c_vp, c_i64, c_vp, c_vp, c_vp]
        lib.sparton_bwd_workspace_bytes.restype = ctypes.c_size_t
        lib.sparton_bwd_workspace_bytes.argtypes = [c_i64, c_i64, c_i64, c_i64, c_int]
        lib.sparton_bwd.restype = c_int
        lib.sparton_bwd.argtypes = [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                    c_i64, c_i64, c_i64, c_i64, c_i64, c_i64,
                                    c_int, c_int, c_vp, ctypes.c_size_t, c_vp]
        lib.sparton_bwd_ex.restype = c_int
        lib.sparton_bwd_ex.argtypes = lib.sparton_bwd.argtypes + [c_vp]
        lib.sparton_mx_scales_bytes.restype = c_i64
        lib.sparton_mx_scales_bytes.argtypes = [c_i64, c_i64, c_i64, c_i64, c_int]
        lib.sparton_quantize_mx.restype = c_int
        lib.sparton_quantize_mx.argtypes = [c_vp, c_i64, c_i64, c_i64, c_i64, c_int, c_vp, c_vp, ctypes.c_size_t, c_vp]
        lib.sparton_fwd_mx.restype = c_int
        lib.sparton_fwd_mx.argtypes = [c_vp] * 8 + [c_i64] * 5 + [c_vp]
        lib.sparton_bwd_fp8.restype = c_int
        lib.sparton_bwd_fp8.argtypes = [c_vp] * 10 + [c_i64] * 6 + [c_int, c_int, c_vp, ctypes.c_size_t, c_vp, c_vp]
        lib.sparton_allreduce_peers.restype = c_int
        lib.sparton_allreduce_peers.argtypes = [ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_int, c_int, c_int,
                                                c_i64, c_vp]
        lib.sparton_allreduce_multimem.restype = c_int
        lib.sparton_allreduce_multimem.argtypes = [c_vp, c_vp, c_int, c_int, c_int, c_i64, c_vp]
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == SPARTON_OK:
        return
    msg = load().sparton_last_error().decode(errors="replace")
    if rc == SPARTON_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"sparton error {rc}: {msg}")
