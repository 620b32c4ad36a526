"""The C-ABI library loads and exports exactly what include/sparton.h declares.

CPU-only: no kernel is launched.  Argument validation happens before any CUDA
call, so EINVAL paths are exercised here too.
"""

from __future__ import annotations

import ctypes
import re

import pytest

from conftest import REPO


def _declared():
    hdr = (REPO / "include" / "sparton.h").read_text()
    return sorted(set(re.findall(r"SPARTON_API\s+[\w\s\*]+?\b(sparton_\w+)\s*\(", hdr)))


def test_header_declares_entry_points():
    names = _declared()
    assert names == sorted(["sparton_abi_version", "sparton_last_error", "sparton_device_sm_count",
                            "sparton_fwd", "sparton_fwd_fp8", "sparton_fwd_multi", "sparton_fwd_multicast",
                            "sparton_quantize_e4m3",
                            "sparton_bwd_workspace_bytes", "sparton_bwd", "sparton_bwd_ex",
                            "sparton_bwd_fp8", "sparton_mx_scales_bytes", "sparton_quantize_mx",
                            "sparton_fwd_mx", "sparton_allreduce_peers", "sparton_allreduce_multimem"])


def test_library_exports_every_declared_symbol():
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTED) == set(_declared())
    assert lib.sparton_abi_version() == 100


def test_workspace_formula():
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    up = lambda x: (x + 255) // 256 * 256
    win = 8192                                   # route window (vocab rows)
    B, S, D, V = 512, 512, 768, 250002
    nwin = -(-V // win)
    base = up(B * V * 8) + up(B * nwin * (S + 1) * 4) + up(V * 4)
    gi = up(B * (V + V % 2) * 8)                 # (s, g) records of the staged dE (S <= 832)
    # fp32 gradients carry dH partial sums in the output; bf16 needs an fp32 dH
    # carry because dH runs in vocab-chunk passes (cfg3: 384 MB of E).  The
    # staged dE keeps its sums in registers over the whole batch: no dE carry.
    st = 256                                     # active-pair count (sparse regime)
    assert lib.sparton_bwd_workspace_bytes(B, S, D, V, _lib.SPARTON_F32) == base + gi + st
    assert lib.sparton_bwd_workspace_bytes(B, S, D, V, _lib.SPARTON_BF16) == base + up(B * S * D * 4) + gi + st
    # S beyond the staged dE's smem limit: gathered dE in batch-chunk passes with an fp32 carry
    S2 = 1024
    base2 = up(B * V * 8) + up(B * nwin * (S2 + 1) * 4) + up(V * 4)
    assert lib.sparton_bwd_workspace_bytes(B, S2, D, V, _lib.SPARTON_BF16) == base2 + up(V * D * 4) + up(B * S2 * D * 4) + st
    # a tiny problem is one window and one pass of each kind: no carry buffers
    assert lib.sparton_bwd_workspace_bytes(2, 3, 8, 5, _lib.SPARTON_BF16) == (
        up(2 * 5 * 8) + up(2 * 1 * 4 * 4) + up(5 * 4) + up(2 * 6 * 8) + st)
    assert lib.sparton_bwd_workspace_bytes(0, S, D, V, 0) == 0


@pytest.mark.parametrize("dims", [(0, 3, 8, 5), (2, 3, 4, 5), (2, -1, 8, 5)])
def test_fwd_rejects_bad_dims_before_any_cuda_call(dims):
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    B, S, D, V = dims
    dummy = ctypes.c_void_p(16)
    rc = lib.sparton_fwd(dummy, dummy, dummy, dummy, dummy, dummy, B, S, D, V, V, 0, None)
    assert rc == _lib.SPARTON_EINVAL
    assert lib.sparton_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_fwd_rejects_null_and_misaligned():
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    a = ctypes.c_void_p(256)
    assert lib.sparton_fwd(None, a, a, a, a, a, 2, 3, 8, 5, 5, 0, None) == _lib.SPARTON_EINVAL
    odd = ctypes.c_void_p(258)
    assert lib.sparton_fwd(odd, a, a, a, a, a, 2, 3, 8, 5, 5, 0, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_fwd(a, a, a, a, a, a, 2, 3, 8, 5, 4, 0, None) == _lib.SPARTON_EINVAL  # ldY < V
    assert lib.sparton_fwd(a, a, a, a, a, a, 2, 3, 8, 5, 5, 3, None) == _lib.SPARTON_EINVAL  # cta_group


def test_fwd_multicast_rejects_bad_arguments_before_any_cuda_call():
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    a = ctypes.c_void_p(256)
    assert lib.sparton_fwd_multicast(a, a, a, a, None, a, 2, 3, 8, 5, 5, 0, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_fwd_multicast(a, a, a, a, a, a, 2, 3, 8, 5, 4, 0, None) == _lib.SPARTON_EINVAL  # ldY < V


def test_bwd_rejects_small_workspace():
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    a = ctypes.c_void_p(256)
    rc = lib.sparton_bwd(a, a, a, a, a, a, a, a, 2, 3, 8, 5, 5, 5, 1, 0, a, 16, None)
    assert rc == _lib.SPARTON_EINVAL
    assert b"workspace" in lib.sparton_last_error()
    rc = lib.sparton_bwd(a, a, a, a, a, a, a, a, 2, 3, 8, 5, 5, 5, 1, 7, a, 1 << 20, None)
    assert rc == _lib.SPARTON_EINVAL


def test_sm_count_query_is_safe_without_gpu():
    from paper_2603_25011_b200 import _lib
    import torch
    n = _lib.load().sparton_device_sm_count()
    if not torch.cuda.is_available():
        assert n == 0
    else:
        assert n > 0


def test_fp8_entry_points_reject_bad_arguments_before_any_cuda_call():
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    d = ctypes.c_void_p(16)
    # D = 8 is not a multiple of 16 (e4m3 TMA stride rule)
    assert lib.sparton_fwd_fp8(d, d, d, d, d, d, d, d, 2, 3, 8, 5, 5, 0, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_fwd_fp8(d, d, None, d, d, d, d, d, 2, 3, 16, 5, 5, 0, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_quantize_e4m3(d, 15, d, d, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_quantize_e4m3(d, 0, d, d, None) == _lib.SPARTON_EINVAL


def test_mx_entry_points_reject_bad_arguments_before_any_cuda_call():
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    d = ctypes.c_void_p(16)
    # scale bytes: E (V, D) = ceil(V/128) * ceil(D/128) chunks of 512 B; H per (batch row, 240-position chunk)
    assert lib.sparton_mx_scales_bytes(1, 1, 768, 250002, _lib.SPARTON_MX_E) == 1954 * 6 * 512
    assert lib.sparton_mx_scales_bytes(512, 512, 768, 1, _lib.SPARTON_MX_H) == 512 * 3 * 6 * 1024
    assert lib.sparton_mx_scales_bytes(8, 32, 64, 1, _lib.SPARTON_MX_H) == 2 * 1 * 1 * 1024   # 7 rows per chunk
    assert lib.sparton_mx_scales_bytes(8, 32, 64, 1, 7) == 0
    assert lib.sparton_quantize_mx(d, 2, 3, 8, 5, _lib.SPARTON_MX_H, d, d, 1 << 20, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_quantize_mx(d, 2, 3, 16, 5, 9, d, d, 1 << 20, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_quantize_mx(d, 2, 3, 16, 5, _lib.SPARTON_MX_E, d, d, 1, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_fwd_mx(d, d, d, d, d, d, d, d, 2, 3, 8, 5, 5, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_fwd_mx(d, None, d, d, d, d, d, d, 2, 3, 16, 5, 5, None) == _lib.SPARTON_EINVAL


def test_experiment_switches_need_the_dev_gate(monkeypatch):
    """The shipped library reads SPARTON_* switches only under SPARTON_DEV=1:
    SPARTON_DE_STAGED=0 (gathered dE, which needs an fp32 dE carry in the
    workspace) changes the workspace layout only inside the gate."""
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    B, S, D, V = 512, 512, 768, 250002
    default = lib.sparton_bwd_workspace_bytes(B, S, D, V, _lib.SPARTON_BF16)
    monkeypatch.delenv("SPARTON_DEV", raising=False)
    monkeypatch.setenv("SPARTON_DE_STAGED", "0")
    monkeypatch.setenv("SPARTON_DH_CHUNK_MB", "400")
    assert lib.sparton_bwd_workspace_bytes(B, S, D, V, _lib.SPARTON_BF16) == default
    monkeypatch.setenv("SPARTON_DEV", "1")
    assert lib.sparton_bwd_workspace_bytes(B, S, D, V, _lib.SPARTON_BF16) != default


def test_staged_de_sequence_limit():
    """The staged dE (S <= 832: two smem stages of an S-row H tile) carries no
    dE workspace; S = 833 switches to the gathered dE (fp32 dE carry when bf16
    gradients need more than one batch-chunk pass)."""
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    up = lambda x: (x + 255) // 256 * 256
    B, D, V = 512, 768, 250002
    nwin = -(-V // 8192)
    for S, staged in ((832, True), (833, False)):
        base = up(B * V * 8) + up(B * nwin * (S + 1) * 4) + up(V * 4)
        extra = up(B * (V + V % 2) * 8) if staged else up(V * D * 4)
        assert lib.sparton_bwd_workspace_bytes(B, S, D, V, _lib.SPARTON_F32) == base + (
            extra if staged else 0) + 256, S


def test_allreduce_entry_points_reject_bad_arguments_before_any_cuda_call():
    """sparton_allreduce_peers / _multimem validate ranks, dtype, n and
    pointers on the host (EINVAL) before touching the device."""
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    d = 0x1000
    arr = (ctypes.c_void_p * 2)(d, d)
    F32, BF16 = _lib.SPARTON_F32, _lib.SPARTON_BF16
    assert lib.sparton_allreduce_peers(arr, arr, 0, 0, F32, 8, None) == _lib.SPARTON_EINVAL      # nranks
    assert lib.sparton_allreduce_peers(arr, arr, 9, 0, F32, 8, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_allreduce_peers(arr, arr, 2, 2, F32, 8, None) == _lib.SPARTON_EINVAL      # rank
    assert lib.sparton_allreduce_peers(arr, arr, 2, 0, 7, 8, None) == _lib.SPARTON_EINVAL        # dtype
    assert lib.sparton_allreduce_peers(arr, arr, 2, 0, F32, 6, None) == _lib.SPARTON_EINVAL      # n % 4
    assert lib.sparton_allreduce_peers(None, arr, 2, 0, F32, 8, None) == _lib.SPARTON_EINVAL
    odd = (ctypes.c_void_p * 2)(d, d + 4)
    assert lib.sparton_allreduce_peers(odd, arr, 2, 0, F32, 8, None) == _lib.SPARTON_EINVAL      # alignment
    assert lib.sparton_allreduce_peers(arr, odd, 2, 0, BF16, 8, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_allreduce_multimem(d, d, 2, 0, F32, 6, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_allreduce_multimem(None, d, 2, 0, F32, 8, None) == _lib.SPARTON_EINVAL
    assert lib.sparton_allreduce_multimem(d, d + 8, 2, 0, F32, 8, None) == _lib.SPARTON_EINVAL
    assert "aligned" in lib.sparton_last_error().decode()
