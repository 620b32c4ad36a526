"""The sharded head's dH reduction over peer memory (``sparton_allreduce_peers``,
``sharded.PeerDHReduce``) on one GPU.

* The kernel with three "ranks" whose buffers are ordinary allocations on
  cuda:0: calling it for every rank leaves every output buffer equal, bit for
  bit, to the rank-ordered fp32 sum ((p0 + p1) + p2) — or its bf16 rounding —
  for slices that do not divide evenly and ranks with empty slices.
* Two processes on cuda:0 whose partial/output buffers are mapped into each
  other by CUDA IPC (the same P2P loads and stores as over NVLink): the
  vocab-sharded backward with ``local_backward(..., dh_reduce=...)`` gives
  both ranks the same dH bit for bit, within fp32 reassociation (bf16:
  rounding) of the unsharded backward, and dE/db shards equal to it.
The NVLS variant (``sparton_allreduce_multimem``) issues multimem.ld_reduce,
which needs a multicast object of >= 2 GPUs (it faults on a unicast address),
so only its argument checks run here (tests/test_abi.py).
"""

from __future__ import annotations

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _allreduce(parts, outs, rank, dtype):
    from paper_2603_25011_b200 import _lib
    lib = _lib.load()
    P = len(parts)
    pa = (ctypes.c_void_p * P)(*[t.data_ptr() for t in parts])
    oa = (ctypes.c_void_p * P)(*[t.data_ptr() for t in outs])
    od = _lib.SPARTON_BF16 if dtype == torch.bfloat16 else _lib.SPARTON_F32
    rc = lib.sparton_allreduce_peers(pa, oa, P, rank, od, parts[0].numel(),
                                     torch.cuda.current_stream().cuda_stream)
    _lib.check(rc)


@pytest.mark.parametrize("n", [4 * 1001, 4, 4 * 3, 512 * 512 * 768])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_allreduce_peers_rank_ordered_sum(cuda_device, n, dtype):
    g = torch.Generator(device=cuda_device).manual_seed(n)
    parts = [torch.randn(n, generator=g, device=cuda_device) for _ in range(3)]
    outs = [torch.full((n,), 7.0, device=cuda_device).to(dtype) for _ in range(3)]
    for r in range(3):
        _allreduce(parts, outs, r, dtype)
    want = ((parts[0] + parts[1]) + parts[2]).to(dtype)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, want)


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(B, S, D, V, dev):
    g = torch.Generator(device=dev).manual_seed(5)
    H = torch.randn((B, S, D), generator=g, device=dev).to(torch.bfloat16)
    E = (torch.randn((V, D), generator=g, device=dev) * 0.05).to(torch.bfloat16)
    b = torch.randn(V, generator=g, device=dev) * 0.1
    m = (torch.rand((B, S), generator=g, device=dev) < 0.9).to(torch.uint8)
    dY = torch.randn((B, V), generator=g, device=dev)
    return H, E, b, m, dY


def _worker(rank, world, port, dims, dtype, qs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_25011_b200 import sparton_forward
        from paper_2603_25011_b200.sharded import PeerDHReduce, local_backward, shard_range
        B, S, D, V = dims
        H, E, b, m, dY = _inputs(B, S, D, V, dev)
        v0, v1, _ = shard_range(V, world, rank)
        Y, I = sparton_forward(H, E, b, m)
        part = torch.full((B, S, D), float("nan"), device=dev)
        out = torch.full((B, S, D), float("nan"), device=dev).to(dtype)
        torch.cuda.synchronize()
        qs[1 - rank].put((part, out))              # CUDA IPC: the peer maps our buffers
        pp, po = qs[rank].get(timeout=120)
        parts = [part.data_ptr(), pp.data_ptr()] if rank == 0 else [pp.data_ptr(), part.data_ptr()]
        outs = [out.data_ptr(), po.data_ptr()] if rank == 0 else [po.data_ptr(), out.data_ptr()]

        def barrier(_channel):
            torch.cuda.synchronize()
            dist.barrier()

        red = PeerDHReduce(part, out, parts, outs, rank, barrier, keepalive=(pp, po))
        res = None
        for _ in range(2):                         # buffer reuse across steps
            dH, dE, db = local_backward(H, E[v0:v1], Y[:, v0:v1], I[:, v0:v1], dY[:, v0:v1],
                                        grad_dtype=dtype, dh_reduce=red)
            torch.cuda.synchronize()
            res = (dH.float().cpu().numpy(), dE.float().cpu().numpy(), db.cpu().numpy(), v0, v1)
        q.put((rank, res))
        dist.barrier()                             # the peer reads our buffers until here
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_peer_dh_reduce_two_ranks_one_gpu(cuda_device, dtype):
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    dims = (3, 200, 128, 3001)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    qs = [ctx.Queue(), ctx.Queue()]
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, dtype, qs, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    B, S, D, V = dims
    H, E, b, m, dY = _inputs(B, S, D, V, cuda_device)
    Y, I = sparton_forward(H, E, b, m)
    dH, dE, db = sparton_backward(H, E, Y, I, dY, grad_dtype=dtype)
    dH, dE, db = dH.float().cpu().numpy(), dE.float().cpu().numpy(), db.cpu().numpy()
    (_, (dH0, _, _, _, _)), (_, (dH1, _, _, _, _)) = res
    assert np.array_equal(dH0, dH1)                                 # one reduction, identical on both ranks
    rtol, atol = (1e-5, 1e-6) if dtype == torch.float32 else (1e-2, 1e-3)
    for rank, (dHr, dEr, dbr, v0, v1) in res:
        assert np.allclose(dHr, dH, rtol=rtol, atol=atol)
        assert np.array_equal(dEr, dE[v0:v1]) and np.array_equal(dbr, db[v0:v1])
