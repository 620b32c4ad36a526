"""The (Y, I) all-gather fused into the forward epilogue (sharded.FusedVocabGather,
sparton_fwd_multi) — the pieces that run on the one available GPU.

* K1 with several destinations (strided column views of wider [B, V] buffers,
  ldY > V) writes identical results to each, exactly the single-destination
  result, and nothing outside its columns.
* Two ranks sharing cuda:0 over gloo with symmetric-memory [B, V] buffers:
  each rank's K1 stores its shard into BOTH ranks' buffers through the
  P2P-mapped pointers; the assembled (Y, I) equals the unsharded forward bit
  for bit, and the backward driven from the strided local columns matches.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _inputs(B, S, D, V, dev, seed=5):
    g = torch.Generator(device=dev).manual_seed(seed)
    H = torch.randn((B, S, D), generator=g, device=dev).to(torch.bfloat16)
    E = (torch.randn((V, D), generator=g, device=dev) * 0.05).to(torch.bfloat16)
    b = torch.randn(V, generator=g, device=dev) * 0.1
    m = (torch.rand((B, S), generator=g, device=dev) < 0.9).to(torch.uint8)
    dY = torch.randn((B, V), generator=g, device=dev)
    return H, E, b, m, dY


@pytest.mark.parametrize("dims", [(3, 300, 256, 1000), (2, 64, 128, 5000), (5, 17, 64, 300)])
def test_multi_destination_forward(cuda_device, dims):
    from paper_2603_25011_b200 import sparton_forward
    B, S, D, V = dims
    dev = cuda_device
    H, E, b, m, _ = _inputs(B, S, D, V, dev)
    Y0, I0 = sparton_forward(H, E, b, m)
    W, off = V + 37, 11
    bufs = [(torch.full((B, W), -7.0, device=dev), torch.full((B, W), -9, dtype=torch.int32, device=dev))
            for _ in range(3)]
    views = [(y[:, off:off + V], i[:, off:off + V]) for y, i in bufs]
    extra = tuple((y.data_ptr(), i.data_ptr()) for y, i in views[1:])
    sparton_forward(H, E, b, m, out=views[0], extra_out=extra)
    torch.cuda.synchronize()
    for (y, i), (yv, iv) in zip(bufs, views):
        assert torch.equal(yv, Y0) and torch.equal(iv, I0)
        assert bool((y[:, :off] == -7).all()) and bool((y[:, off + V:] == -7).all())
        assert bool((i[:, :off] == -9).all()) and bool((i[:, off + V:] == -9).all())


@pytest.mark.parametrize("dims", [(3, 300, 256, 1000), (5, 17, 64, 300)])
def test_multicast_store_path_addressing(cuda_device, dims):
    """The NVLS store path (sparton_fwd_multicast: multimem.st.relaxed.sys,
    i.e. STG.E.STRONG.SYS to the given address) aimed at an ordinary device
    buffer: the switch replication needs >= 2 GPUs, but the epilogue's
    addressing (strided column view, row stride ldY) is checked here — the
    buffer receives exactly the plain forward's results and nothing outside
    its columns; the `out` buffer itself is left untouched."""
    from paper_2603_25011_b200 import sparton_forward
    B, S, D, V = dims
    dev = cuda_device
    H, E, b, m, _ = _inputs(B, S, D, V, dev)
    Y0, I0 = sparton_forward(H, E, b, m)
    W, off = V + 29, 13
    y, i = torch.full((B, W), -7.0, device=dev), torch.full((B, W), -9, dtype=torch.int32, device=dev)
    oy, oi = torch.full((B, W), -5.0, device=dev), torch.full((B, W), -3, dtype=torch.int32, device=dev)
    sparton_forward(H, E, b, m, out=(oy[:, off:off + V], oi[:, off:off + V]),
                    multicast_out=(y[:, off:].data_ptr(), i[:, off:].data_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(y[:, off:off + V], Y0) and torch.equal(i[:, off:off + V], I0)
    assert bool((y[:, :off] == -7).all()) and bool((y[:, off + V:] == -7).all())
    assert bool((i[:, :off] == -9).all()) and bool((i[:, off + V:] == -9).all())
    assert bool((oy == -5).all()) and bool((oi == -3).all())


def test_multi_destination_rejects_more_than_eight(cuda_device):
    from paper_2603_25011_b200 import sparton_forward
    H, E, b, m, _ = _inputs(2, 8, 16, 10, cuda_device)
    Y = torch.empty((2, 10), device=cuda_device)
    I = torch.empty((2, 10), dtype=torch.int32, device=cuda_device)
    with pytest.raises(ValueError):
        sparton_forward(H, E, b, m, out=(Y, I), extra_out=((Y.data_ptr(), I.data_ptr()),) * 8)


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, qs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_25011_b200.sharded import FusedVocabGather, local_backward, shard_range
        B, S, D, V = dims
        H, E, b, m, dY = _inputs(B, S, D, V, dev)
        v0, v1, _ = shard_range(V, world, rank)
        # Each rank's [B, V] buffers, mapped into the other rank by CUDA IPC
        # (torch.multiprocessing shares CUDA tensors through the queue).
        Yb = torch.full((B, V), float("nan"), device=dev)
        Ib = torch.full((B, V), -5, dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        qs[1 - rank].put((Yb, Ib))
        Yp, Ip = qs[rank].get(timeout=120)

        def barrier(_channel):
            torch.cuda.synchronize()
            dist.barrier()

        fg = FusedVocabGather(Yb, Ib, [(Yp.data_ptr(), Ip.data_ptr())], barrier, keepalive=(Yp, Ip))
        for _ in range(2):                       # reuse of the buffers across steps
            Y, I = fg.forward(H, E[v0:v1], b[v0:v1], m, v0)
        dH, dE, db = local_backward(H, E[v0:v1], Y[:, v0:v1], I[:, v0:v1], dY[:, v0:v1], group=None)
        torch.cuda.synchronize()
        q.put((rank, (Y.cpu().numpy(), I.cpu().numpy(), dH.cpu().numpy(), dE.cpu().numpy(),
                      db.cpu().numpy(), v0, v1)))
        dist.barrier()                           # the peer keeps using our buffers until here
    finally:
        dist.destroy_process_group()


def test_fused_gather_two_ranks_one_gpu(cuda_device):
    """Two processes on cuda:0; each K1 writes its shard into both ranks'
    buffers (the peer's through an IPC mapping, i.e. a P2P store from the
    kernel), exactly the production FusedVocabGather code path."""
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    dims = (3, 200, 128, 3001)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    qs = [ctx.Queue(), ctx.Queue()]
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, qs, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    B, S, D, V = dims
    H, E, b, m, dY = _inputs(B, S, D, V, cuda_device)
    Y, I = sparton_forward(H, E, b, m)
    dH, dE, db = sparton_backward(H, E, Y, I, dY)
    for rank, (Yr, Ir, dHr, dEr, dbr, v0, v1) in res:
        assert np.array_equal(Yr, Y.cpu().numpy()) and np.array_equal(Ir, I.cpu().numpy())
        assert np.array_equal(dEr, dE[v0:v1].cpu().numpy()) and np.array_equal(dbr, db[v0:v1].cpu().numpy())
        assert np.allclose(dHr, dH.cpu().numpy(), rtol=1e-5, atol=1e-6)   # all-reduced partial dH
