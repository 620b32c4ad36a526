"""CPU, world_size 2 over gloo: the vocab-sharded head's assembly logic.

Each rank owns a vocab shard [p*Vp, min((p+1)*Vp, V)); the local compute is
injected (here the CPU oracle, as the checker stand-in for the sm_100a kernel)
so the all-gather assembly of (Y, I) and the all-reduce of the partial dH are
exercised exactly as on GPUs.  Sharded results must equal the unsharded ones:
(Y, I) bit-exactly (same per-column arithmetic), dH within fp32 reassociation.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sparton_oracle as orc


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_25011_b200.sharded import forward_sharded, local_backward, shard_range
        B, S, D, V = dims
        H, E, b, m = orc.seeded_inputs(B, S, D, V, 11, mask_keep=0.8)
        dY = orc.seeded_uniform((B, V), 12)
        v0, v1, Vp = shard_range(V, world, rank)

        def local_fn(Ht, Es, bs, mt):
            Y, I = orc.forward(Ht.numpy(), Es.numpy(), bs.numpy(), mt.numpy(), deterministic=True)
            return torch.from_numpy(Y), torch.from_numpy(I)

        def local_bwd(Ht, Es, Yp, Ip, dYp, include_bias_grad=True, grad_dtype=None):
            dH, dE, db = orc.backward(Ht.numpy(), Es.numpy(), None, Yp.numpy(), Ip.numpy(), dYp.numpy())
            return torch.from_numpy(dH), torch.from_numpy(dE), torch.from_numpy(db)

        Ht = torch.from_numpy(H)
        Es = torch.from_numpy(E[v0:v1])
        Y, I = forward_sharded(Ht, Es, torch.from_numpy(b[v0:v1]), torch.from_numpy(m), V, local_fn=local_fn)
        Yp, Ip = Y[:, v0:v1].contiguous(), I[:, v0:v1].contiguous()
        dH, dE, db = local_backward(Ht, Es, Yp, Ip, torch.from_numpy(dY[:, v0:v1].copy()), local_bwd=local_bwd)
        q.put((rank, Y.numpy(), I.numpy(), dH.numpy(), dE.numpy(), db.numpy(), v0, v1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims", [(3, 7, 8, 23), (2, 16, 16, 64), (4, 5, 4, 3)])
def test_vocab_sharded_matches_unsharded(dims):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    B, S, D, V = dims
    H, E, b, m = orc.seeded_inputs(B, S, D, V, 11, mask_keep=0.8)
    dY = orc.seeded_uniform((B, V), 12)
    Yr, Ir = orc.forward(H, E, b, m, deterministic=True)
    dHr, dEr, dbr = orc.backward(H, E, b, Yr, Ir, dY)
    for rank, Y, I, dH, dE, db, v0, v1 in res:
        assert Y.tobytes() == Yr.tobytes() and np.array_equal(I, Ir)
        assert np.allclose(dH, dHr, rtol=1e-5, atol=1e-6)
        assert dE.tobytes() == dEr[v0:v1].tobytes() and db.tobytes() == dbr[v0:v1].tobytes()


def test_fused_gather_multicast_selection():
    """FusedVocabGather.pick_multicast: NVLS only when both symmetric buffers
    have a multicast mapping (auto), required on request, never when off."""
    from types import SimpleNamespace as NS
    from paper_2603_25011_b200.sharded import FusedVocabGather as F
    with_mc = (NS(multicast_ptr=0x1000), NS(multicast_ptr=0x2000))
    without = (NS(multicast_ptr=0), NS(multicast_ptr=0x2000))
    assert F.pick_multicast(*with_mc, None) == (0x1000, 0x2000)
    assert F.pick_multicast(*with_mc, True) == (0x1000, 0x2000)
    assert F.pick_multicast(*with_mc, False) is None
    assert F.pick_multicast(*without, None) is None
    assert F.pick_multicast(NS(), NS(), None) is None
    with pytest.raises(RuntimeError):
        F.pick_multicast(*without, True)


def _reduce_worker(rank, world, port, shape, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_25011_b200.sharded import reduce_dh
        g = torch.Generator().manual_seed(100 + rank)
        part = torch.randn(shape, generator=g)
        ref = part.clone()
        dist.all_reduce(ref)
        out = {}
        for dt in (torch.bfloat16, torch.float32):
            r = reduce_dh(part.clone(), dt)
            out[str(dt)] = (r.dtype == dt, tuple(r.shape) == shape, torch.equal(r, ref.to(dt)))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape", [(2, 6, 8), (3, 5, 7)])   # divisible by the world size / not (all-reduce fallback)
def test_reduce_dh_matches_fp32_allreduce_then_cast(shape):
    """sharded.reduce_dh: the bf16 result of the fp32 reduce-scatter + bf16
    all-gather equals an fp32 all-reduce followed by the cast (two ranks:
    the fp32 sums are order-independent), for both the flat path and the
    all-reduce fallback; fp32 stays an fp32 all-reduce."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_reduce_worker, args=(r, world, port, shape, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out in res:
        for dt, checks in out.items():
            assert all(checks), (rank, dt, checks)
