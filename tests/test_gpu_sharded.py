"""GPU: the vocab-sharded head end to end with real kernels, world_size 2.

Only one GPU is available, so both ranks share cuda:0 and talk over gloo (NCCL
refuses two ranks on one device); the kernels, the shard arithmetic, the
(Y, I) all-gather assembly and the dH all-reduce are the production code.
Sharded (Y, I) must equal the single-GPU result bit-exactly (same per-column
arithmetic); dE/db shards bit-exactly; dH within fp32 reassociation."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


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


def _worker(rank, world, port, dims, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_25011_b200.sharded import ShardedSpartonHeadFn, shard_range
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        B, S, D, V = dims
        H, E, b, m, dY = _inputs(B, S, D, V, dev)
        v0, v1, _ = shard_range(V, world, rank)
        Hq = H.clone().requires_grad_(True)
        Es = E[v0:v1].clone().requires_grad_(True)
        bs = b[v0:v1].clone().requires_grad_(True)
        Y = ShardedSpartonHeadFn.apply(Hq, Es, bs, m, V)
        Y.backward(dY)
        torch.cuda.synchronize()
        q.put((rank, Y.detach().cpu().numpy(), Hq.grad.float().cpu().numpy(), Es.grad.float().cpu().numpy(),
               bs.grad.cpu().numpy(), v0, v1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims", [(4, 96, 128, 1001), (2, 300, 768, 2049)])
def test_sharded_matches_single(cuda_device, dims):
    from paper_2603_25011_b200 import sparton_head
    B, S, D, V = dims
    H, E, b, m, dY = _inputs(B, S, D, V, cuda_device)
    Hq = H.clone().requires_grad_(True)
    Eq = E.clone().requires_grad_(True)
    bq = b.clone().requires_grad_(True)
    Y = sparton_head(Hq, Eq, bq, m)
    Y.backward(dY)
    ref = (Y.detach().cpu().numpy(), Hq.grad.float().cpu().numpy(), Eq.grad.float().cpu().numpy(),
           bq.grad.cpu().numpy())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, Ys, dH, dE, db, v0, v1 in res:
        assert Ys.tobytes() == ref[0].tobytes()
        assert dE.tobytes() == ref[2][v0:v1].tobytes()
        assert db.tobytes() == ref[3][v0:v1].tobytes()
        # dH: fp32 partial sums reduced across ranks, then rounded to bf16
        assert np.allclose(dH, ref[1], rtol=1e-2, atol=1e-2)


def _fullsize_worker(rank, world, port, dims, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_25011_b200 import sparton_head
        from paper_2603_25011_b200.sharded import ShardedSpartonHeadFn, shard_range
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        B, S, D, V = dims
        H, E, b, m, dY = _inputs(B, S, D, V, dev)
        v0, v1, _ = shard_range(V, world, rank)
        Hq = H.clone().requires_grad_(True)
        Es = E[v0:v1].clone().requires_grad_(True)
        bs = b[v0:v1].clone().requires_grad_(True)
        Y = ShardedSpartonHeadFn.apply(Hq, Es, bs, m, V)
        Y.backward(dY)
        # the unsharded head on the same GPU, compared here (no 0.5 GB arrays through the queue)
        Hr = H.clone().requires_grad_(True)
        Er = E.clone().requires_grad_(True)
        br = b.clone().requires_grad_(True)
        Yr = sparton_head(Hr, Er, br, m)
        Yr.backward(dY)
        torch.cuda.synchronize()
        dh_err = float((Hq.grad.float() - Hr.grad.float()).abs().max())
        dh_tol = float(1e-2 * Hr.grad.float().abs().max() + 1e-3)
        q.put((rank, bool(torch.equal(Y.detach(), Yr.detach())), bool(torch.equal(Es.grad, Er.grad[v0:v1])),
               bool(torch.equal(bs.grad, br.grad[v0:v1])), dh_err, dh_tol))
    finally:
        dist.destroy_process_group()


def test_sharded_matches_single_at_cfg3(cuda_device):
    """The sharded autograd head at cfg3's full size (B=S=512, D=768,
    V=250002; two ranks): Y equal bit for bit to the single-GPU head, dE/db
    shards equal bit for bit, dH (bf16, summed across ranks) within bf16
    rounding of the single-GPU dH."""
    dims = (512, 512, 768, 250002)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_fullsize_worker, args=(r, 2, port, dims, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    for rank, y_eq, de_eq, db_eq, dh_err, dh_tol in res:
        assert y_eq and de_eq and db_eq, (rank, y_eq, de_eq, db_eq)
        assert dh_err <= dh_tol, (rank, dh_err, dh_tol)
