"""Vocab-sharded (column-parallel) Sparton head over torch.distributed / NCCL.

Each output column v depends only on E[v] and b[v], so rank p
owns vocab rows [p·Vp, min((p+1)·Vp, V)) with Vp = ⌈V/P⌉ and runs the fused
forward on its shard with no communication; the B×V output is assembled by
one all-gather of the (Y, I) shards.  The backward is local for dE/db; dH is a
sum over every rank's vocab shard, so the per-rank partial dH (fp32) is
all-reduced.  H, mask and dY are replicated (dY columns are sliced in place).

The local compute is injectable (``local_fn`` / ``local_bwd``) so the sharding
and assembly logic is tested on CPU with the gloo backend; on GPU it is the
sm_100a kernels.
"""

from __future__ import annotations

import ctypes
from typing import Callable

import torch
import torch.distributed as dist

from . import _lib
from .head import _stream_ptr, sparton_backward, sparton_forward


def shard_range(V: int, world: int, rank: int) -> tuple[int, int, int]:
    """(v0, v1, Vp): this rank's vocab rows [v0, v1) and the padded shard width."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    Vp = (V + world - 1) // world
    v0 = min(V, rank * Vp)
    v1 = min(V, (rank + 1) * Vp)
    return v0, v1, Vp


def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def local_forward(H, E_shard, bias_shard, mask, out=None):
    """K1 on this rank's vocab shard."""
    return sparton_forward(H, E_shard, bias_shard, mask, out=out)


def gather_vocab(Y_p: torch.Tensor, I_p: torch.Tensor, V: int, Vp: int, group=None):
    """All-gather the per-rank (Y, I) column shards into full [B, V] tensors.

    Shards are padded to Vp columns (NCCL needs equal counts); the padding sits
    only at the tail of the last shard(s), so concatenating shards in rank
    order and cutting at V is exact."""
    world, _ = _world(group)
    B, n = Y_p.shape
    if world == 1:
        return Y_p, I_p
    Yb = torch.zeros((B, Vp), dtype=Y_p.dtype, device=Y_p.device)
    Ib = torch.zeros((B, Vp), dtype=I_p.dtype, device=I_p.device)
    Yb[:, :n] = Y_p
    Ib[:, :n] = I_p
    if _flat_collectives(group, Y_p):
        # One [P, B, Vp] buffer per output, then one permute copy to [B, V].
        ys = torch.empty((world * B, Vp), dtype=Y_p.dtype, device=Y_p.device)
        is_ = torch.empty((world * B, Vp), dtype=I_p.dtype, device=I_p.device)
        dist.all_gather_into_tensor(ys, Yb, group=group)
        dist.all_gather_into_tensor(is_, Ib, group=group)
        Y = ys.view(world, B, Vp).permute(1, 0, 2).reshape(B, world * Vp)[:, :V].contiguous()
        I = is_.view(world, B, Vp).permute(1, 0, 2).reshape(B, world * Vp)[:, :V].contiguous()
        return Y, I
    ys = [torch.empty_like(Yb) for _ in range(world)]
    is_ = [torch.empty_like(Ib) for _ in range(world)]
    dist.all_gather(ys, Yb, group=group)
    dist.all_gather(is_, Ib, group=group)
    Y = torch.cat(ys, dim=1)[:, :V].contiguous()
    I = torch.cat(is_, dim=1)[:, :V].contiguous()
    return Y, I


def _flat_collectives(group, t: torch.Tensor) -> bool:
    """NCCL (or any backend on CPU tensors) takes the flat tensor collectives
    (all_gather_into_tensor / reduce_scatter_tensor); gloo with CUDA tensors
    (the one-GPU multi-rank tests) keeps the list / all-reduce forms."""
    return not t.is_cuda or dist.get_backend(group) == "nccl"


def reduce_dh(dH: torch.Tensor, grad_dtype: torch.dtype, group=None) -> torch.Tensor:
    """Sum the per-rank partial dH (fp32) over the group and return it in
    ``grad_dtype``.  For a narrower ``grad_dtype`` the sum is a reduce-scatter
    in fp32 (the reference's accumulation precision), the cast of each rank's
    reduced rows, and an all-gather of the cast rows: the same values as an
    fp32 all-reduce followed by the cast, with 2/3 of its bytes on the wire
    for bf16 (fp32 reduce-scatter + bf16 all-gather vs two fp32 phases)."""
    world, _ = _world(group)
    if world == 1:
        return dH if grad_dtype == torch.float32 else dH.to(grad_dtype)
    n = dH.numel()
    if grad_dtype != torch.float32 and n % world == 0 and _flat_collectives(group, dH):
        flat = dH.reshape(-1)
        part = torch.empty(n // world, dtype=torch.float32, device=dH.device)
        dist.reduce_scatter_tensor(part, flat, op=dist.ReduceOp.SUM, group=group)
        out = torch.empty(n, dtype=grad_dtype, device=dH.device)
        dist.all_gather_into_tensor(out, part.to(grad_dtype), group=group)
        return out.view(dH.shape)
    dist.all_reduce(dH, op=dist.ReduceOp.SUM, group=group)
    return dH if grad_dtype == torch.float32 else dH.to(grad_dtype)


class FusedVocabGather:
    """The (Y, I) all-gather fused into K1's epilogue.

    Every rank holds a [B, V] (Y, I) pair that all other ranks can address:
    rank p's forward stores each result of its shard into EVERY rank's copy at
    columns [v0_p, v1_p) through the peers' mapped pointers
    (``sparton_fwd_multi``, up to 8 ranks) — no NCCL all-gather, no padded
    [P, B, Vp] staging and no permute copy, and the NVLink transfer overlaps
    the MMAs unit by unit.  A barrier before the launch (peers are done reading
    the previous contents) and after it (every shard has landed) orders the
    exchange.  The returned tensors are the local buffers, valid until the
    next ``forward``.

    ``FusedVocabGather.symmetric(B, V, device, group)`` is the production
    constructor: torch symmetric memory (P2P-mapped across the NVLink domain)
    and its device-side barrier on the current stream.  The plain constructor
    takes already-mapped peer buffers and a barrier callable (the one-GPU test
    maps the peers' buffers with CUDA IPC)."""

    def __init__(self, Y: torch.Tensor, I: torch.Tensor, peers, barrier: Callable[[int], None],
                 keepalive=(), multicast: tuple[int, int] | None = None):
        if Y.shape != I.shape or Y.dtype != torch.float32 or I.dtype != torch.int32:
            raise ValueError("Y must be float32 and I int32 of the same [B, V] shape")
        if len(peers) > 7 and multicast is None:
            raise ValueError("the fused gather addresses at most 8 ranks (sparton_fwd_multi)")
        self.Y, self.I = Y, I
        self.B, self.V = Y.shape
        self.peers = [(int(y), int(i)) for y, i in peers]
        self.multicast = None if multicast is None else (int(multicast[0]), int(multicast[1]))
        self.barrier = barrier
        self._keepalive = keepalive

    @staticmethod
    def pick_multicast(hY, hI, multicast: bool | None):
        """The (Y, I) multicast base addresses to store through, or None for
        P2P stores.  ``multicast`` None = use NVLS when both symmetric buffers
        have a multicast mapping (torch reports 0 without NVLS); True =
        require it; False = P2P stores."""
        ptrs = (int(getattr(hY, "multicast_ptr", 0) or 0), int(getattr(hI, "multicast_ptr", 0) or 0))
        have = ptrs[0] != 0 and ptrs[1] != 0
        if multicast and not have:
            raise RuntimeError("NVLS multicast requested but the symmetric buffers have no multicast mapping")
        return ptrs if (have and multicast is not False) else None

    @classmethod
    def symmetric(cls, B: int, V: int, device, group=None, multicast: bool | None = False) -> "FusedVocabGather":
        """``multicast``: store through the NVLS multicast mapping (one
        multimem.st per result, replicated by the switch) instead of P2P
        stores to every peer — see ``pick_multicast``.  Off by default: the
        one-GPU hosts this was built on cannot create a multicast object
        (tools/nvls_probe.py), so the P2P path is the validated one."""
        import torch.distributed._symmetric_memory as symm_mem
        world, rank = _world(group)
        grp = group if group is not None else dist.group.WORLD
        Y = symm_mem.empty((B, V), dtype=torch.float32, device=device)
        I = symm_mem.empty((B, V), dtype=torch.int32, device=device)
        hY = symm_mem.rendezvous(Y, grp)
        hI = symm_mem.rendezvous(I, grp)
        peers = [(hY.buffer_ptrs[r], hI.buffer_ptrs[r]) for r in range(world) if r != rank]
        return cls(Y, I, peers, lambda ch: hY.barrier(channel=ch), keepalive=(hY, hI),
                   multicast=cls.pick_multicast(hY, hI, multicast))

    def forward(self, H, E_shard, bias_shard, mask, v0: int):
        v1 = v0 + E_shard.shape[0]
        if not 0 <= v0 <= v1 <= self.V:
            raise ValueError(f"shard columns [{v0}, {v1}) outside [0, {self.V})")
        self.barrier(0)
        if v1 > v0 and self.multicast is not None:
            ym, im = self.multicast
            sparton_forward(H, E_shard, bias_shard, mask, out=(self.Y[:, v0:v1], self.I[:, v0:v1]),
                            multicast_out=(ym + 4 * v0, im + 4 * v0))
        elif v1 > v0:
            sparton_forward(H, E_shard, bias_shard, mask, out=(self.Y[:, v0:v1], self.I[:, v0:v1]),
                            extra_out=tuple((y + 4 * v0, i + 4 * v0) for y, i in self.peers))
        self.barrier(1)
        return self.Y, self.I


class PeerDHReduce:
    """The partial-dH sum of the sharded head in one kernel over NVLink peer
    memory (``sparton_allreduce_peers``) instead of an NCCL
    all-reduce.

    Every rank owns a fp32 partial buffer ``part`` (the backward writes its
    shard's dH contribution straight into it, ``out_dH``) and an output buffer
    ``out`` in the gradient dtype, both addressable by every rank.  ``reduce``
    runs barrier → kernel → barrier on the current stream: rank r sums its
    slice of every rank's partial in rank order (deterministic, identical on
    all ranks, the fp32 accumulation of the reference) and stores it — fp32,
    or bf16 rounded once — into every rank's ``out``.  With ``multicast``
    (NVLS) the sum is one ``multimem.ld_reduce`` per 16 bytes and the store
    one ``multimem.st`` (``sparton_allreduce_multimem``).

    ``PeerDHReduce.symmetric(shape, dtype, device, group)`` is the production
    constructor (torch symmetric memory and its device barrier); the plain
    constructor takes already-mapped peer addresses (rank order, own
    included) and a barrier callable (the one-GPU test maps them by CUDA IPC)."""

    def __init__(self, part: torch.Tensor, out: torch.Tensor, part_ptrs, out_ptrs, rank: int,
                 barrier: Callable[[int], None], keepalive=(), multicast: tuple[int, int] | None = None):
        if part.dtype != torch.float32 or out.shape != part.shape or out.dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("part must be float32 and out float32/bfloat16 of the same shape")
        if len(part_ptrs) != len(out_ptrs) or not 1 <= len(part_ptrs) <= 8 or not 0 <= rank < len(part_ptrs):
            raise ValueError("one (part, out) address pair per rank, 1..8 ranks")
        if part.numel() % 4:
            raise ValueError("the reduced buffer must hold a multiple of 4 elements")
        self.part, self.out, self.rank, self.barrier = part, out, rank, barrier
        self.world = len(part_ptrs)
        self._parts = (ctypes.c_void_p * self.world)(*[int(p) for p in part_ptrs])
        self._outs = (ctypes.c_void_p * self.world)(*[int(p) for p in out_ptrs])
        self.multicast = None if multicast is None else (int(multicast[0]), int(multicast[1]))
        self._keepalive = keepalive

    @classmethod
    def symmetric(cls, shape, dtype, device, group=None, multicast: bool | None = False) -> "PeerDHReduce":
        """``multicast`` as ``FusedVocabGather.symmetric``: False = P2P loads
        and stores, True = require NVLS, None = NVLS when mapped."""
        import torch.distributed._symmetric_memory as symm_mem
        world, rank = _world(group)
        grp = group if group is not None else dist.group.WORLD
        part = symm_mem.empty(tuple(shape), dtype=torch.float32, device=device)
        out = symm_mem.empty(tuple(shape), dtype=dtype, device=device)
        hp = symm_mem.rendezvous(part, grp)
        ho = symm_mem.rendezvous(out, grp)
        return cls(part, out, [hp.buffer_ptrs[r] for r in range(world)], [ho.buffer_ptrs[r] for r in range(world)],
                   rank, lambda ch: hp.barrier(channel=ch), keepalive=(hp, ho),
                   multicast=FusedVocabGather.pick_multicast(hp, ho, multicast))

    def reduce(self) -> torch.Tensor:
        lib = _lib.load()
        od = _lib.SPARTON_BF16 if self.out.dtype == torch.bfloat16 else _lib.SPARTON_F32
        self.barrier(0)                       # every rank's partial is written
        with torch.cuda.device(self.part.device):
            if self.multicast is not None:
                rc = lib.sparton_allreduce_multimem(self.multicast[0], self.multicast[1], self.world, self.rank, od,
                                                    self.part.numel(), _stream_ptr())
            else:
                rc = lib.sparton_allreduce_peers(self._parts, self._outs, self.world, self.rank, od,
                                                 self.part.numel(), _stream_ptr())
        _lib.check(rc)
        self.barrier(1)                       # every rank's slice has landed in our `out`
        return self.out


def local_backward(H, E_shard, Y_p, I_p, dY_p, *, grad_dtype=torch.float32, include_bias_grad=True,
                   group=None, local_bwd: Callable | None = None, dh_reduce: PeerDHReduce | None = None):
    """Shard-local K2/K3, then the all-reduce of the partial dH (fp32).

    ``dY_p`` may be the column slice ``dY[:, v0:v1]`` of the replicated dY
    (passed with its row stride, no copy).  On CUDA with the library's
    backward, the all-reduce runs on its own stream as soon as dH is final
    (``dh_ready`` event) and overlaps the shard's dE, which the library runs
    on a side stream; the caller's stream waits for both.  The reduction is
    in fp32 (the reference accumulates in fp32), then cast to ``grad_dtype``
    (``reduce_dh``: reduce-scatter, cast, all-gather for a bf16 result)."""
    world, _ = _world(group)
    if dh_reduce is not None:
        # Partial dH straight into the peer-addressable buffer; the reduction
        # kernel runs on the communication stream once dH is final, beside dE.
        if dh_reduce.out.dtype != grad_dtype:
            raise ValueError(f"dh_reduce produces {dh_reduce.out.dtype}, asked for {grad_dtype}")
        main = torch.cuda.current_stream(H.device)
        ready = torch.cuda.Event()
        _, dE, db = sparton_backward(H, E_shard, Y_p, I_p, dY_p, include_bias_grad=include_bias_grad,
                                     grad_dtype=torch.float32, dh_ready=ready, out_dH=dh_reduce.part)
        comm = _comm_stream(H.device)
        comm.wait_event(ready)
        with torch.cuda.stream(comm):
            dH = dh_reduce.reduce()
        main.wait_stream(comm)
        if grad_dtype != torch.float32:
            dE = dE.to(grad_dtype)
        return dH, dE, db
    if local_bwd is not None or not H.is_cuda or world == 1:
        fn = local_bwd or sparton_backward
        dH, dE, db = fn(H, E_shard, Y_p, I_p, dY_p, include_bias_grad=include_bias_grad,
                        grad_dtype=torch.float32)
        dH = reduce_dh(dH, grad_dtype, group)
    else:
        main = torch.cuda.current_stream(H.device)
        ready = torch.cuda.Event()
        dH32, dE, db = sparton_backward(H, E_shard, Y_p, I_p, dY_p, include_bias_grad=include_bias_grad,
                                        grad_dtype=torch.float32, dh_ready=ready)
        comm = _comm_stream(H.device)
        comm.wait_event(ready)
        with torch.cuda.stream(comm):
            dH = reduce_dh(dH32, grad_dtype, group)
        dH32.record_stream(comm)
        dH.record_stream(comm)
        main.wait_stream(comm)
    if grad_dtype != torch.float32:
        dE = dE.to(grad_dtype)
    return dH, dE, db


_COMM_STREAMS: dict = {}


def _comm_stream(device) -> torch.cuda.Stream:
    key = torch.device(device).index
    s = _COMM_STREAMS.get(key)
    if s is None:
        s = _COMM_STREAMS[key] = torch.cuda.Stream(device=device)
    return s


def forward_sharded(H, E_shard, bias_shard, mask, V: int, *, group=None,
                    local_fn: Callable | None = None):
    """Full (Y, I) [B, V] from this rank's vocab shard of E/bias."""
    world, rank = _world(group)
    v0, v1, Vp = shard_range(V, world, rank)
    if E_shard.shape[0] != v1 - v0:
        raise ValueError(f"rank {rank} expects {v1 - v0} vocab rows, got {E_shard.shape[0]}")
    B = H.shape[0]
    fn = local_fn or local_forward
    if v1 > v0:
        Y_p, I_p = fn(H, E_shard, bias_shard, mask)
    else:
        Y_p = torch.zeros((B, 0), dtype=torch.float32, device=H.device)
        I_p = torch.zeros((B, 0), dtype=torch.int32, device=H.device)
    return gather_vocab(Y_p, I_p, V, Vp, group=group)


class ShardedSpartonHeadFn(torch.autograd.Function):
    """Autograd op for the vocab-sharded head: returns the full Y [B, V];
    gradients: dH (all-reduced), dE/db for this rank's shard only."""

    @staticmethod
    def forward(ctx, H, E_shard, bias_shard, mask, V, group=None):
        world, rank = _world(group)
        v0, v1, Vp = shard_range(V, world, rank)
        Y_p, I_p = local_forward(H, E_shard, bias_shard, mask)
        ctx.save_for_backward(H, E_shard, Y_p, I_p)
        ctx.v = (v0, v1)
        ctx.group = group
        Y, _ = gather_vocab(Y_p, I_p, V, Vp, group=group)
        return Y

    @staticmethod
    def backward(ctx, dY):
        H, E_shard, Y_p, I_p = ctx.saved_tensors
        v0, v1 = ctx.v
        dYs = dY[:, v0:v1]
        if dYs.dtype != torch.float32:
            dYs = dYs.float()
        dH, dE, db = local_backward(H, E_shard, Y_p, I_p, dYs, grad_dtype=H.dtype, group=ctx.group)
        return dH, dE.to(E_shard.dtype), db, None, None, None
