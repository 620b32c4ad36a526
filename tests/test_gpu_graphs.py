"""CUDA-graph capture of the head (the framework's answer to a tracing
compiler, for launch-bound small shapes such as SPLADE query batches): the
forward + backward captured once and replayed give bit-for-bit the eager
results on every path — staged dE (S <= 832), gathered dE (S > 832),
multi-pass dH with the fp32 carry, the sparse regime, fp32 and bf16
gradients.  The library enqueues only stream-ordered work (its side stream
joins the capturing stream through events), so capture needs nothing
special from the caller."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


def _inputs(B, S, D, V, dev, bias=0.0):
    g = torch.Generator(device=dev).manual_seed(3)
    H = torch.randn((B, S, D), generator=g, device=dev).to(torch.bfloat16)
    E = (torch.randn((V, D), generator=g, device=dev) * 0.05).to(torch.bfloat16)
    b = torch.randn(V, generator=g, device=dev) * 0.1 + bias
    m = (torch.rand((B, S), generator=g, device=dev) < 0.9).to(torch.uint8)
    dY = torch.randn((B, V), generator=g, device=dev)
    return H, E, b, m, dY


@pytest.mark.parametrize("dims,bias", [((8, 128, 768, 30522), 0.0),      # cfg1 shape, one dH pass
                                       ((4, 512, 768, 100000), 0.0),     # 4 dH passes (fp32 carry)
                                       ((3, 1000, 256, 20000), 0.0),     # gathered dE (S > 832)
                                       ((4, 512, 768, 100000), -2.0)])   # sparse-regime backward
@pytest.mark.parametrize("grad_dtype", [torch.bfloat16, torch.float32])
def test_graph_replay_equals_eager(cuda_device, dims, bias, grad_dtype):
    from paper_2603_25011_b200 import sparton_backward, sparton_forward
    H, E, b, m, dY = _inputs(*dims, cuda_device, bias)
    Y0, I0 = sparton_forward(H, E, b, m)
    ref = sparton_backward(H, E, Y0, I0, dY, grad_dtype=grad_dtype)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):                 # warm-up outside the capture (allocator, attributes)
        for _ in range(2):
            Y, I = sparton_forward(H, E, b, m)
            sparton_backward(H, E, Y, I, dY, grad_dtype=grad_dtype)
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        Y, I = sparton_forward(H, E, b, m)
        grads = sparton_backward(H, E, Y, I, dY, grad_dtype=grad_dtype)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(Y, Y0) and torch.equal(I, I0)
    for got, want in zip(grads, ref):
        assert torch.equal(got, want)
    # new inputs copied into the captured buffers are picked up by the replay
    H.mul_(-1.0)
    graph.replay()
    Y1, I1 = sparton_forward(H, E, b, m)
    torch.cuda.synchronize()
    assert torch.equal(Y, Y1) and torch.equal(I, I1)
