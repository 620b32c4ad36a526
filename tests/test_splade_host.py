"""Host-side pieces of the end-to-end SPLADE step (CPU): the loss matches its
definition, the synthetic batch is well-formed, and the fused head refuses
CPU tensors (no CPU fallback)."""

from __future__ import annotations

import math

import pytest
import torch


def test_splade_loss_definition():
    from paper_2603_25011_b200.splade import splade_loss
    g = torch.Generator().manual_seed(0)
    Yq = torch.rand((4, 11), generator=g)
    Yd = torch.rand((4, 11), generator=g)
    loss, parts = splade_loss(Yq, Yd, lambda_q=0.5, lambda_d=0.25)
    scores = Yq @ Yd.t()
    ce = -sum(math.log(math.exp(scores[i, i]) / float(torch.exp(scores[i]).sum())) for i in range(4)) / 4
    fq = float((Yq.mean(0) ** 2).sum())
    fd = float((Yd.mean(0) ** 2).sum())
    assert float(loss) == pytest.approx(ce + 0.5 * fq + 0.25 * fd, rel=1e-5)
    assert float(parts["flops_q"]) == pytest.approx(fq, rel=1e-6)


def test_synthetic_batch_masks_are_prefixes():
    from paper_2603_25011_b200.splade import synthetic_batch
    q, qm, d, dm = synthetic_batch(5, 8, 16, 100, "cpu", seed=1)
    assert q.shape == (5, 8) and d.shape == (5, 16) and qm.dtype == torch.uint8
    for m in (qm, dm):
        lens = m.sum(1)
        assert (lens >= 1).all()
        assert torch.equal(m, (torch.arange(m.shape[1])[None] < lens[:, None]).to(torch.uint8))
    assert int(q.min()) >= 1 and int(q.max()) < 100


def test_fused_head_has_no_cpu_path():
    from paper_2603_25011_b200.splade import sparton_splade_head
    H = torch.zeros((1, 2, 8), dtype=torch.bfloat16)
    E = torch.zeros((3, 8))
    with pytest.raises(RuntimeError):
        sparton_splade_head(H, E, torch.zeros(3), torch.ones((1, 2), dtype=torch.uint8))


def test_naive_head_matches_definition_on_cpu():
    from paper_2603_25011_b200.splade import naive_splade_head
    g = torch.Generator().manual_seed(2)
    H = torch.randn((2, 5, 8), generator=g)
    E = torch.randn((7, 8), generator=g)
    b = torch.randn(7, generator=g)
    m = torch.tensor([[1, 1, 1, 0, 0], [1, 1, 1, 1, 1]], dtype=torch.uint8)
    Y = naive_splade_head(H, E, b, m, compute_dtype=torch.float32)
    Eb = E.to(torch.bfloat16).float()
    L = (H @ Eb.t() + b) * m[..., None]
    assert torch.allclose(Y, torch.log1p(torch.relu(L.amax(1))), rtol=1e-6, atol=1e-6)
