"""End-to-end SPLADE training step: the fused Sparton
head and the naive PyTorch head (fp32 logits) give the same loss and the same
parameter gradients on the same random-init encoder; a few optimiser steps
with the fused head stay finite.  There is no reference implementation of the
training step, so parity is anchored on the head.
Tolerance: loss rtol 1e-3; gradients relative L2 error <= 1e-2 (bf16 head
inputs on both sides, fp32 accumulation)."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


def _tiny():
    from paper_2603_25011_b200.splade import EncoderConfig
    return EncoderConfig(vocab=3001, hidden=256, layers=2, heads=4, ffn=512, max_len=128)


def _grads_and_loss(head_fn, seed=0):
    from paper_2603_25011_b200.splade import SpladeTrainer, splade_loss, synthetic_batch
    tr = SpladeTrainer(_tiny(), head="sparton", seed=seed)
    q, qm, d, dm = synthetic_batch(6, 16, 48, 3001, "cuda", seed=seed)
    m = tr.model
    with torch.autocast("cuda", dtype=torch.bfloat16):
        Hq = m.hidden_states(q, qm)
        Hd = m.hidden_states(d, dm)
    Yq = head_fn(Hq.to(torch.bfloat16), m.word.weight, m.vocab_bias, qm)
    Yd = head_fn(Hd.to(torch.bfloat16), m.word.weight, m.vocab_bias, dm)
    loss, _ = splade_loss(Yq, Yd)
    loss.backward()
    return float(loss), {n: p.grad.detach().float().clone() for n, p in m.named_parameters() if p.grad is not None}


def test_fused_head_matches_naive_head_in_training_step(cuda_device):
    from paper_2603_25011_b200.splade import naive_splade_head, sparton_splade_head
    lf, gf = _grads_and_loss(sparton_splade_head)
    ln, gn = _grads_and_loss(lambda H, E, b, m: naive_splade_head(H, E, b, m, compute_dtype=torch.float32))
    assert abs(lf - ln) <= 1e-3 * abs(ln), (lf, ln)
    assert set(gf) == set(gn)
    errs = {n: float((gf[n] - gn[n]).norm() / max(gn[n].norm(), 1e-12)) for n in gf}
    assert max(errs.values()) <= 1e-2, errs


def test_training_steps_finite_and_loss_moves(cuda_device):
    from paper_2603_25011_b200.splade import SpladeTrainer, synthetic_batch
    tr = SpladeTrainer(_tiny(), head="sparton", lr=1e-3)
    batch = synthetic_batch(8, 16, 48, 3001, "cuda", seed=3)
    losses = [float(tr.step(*batch)) for _ in range(5)]
    assert all(torch.isfinite(torch.tensor(losses)))
    assert losses[-1] < losses[0]
