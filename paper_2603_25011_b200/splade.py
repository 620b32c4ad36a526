"""End-to-end SPLADE training step with the Sparton head (SURVEY.md §8f rank 1,
BASELINE.json configs[4]).

A DistilBERT-shaped encoder (6 layers, hidden 768, 12 heads, FFN 3072,
vocabulary 30522, random init; torch modules are plumbing here) produces hidden
states H; the MLM transform (dense + GELU + LayerNorm) feeds the SPLADE head
``Y = max_s log1p(relu(H_s·Eᵀ + b)) · M_s`` whose vocabulary projection E is
tied to the word embeddings, exactly as in SPLADE/DistilBERT.  The head is
either the fused sm_100a Sparton head (``SpartonHeadFn``: B×V output, argmax
routed backward) or the naive PyTorch composition that materialises the
B×S×V logits — same math, same parameters.

Loss (the paper's training objective, §5): in-batch contrastive
InfoNCE over query/document sparse vectors, scores = Y_q·Y_dᵀ, plus the FLOPS
regulariser Σ_v (mean_b Y[b, v])² for queries and documents.

There is no reference implementation of this step (SPEC.md:16 scopes it out),
so parity is anchored on the head: ``tests/test_gpu_splade.py`` checks that
both heads give the same loss and gradients on the same model.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn as nn
import torch.nn.functional as F

from .head import SpartonHeadFn


@dataclass
class EncoderConfig:
    vocab: int = 30522
    hidden: int = 768
    layers: int = 6
    heads: int = 12
    ffn: int = 3072
    max_len: int = 512


class SpladeEncoder(nn.Module):
    """DistilBERT-shaped encoder + MLM transform; the vocabulary projection is
    the (tied) word-embedding matrix, consumed by the SPLADE head."""

    def __init__(self, cfg: EncoderConfig):
        super().__init__()
        self.cfg = cfg
        self.word = nn.Embedding(cfg.vocab, cfg.hidden)
        self.pos = nn.Embedding(cfg.max_len, cfg.hidden)
        self.emb_ln = nn.LayerNorm(cfg.hidden)
        layer = nn.TransformerEncoderLayer(cfg.hidden, cfg.heads, cfg.ffn, dropout=0.0, activation="gelu",
                                           batch_first=True, norm_first=False)
        self.encoder = nn.TransformerEncoder(layer, cfg.layers, enable_nested_tensor=False)
        self.mlm_dense = nn.Linear(cfg.hidden, cfg.hidden)
        self.mlm_ln = nn.LayerNorm(cfg.hidden)
        self.vocab_bias = nn.Parameter(torch.zeros(cfg.vocab))
        nn.init.normal_(self.word.weight, std=0.02)
        nn.init.normal_(self.pos.weight, std=0.02)

    def hidden_states(self, ids: torch.Tensor, mask: torch.Tensor) -> torch.Tensor:
        """(B, S) token ids + (B, S) {0,1} mask -> (B, S, hidden) MLM-transformed states."""
        S = ids.shape[1]
        pos = torch.arange(S, device=ids.device)
        x = self.emb_ln(self.word(ids) + self.pos(pos)[None])
        x = self.encoder(x, src_key_padding_mask=~mask.bool())
        return self.mlm_ln(F.gelu(self.mlm_dense(x)))


def sparton_splade_head(H: torch.Tensor, E: torch.Tensor, bias: torch.Tensor, mask: torch.Tensor) -> torch.Tensor:
    """Fused head: H (B,S,D) bf16, E (V,D) -> Y (B,V) f32.  Gradients flow to H, E, bias."""
    Y, _ = SpartonHeadFn.apply(H.contiguous(), E.to(torch.bfloat16).contiguous(), bias.float().contiguous(),
                               mask.to(torch.uint8).contiguous(), True)
    return Y


def naive_splade_head(H: torch.Tensor, E: torch.Tensor, bias: torch.Tensor, mask: torch.Tensor,
                      compute_dtype: torch.dtype | None = None) -> torch.Tensor:
    """The unfused composition: materialises B×S×V logits (in H's dtype, bf16 in
    training; fp32 when ``compute_dtype`` says so, for parity checks)."""
    dt = compute_dtype or H.dtype
    Eb = E.to(torch.bfloat16)          # the head consumes bf16 E either way
    L = (H.to(dt) @ Eb.to(dt).t() + bias.to(dt)) * mask[..., None].to(dt)
    return L.relu().log1p().amax(dim=1).float()


HEADS = {"sparton": sparton_splade_head, "naive": naive_splade_head}


def splade_loss(Yq: torch.Tensor, Yd: torch.Tensor, lambda_q: float = 3e-4, lambda_d: float = 1e-4,
                temperature: float = 1.0) -> tuple[torch.Tensor, dict]:
    """In-batch contrastive InfoNCE (document i is the positive of query i) plus
    the FLOPS regulariser sum_v (mean_b Y[b, v])^2 on queries and documents."""
    scores = (Yq @ Yd.t()) / temperature
    target = torch.arange(Yq.shape[0], device=Yq.device)
    ce = F.cross_entropy(scores, target)
    flops_q = (Yq.mean(dim=0) ** 2).sum()
    flops_d = (Yd.mean(dim=0) ** 2).sum()
    loss = ce + lambda_q * flops_q + lambda_d * flops_d
    return loss, {"ce": ce.detach(), "flops_q": flops_q.detach(), "flops_d": flops_d.detach()}


class SpladeTrainer:
    """One optimiser step = encode queries and documents, SPLADE head, loss,
    backward, AdamW update.  bf16 autocast for the encoder; fp32 master weights."""

    def __init__(self, cfg: EncoderConfig | None = None, head: str = "sparton", lr: float = 2e-5,
                 device: torch.device | str = "cuda", seed: int = 0):
        torch.manual_seed(seed)
        self.model = SpladeEncoder(cfg or EncoderConfig()).to(device)
        self.head = HEADS[head]
        self.opt = torch.optim.AdamW(self.model.parameters(), lr=lr, fused=True)

    def loss(self, q_ids, q_mask, d_ids, d_mask):
        m = self.model
        with torch.autocast("cuda", dtype=torch.bfloat16):
            Hq = m.hidden_states(q_ids, q_mask)
            Hd = m.hidden_states(d_ids, d_mask)
        Yq = self.head(Hq.to(torch.bfloat16), m.word.weight, m.vocab_bias, q_mask)
        Yd = self.head(Hd.to(torch.bfloat16), m.word.weight, m.vocab_bias, d_mask)
        return splade_loss(Yq, Yd)

    def step(self, q_ids, q_mask, d_ids, d_mask) -> float:
        self.opt.zero_grad(set_to_none=True)
        loss, _ = self.loss(q_ids, q_mask, d_ids, d_mask)
        loss.backward()
        self.opt.step()
        return loss.detach()


def synthetic_batch(B: int, Sq: int, Sd: int, vocab: int, device, seed: int = 0):
    """Random token ids with ragged lengths (padding masked out), as a retrieval batch."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    q_ids = torch.randint(1, vocab, (B, Sq), generator=g)
    d_ids = torch.randint(1, vocab, (B, Sd), generator=g)
    q_len = torch.randint(max(1, Sq // 4), Sq + 1, (B,), generator=g)
    d_len = torch.randint(max(1, Sd // 2), Sd + 1, (B,), generator=g)
    q_mask = (torch.arange(Sq)[None] < q_len[:, None]).to(torch.uint8)
    d_mask = (torch.arange(Sd)[None] < d_len[:, None]).to(torch.uint8)
    return tuple(t.to(device) for t in (q_ids, q_mask, d_ids, d_mask))


def step_flops_head(B: int, Sq: int, Sd: int, cfg: EncoderConfig) -> float:
    """Algorithmic head FLOPs per step (forward 2·B·S·V·D + backward 4·B·V·D, both sides)."""
    D, V = cfg.hidden, cfg.vocab
    return sum(2 * B * S * V * D + 4 * B * V * D for S in (Sq, Sd))


__all__ = ["EncoderConfig", "SpladeEncoder", "SpladeTrainer", "splade_loss", "sparton_splade_head",
           "naive_splade_head", "synthetic_batch", "step_flops_head", "HEADS"]
