"""End-to-end SPLADE training step (BASELINE.json configs[4]): DistilBERT-shaped
random-init encoder + SPLADE head + in-batch InfoNCE + FLOPS regulariser, AdamW.
For each head (fused Sparton / naive PyTorch) doubles the batch until OOM and
reports step time and peak HBM per batch size; prints one JSON line per point."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2603_25011_b200.splade import EncoderConfig, SpladeTrainer, step_flops_head, synthetic_batch  # noqa: E402

SQ, SD = int(sys.argv[1]) if len(sys.argv) > 1 else 64, int(sys.argv[2]) if len(sys.argv) > 2 else 256
VOCAB = int(sys.argv[3]) if len(sys.argv) > 3 else 30522      # 250002: the XLM-R vocabulary (paper's 26x-batch case)
cfg = EncoderConfig(vocab=VOCAB)
for head in ("sparton", "naive"):
    B = 8 if VOCAB > 100000 else 64
    while B <= 8192:
        torch.cuda.empty_cache()
        torch.cuda.reset_peak_memory_stats()
        try:
            tr = SpladeTrainer(cfg, head=head)
            batch = synthetic_batch(B, SQ, SD, cfg.vocab, "cuda")
            for _ in range(2):
                tr.step(*batch)
            torch.cuda.synchronize()
            n = 5
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(n):
                loss = tr.step(*batch)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / n
            print(json.dumps({"head": head, "V": VOCAB, "B": B, "Sq": SQ, "Sd": SD, "ms_per_step": ms,
                              "pairs_per_s": B / ms * 1e3, "peak_hbm_gb": torch.cuda.max_memory_allocated() / 1e9,
                              "head_tflops_alg": step_flops_head(B, SQ, SD, cfg) / ms / 1e9,
                              "loss": float(loss)}), flush=True)
        except torch.OutOfMemoryError:
            print(json.dumps({"head": head, "V": VOCAB, "B": B, "Sq": SQ, "Sd": SD, "result": "OOM"}), flush=True)
            break
        finally:
            tr = batch = None
        B *= 2
