"""The unfused PEFT-style torch LoRA linear: the denominator of the ">= 1.25x" target.

Y = F.linear(X, W) + scaling * F.linear(F.linear(dropout(X), A), B) with W frozen — cuBLAS
GEMMs plus elementwise kernels, the "torch LoRA" the paper measures against (PAPER.md:
269-292, 707). Its kernel list is the reference's ``unfused`` variant
(ls/costmodel.py:230-249). Dropout may take an explicit keep mask so the baseline and the
fused layer can be compared on the same mask.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F


def unfused_lora(x, weight, lora_a, lora_b, scaling: float, dropout_p: float = 0.0, keep_mask=None,
                 training: bool = True):
    if training and keep_mask is not None:
        xd = x * keep_mask.to(x.dtype) * (1.0 / (1.0 - dropout_p))
    elif training and dropout_p > 0:
        xd = F.dropout(x, dropout_p, training=True)
    else:
        xd = x
    return F.linear(x, weight) + scaling * F.linear(F.linear(xd, lora_a), lora_b)


def unfused_multi_lora(x, weight, lora_a, lora_b, adapters, segments, training: bool = True):
    """Torch multi-adapter LoRA over a packed microbatch: one cuBLAS base GEMM, then a
    per-segment loop of dropout + the adapter's two skinny GEMMs + scale, concatenated back
    (rows outside every segment get no LoRA term). The paper's "torch LoRA" for mixed-adapter
    batches."""
    y = F.linear(x, weight)
    parts, row = [], 0
    for seg in sorted(segments, key=lambda s: s.row_start):
        if seg.row_start > row:
            parts.append(x.new_zeros(seg.row_start - row, weight.shape[0]))
        cfg = adapters[seg.adapter]
        xs = x[seg.row_start:seg.row_end]
        xd = F.dropout(xs, cfg.dropout_p, training=True) if training and cfg.dropout_p > 0 else xs
        parts.append(cfg.scaling * F.linear(F.linear(xd, lora_a[seg.adapter]), lora_b[seg.adapter]))
        row = seg.row_end
    if row < x.shape[0]:
        parts.append(x.new_zeros(x.shape[0] - row, weight.shape[0]))
    return y + torch.cat(parts)
