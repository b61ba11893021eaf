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
