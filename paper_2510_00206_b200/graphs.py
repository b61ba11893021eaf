"""CUDA-graph capture of fused LoRA training steps.

A FusedLoRA forward+backward is a handful of launches plus host work (segment plan,
C-ABI argument packing, autograd); at small token counts (C1: 2048 tokens) the host side
takes longer than the kernels. Capturing the whole step once and replaying it removes
the host from the loop. Layers must be built with ``capturable=True`` so the Philox step
counter advances on the device (a fresh dropout mask per replay, SPEC.md §3) and the bf16
operands are persistent copies the graph reads at fixed addresses (functional.ShadowOperands):
refreshed after every optimizer step and, before each replay, for any adapter weight whose
in-place version changed (updates through ``p.data`` need invalidate_operand_caches()).

    step = GraphedStep(lambda: train_step(...))   # warm-up + capture
    for _ in range(n):
        step.replay()

Inputs/outputs of the captured region are static: refill input tensors in place (copy_)
before a replay; gradients land in the same ``.grad`` tensors every replay.
"""
from __future__ import annotations

from typing import Callable

import torch

from .errors import ValidationError
from .functional import refresh_stale_operand_shadows


class GraphedStep:
    """Warm ``fn`` up on a side stream, then capture one call of it into a CUDA graph."""

    def __init__(self, fn: Callable[[], object], warmup: int = 3, pool=None):
        if not torch.cuda.is_available():
            raise ValidationError("CUDA graphs need a CUDA device")
        self.fn = fn
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                fn()
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, pool=pool):
            out = fn()
        # keep only the static output buffer, never the captured autograd graph (a live
        # graph pins AccumulateGrad nodes to the capture stream)
        self.output = out.detach() if isinstance(out, torch.Tensor) else out

    def replay(self):
        refresh_stale_operand_shadows()  # adapter weights changed in place since the last replay
        self.graph.replay()
        return self.output
