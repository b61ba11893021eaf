"""Data-parallel plumbing for FusedLoRA training on one node.

Token rows are independent, so microbatches shard across GPUs with the frozen base
weight replicated; the only exchange is one SUM all-reduce of the small fp32 adapter
gradients per optimizer step (NCCL over NVLink/NVSwitch on B200; gloo in CPU tests).

* :func:`assign_microbatches` — longest-processing-time assignment of microbatches to
  ranks by padded token count; the step time is the max over ranks, and
  :func:`imbalance` reports 1 − mean/max exactly as the reference's DP model
  (``simulate_dp``, ls/pipesim.py:275-312).
* :class:`AdapterGradReducer` — flattens every adapter gradient into fixed-size fp32
  buckets and all-reduces them asynchronously (launch after backward, or per layer as
  its gradients become ready), then scatters the result back into ``.grad``.
"""
from __future__ import annotations

import heapq
from typing import Iterable, Sequence

import torch
import torch.distributed as dist

from .errors import ValidationError


def assign_microbatches(token_counts: Sequence[int], world: int) -> list[list[int]]:
    """Indices of microbatches per rank (LPT greedy on padded tokens; deterministic)."""
    if world < 1:
        raise ValidationError(f"world size must be >= 1, got {world}")
    order = sorted(range(len(token_counts)), key=lambda i: (-int(token_counts[i]), i))
    heap = [(0, r) for r in range(world)]
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + int(token_counts[i]), r))
    for lst in out:
        lst.sort()
    return out


def rank_loads(token_counts: Sequence[int], assignment: Sequence[Sequence[int]]) -> list[int]:
    return [sum(int(token_counts[i]) for i in idx) for idx in assignment]


def imbalance(loads: Sequence[float]) -> float:
    """1 − mean/max over ranks (0 = perfectly balanced), as ls/pipesim.py:275-312."""
    mx = max(loads) if loads else 0
    return 0.0 if mx <= 0 else 1.0 - (sum(loads) / len(loads)) / mx


class AdapterGradReducer:
    """Bucketed async SUM all-reduce of adapter gradients (fp32)."""

    def __init__(self, params: Iterable[torch.nn.Parameter], bucket_bytes: int = 32 << 20, group=None,
                 average: bool = False):
        self.params = [p for p in params if p.requires_grad]
        if not self.params:
            raise ValidationError("no trainable adapter parameters to reduce")
        self.group = group
        self.average = average
        self.buckets: list[list[torch.nn.Parameter]] = []
        cur, size = [], 0
        for p in self.params:
            nbytes = p.numel() * 4
            if cur and size + nbytes > bucket_bytes:
                self.buckets.append(cur)
                cur, size = [], 0
            cur.append(p)
            size += nbytes
        if cur:
            self.buckets.append(cur)
        self._pending: list[tuple[list, torch.Tensor, object]] = []

    def launch(self) -> None:
        """Flatten and start the all-reduce of every bucket (non-blocking)."""
        for bucket in self.buckets:
            flat = torch.cat([(p.grad if p.grad is not None else torch.zeros_like(p)).reshape(-1).float()
                              for p in bucket])
            work = dist.all_reduce(flat, group=self.group, async_op=True)
            self._pending.append((bucket, flat, work))

    def wait(self) -> None:
        """Finish the reductions and write the summed (or averaged) gradients back."""
        world = dist.get_world_size(self.group)
        for bucket, flat, work in self._pending:
            work.wait()
            if self.average:
                flat.div_(world)
            off = 0
            for p in bucket:
                n = p.numel()
                g = flat[off:off + n].view_as(p).to(p.dtype)
                if p.grad is None:
                    p.grad = g.clone()
                else:
                    p.grad.copy_(g)
                off += n
        self._pending.clear()

    def reduce(self) -> None:
        self.launch()
        self.wait()
