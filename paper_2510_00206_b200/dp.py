"""Data-parallel plumbing for FusedLoRA training on one node.

Token rows are independent, so microbatches shard across GPUs with the frozen base
weight replicated; the only exchange is one SUM all-reduce of the small fp32 adapter
gradients per optimizer step (NCCL over NVLink/NVSwitch on B200; gloo in CPU tests).

* :func:`assign_microbatches` — longest-processing-time assignment of microbatches to
  ranks by padded token count; the step time is the max over ranks, and
  :func:`imbalance` reports 1 − mean/max exactly as the reference's DP model
  (``simulate_dp``, ls/pipesim.py:275-312).
* :class:`AdapterGradReducer` — flattens every adapter gradient into fixed-size fp32
  buckets and all-reduces them asynchronously, then scatters the result back into
  ``.grad``. Either after backward (``reduce``), or overlapped with it: ``attach()``
  registers post-accumulate-grad hooks, ``arm()`` before the step's last backward, and
  each bucket's all-reduce starts the moment its last gradient is final (the backward of
  the remaining layers runs underneath, as in DDP); ``wait()`` finishes the step.
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
        # buckets in reverse registration order: backward finalizes the last layers first
        for p in reversed(self.params):
            nbytes = p.numel() * 4
            if cur and size + nbytes > bucket_bytes:
                self.buckets.append(cur)
                cur, size = [], 0
            cur.append(p)
            size += nbytes
        if cur:
            self.buckets.append(cur)
        self._pending: list[tuple[list, torch.Tensor, object]] = []
        self._bucket_of = {id(p): b for b, bucket in enumerate(self.buckets) for p in bucket}
        self._hooks: list = []
        self._armed = False
        self._ready: list[int] = []
        self._launched: list[bool] = []

    def _launch_bucket(self, b: int) -> None:
        bucket = self.buckets[b]
        flat = torch.cat([(p.grad if p.grad is not None else torch.zeros_like(p)).reshape(-1).float()
                          for p in bucket])
        work = dist.all_reduce(flat, group=self.group, async_op=True)
        self._pending.append((bucket, flat, work))
        self._launched[b] = True

    def launch(self) -> None:
        """Flatten and start the all-reduce of every bucket not yet started (non-blocking,
        in bucket order)."""
        if len(self._launched) != len(self.buckets):
            self._launched = [False] * len(self.buckets)
        for b in range(len(self.buckets)):
            if not self._launched[b]:
                self._launch_bucket(b)
        self._next = len(self.buckets)

    # -- overlap with backward ---------------------------------------------------------
    def attach(self) -> "AdapterGradReducer":
        """Register the post-accumulate-grad hooks that drive ``arm()``ed steps."""
        if not self._hooks:
            self._hooks = [p.register_post_accumulate_grad_hook(self._on_grad) for p in self.params]
        return self

    def detach(self) -> None:
        for h in self._hooks:
            h.remove()
        self._hooks = []

    def arm(self) -> None:
        """The next backward is the step's last: launch buckets as they complete. Buckets
        start strictly in index order on every rank (collectives must match across ranks:
        a bucket whose gradients are final waits for the ones before it), each exactly
        once per armed step; ``wait`` launches those that never completed (parameters
        without a gradient in this backward)."""
        if not self._hooks:
            raise ValidationError("attach() the reducer before arm()")
        self._armed = True
        self._ready = [0] * len(self.buckets)
        self._launched = [False] * len(self.buckets)
        self._next = 0

    def _on_grad(self, p: torch.Tensor) -> None:
        if not self._armed:
            return
        self._ready[self._bucket_of[id(p)]] += 1
        while self._next < len(self.buckets) and self._ready[self._next] == len(self.buckets[self._next]):
            self._launch_bucket(self._next)
            self._next += 1

    def wait(self) -> None:
        """Finish the reductions and write the summed (or averaged) gradients back."""
        if self._armed:
            self.launch()  # buckets whose parameters received no gradient this step
            self._armed = False
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
        self._launched = [False] * len(self.buckets)
        self.launch()
        self.wait()
