"""``FusedLoRA`` and ``FusedMultiLoRA`` modules (PEFT-compatible parameter names).

Both wrap a frozen ``nn.Linear`` (or its weight) and keep adapter parameters under the
PEFT names ``lora_A.weight`` (r x k) and ``lora_B.weight`` (n x r), so a PEFT/HF LoRA
layer's state dict maps onto them directly. Adapter parameters default to fp32 master
weights: their bf16 rank-concat operands are built once per weight update and reused
(functional.OperandCache, keyed by the parameters' in-place versions), and gradients
arrive in fp32 for the optimizer and the DP all-reduce; the base weight and activations
are bf16.

Dropout masks come from SPEC.md §3's counter-based Philox stream keyed by the adapter
seed and a per-forward 64-bit offset; backward reuses the forward's pair through the
packed keep mask, so no byte mask is ever stored. Where the offset comes from
(``dropout_rng``):

* ``"torch"`` (default without ``capturable``): drawn from torch's CUDA generator on the
  device (one int64 per training forward) — dropout then follows ``torch.manual_seed`` like
  ``nn.Dropout`` and ``torch.utils.checkpoint`` (which restores the RNG state before
  recomputing) redraws the original mask.
* ``"counter"`` (default with ``capturable=True``): a per-module step counter (on the host,
  or on the device for capturable modules), advanced once per training forward —
  deterministic offsets 0, 1, 2, ... that ``dropout_state()`` saves and restores. A CUDA
  graph replays it with one tiny add per forward; a random draw inside a graph costs a
  launch gap of ~30 µs per forward on B200 (profiles/r02_step_breakdown.txt). Not
  checkpoint-safe: a recomputed forward would advance it again.
"""
from __future__ import annotations

import math
from typing import Sequence

import torch
from torch import nn

from . import _lib
from .errors import ValidationError
from .functional import (OperandCache, ShadowOperands, _apply, _cache_handle, _check_call, _EmptyBatchFn,
                         _flatten_input, fused_multi_lora, pack_adapters)
from .plan import AdapterConfig, Segment


def _init_lora(a: nn.Linear, b: nn.Linear, init: str, generator: torch.Generator | None = None) -> None:
    with torch.no_grad():
        if init == "peft":
            # PEFT default: kaiming-uniform A, zero B
            nn.init.kaiming_uniform_(a.weight, a=math.sqrt(5), generator=generator)
            nn.init.zeros_(b.weight)
        elif init == "gaussian":
            k = a.weight.shape[1]
            a.weight.uniform_(-1.0 / math.sqrt(k), 1.0 / math.sqrt(k), generator=generator)
            b.weight.normal_(0.0, 1.0 / math.sqrt(b.weight.shape[1]), generator=generator)
        else:
            raise ValidationError(f"unknown init {init!r} (expected 'peft' or 'gaussian')")


def _frozen_base(base: nn.Linear | torch.Tensor) -> tuple[torch.Tensor, torch.Tensor | None]:
    """The frozen base weight (and bias): only the adapters train, so both stop requiring grad."""
    if isinstance(base, nn.Linear):
        w, bias = base.weight, base.bias
        if bias is not None:
            bias.requires_grad_(False)
    elif isinstance(base, torch.Tensor):
        w, bias = base, None
    else:
        raise ValidationError("base must be an nn.Linear or a weight tensor of shape (out_features, in_features)")
    if w.dim() != 2:
        raise ValidationError("base weight must be 2-D (out_features, in_features)")
    return w, bias


_DROPOUT_RNGS = ("torch", "counter")


def _init_capturable(mod: nn.Module, capturable: bool, device, dropout_rng: str | None) -> None:
    """``capturable=True`` (as torch.optim's flag): the bf16 operand copies of the fp32
    adapter weights are re-cast inside each call (no host-side cache), and in ``"counter"``
    mode the Philox step counter lives on the device and is advanced there by every training
    forward — so a forward+backward captured in a CUDA graph replays with a fresh dropout
    mask and the current weights (``"torch"`` mode draws its offsets on the device anyway)."""
    if dropout_rng is None:
        dropout_rng = "counter" if capturable else "torch"
    if dropout_rng not in _DROPOUT_RNGS:
        raise ValidationError(f"dropout_rng must be one of {_DROPOUT_RNGS}, got {dropout_rng!r}")
    mod.capturable = bool(capturable)
    mod.dropout_rng = dropout_rng
    if mod.capturable and dropout_rng == "counter":
        mod.register_buffer("step_counter", torch.zeros(1, dtype=torch.int64, device=device), persistent=False)


def _dropout_state(mod: nn.Module) -> dict:
    """The Philox step counter, for checkpoints (``"counter"`` mode): restoring it makes a
    resumed run draw exactly the dropout masks the uninterrupted run would have drawn
    (SPEC.md §3). In ``"torch"`` mode the offsets follow torch's RNG state, which training
    checkpoints save themselves. Kept out of ``state_dict`` so PEFT-style state dicts load
    strictly into the modules."""
    if mod.dropout_rng == "torch":
        return {"dropout_rng": "torch"}
    step = int(mod.step_counter.item()) if mod.capturable else int(mod._offset)
    return {"philox_step": step, "capturable": mod.capturable, "dropout_rng": "counter"}


def _load_dropout_state(mod: nn.Module, state: dict) -> None:
    if mod.dropout_rng == "torch":
        return
    step = int(state.get("philox_step", 0))
    if mod.capturable:
        with torch.no_grad():
            mod.step_counter.fill_(step)
    else:
        mod._offset = step


_OFFSET_HIGH = 2**62


def _step_offsets(mod: nn.Module, device: torch.device, has_dropout: bool) -> tuple[int, torch.Tensor | None]:
    """(host offset, device offset) of this forward (SPEC.md §3)."""
    if not mod.training or not has_dropout:
        return 0, None
    if mod.dropout_rng == "torch":
        return 0, torch.randint(0, _OFFSET_HIGH, (1,), dtype=torch.int64, device=device)
    if mod.capturable:
        mod.step_counter.add_(1)  # on the device: captured into a graph with the kernels
        return 0, mod.step_counter
    return mod.next_offset(), None


class FusedLoRA(nn.Module):
    """Single-adapter LoRA linear: Y = X·Wᵀ (+ bias) + scaling·dropout(X)·Aᵀ·Bᵀ."""

    def __init__(
        self,
        base: nn.Linear | torch.Tensor,
        rank: int,
        scaling: float | None = None,
        dropout_p: float = 0.0,
        *,
        alpha: float | None = None,
        seed: int = 0,
        init: str = "peft",
        dtype: torch.dtype = torch.float32,
        generator: torch.Generator | None = None,
        capturable: bool = False,
        dropout_rng: str | None = None,
    ):
        super().__init__()
        w, bias = _frozen_base(base)
        w.requires_grad_(False)
        self.base = base if isinstance(base, nn.Linear) else None
        self.register_buffer("weight", w, persistent=False) if self.base is None else None
        self.out_features, self.in_features = w.shape
        _init_capturable(self, capturable, w.device, dropout_rng)
        if scaling is None:
            scaling = (alpha if alpha is not None else 32.0) / rank
        self.config = AdapterConfig(rank=rank, scaling=float(scaling), dropout_p=float(dropout_p), seed=int(seed))
        self._packed = pack_adapters([self.config])
        dev = w.device
        self.lora_A = nn.Linear(self.in_features, rank, bias=False, device=dev, dtype=dtype)
        self.lora_B = nn.Linear(rank, self.out_features, bias=False, device=dev, dtype=dtype)
        _init_lora(self.lora_A, self.lora_B, init, generator)
        self._offset = 0
        # bf16 operands: a version-keyed cache (eager), or persistent copies a CUDA graph can
        # read at fixed addresses, refreshed after every optimizer step (capturable)
        self._operands = ShadowOperands() if capturable else OperandCache()

    @property
    def base_weight(self) -> torch.Tensor:
        return self.base.weight if self.base is not None else self.weight

    @property
    def base_bias(self) -> torch.Tensor | None:
        return self.base.bias if self.base is not None else None

    def next_offset(self) -> int:
        off = self._offset
        self._offset += 1
        return off

    def dropout_state(self) -> dict:
        return _dropout_state(self)

    def load_dropout_state(self, state: dict) -> None:
        _load_dropout_state(self, state)

    def invalidate_operands(self) -> None:
        """Drop the cached bf16 operands (after changing lora_A/lora_B outside an optimizer step)."""
        self._operands.clear()

    def forward(self, x: torch.Tensor, keep_mask: torch.Tensor | None = None) -> torch.Tensor:
        k, n = self.in_features, self.out_features
        w = self.base_weight
        x2, lead = _flatten_input(x, k)
        a, b = self.lora_A.weight, self.lora_B.weight
        _check_call(x2, w, [a], [b], self._packed[0], k, n, keep_mask, None)
        m = x2.shape[0]
        if m == 0:
            y = _EmptyBatchFn.apply(x2, n, a, b)
        else:
            off, off_dev = _step_offsets(self, x2.device, self.config.dropout_p > 0 and keep_mask is None)
            y = _apply(x2, w, [a], [b], self._packed, [0, 0, m, 0], off, off_dev, keep_mask, self.training, True, 0,
                       _cache_handle(self._operands))
        y = y.reshape(lead + (n,))
        if self.base_bias is not None:
            y = y + self.base_bias.to(y.dtype)
        return y

    def extra_repr(self) -> str:
        c = self.config
        return (f"in_features={self.in_features}, out_features={self.out_features}, rank={c.rank}, "
                f"scaling={c.scaling}, dropout_p={c.dropout_p}")


class FusedMultiLoRA(nn.Module):
    """Several adapters sharing one frozen base linear; each microbatch row segment is
    routed to its adapter (rank, scaling, dropout) inside the same fused launches."""

    def __init__(
        self,
        base: nn.Linear | torch.Tensor,
        adapters: Sequence[AdapterConfig],
        *,
        init: str = "peft",
        dtype: torch.dtype = torch.float32,
        track_slot_grads: bool = False,
        generator: torch.Generator | None = None,
        capturable: bool = False,
        dropout_rng: str | None = None,
    ):
        super().__init__()
        if not adapters:
            raise ValidationError("FusedMultiLoRA needs at least one adapter")
        w, bias = _frozen_base(base)
        w.requires_grad_(False)
        self.base = base if isinstance(base, nn.Linear) else None
        self.register_buffer("weight", w, persistent=False) if self.base is None else None
        self.out_features, self.in_features = w.shape
        _init_capturable(self, capturable, w.device, dropout_rng)
        self.adapters = list(adapters)
        dev = w.device
        self.lora_A = nn.ModuleList(
            nn.Linear(self.in_features, a.rank, bias=False, device=dev, dtype=dtype) for a in self.adapters)
        self.lora_B = nn.ModuleList(
            nn.Linear(a.rank, self.out_features, bias=False, device=dev, dtype=dtype) for a in self.adapters)
        for la, lb in zip(self.lora_A, self.lora_B):
            _init_lora(la, lb, init, generator)
        self._offset = 0
        # bf16 operands: a version-keyed cache (eager), or persistent copies a CUDA graph can
        # read at fixed addresses, refreshed after every optimizer step (capturable)
        self._operands = ShadowOperands() if capturable else OperandCache()
        self.track_slot_grads = track_slot_grads
        # (adapter slot, global batch) -> [dA (r x k) fp32, dB (n x r) fp32]
        self.slot_grads: dict[tuple[int, int], list[torch.Tensor]] = {}

    @property
    def base_weight(self) -> torch.Tensor:
        return self.base.weight if self.base is not None else self.weight

    def next_offset(self) -> int:
        off = self._offset
        self._offset += 1
        return off

    def dropout_state(self) -> dict:
        return _dropout_state(self)

    def load_dropout_state(self, state: dict) -> None:
        _load_dropout_state(self, state)

    def invalidate_operands(self) -> None:
        """Drop the cached bf16 operands (after changing lora_A/lora_B outside an optimizer step)."""
        self._operands.clear()

    def _sink(self, layout, da: torch.Tensor, db: torch.Tensor) -> None:
        for adapter, batch, c0, r in layout.segment_grad_slices():
            ga, gb = da[c0:c0 + r], db[:, c0:c0 + r]
            slot = self.slot_grads.get((adapter, batch))
            if slot is None:
                self.slot_grads[(adapter, batch)] = [ga.clone(), gb.clone()]
            else:
                slot[0].add_(ga)
                slot[1].add_(gb)

    def forward(self, x: torch.Tensor, segments: Sequence[Segment],
                keep_mask: torch.Tensor | None = None) -> torch.Tensor:
        has_dropout = keep_mask is None and any(
            self.adapters[s_.adapter].dropout_p > 0 for s_ in segments)
        off, off_dev = _step_offsets(self, self.base_weight.device, has_dropout)
        y = fused_multi_lora(
            x,
            self.base_weight,
            [la.weight for la in self.lora_A],
            [lb.weight for lb in self.lora_B],
            self.adapters,
            segments,
            offset=off,
            keep_mask=keep_mask,
            training=self.training,
            grad_sink=self._sink if self.track_slot_grads else None,
            offset_dev=off_dev,
            operand_cache=self._operands,
        )
        if self.base is not None and self.base.bias is not None:
            y = y + self.base.bias.to(y.dtype)
        return y


class FusedLoRAGroup(nn.Module):
    """Several LoRA linears that read the same input — q/k/v of an attention block, gate/up
    of a SwiGLU MLP — as one module (shared-input fusion).

    ``projections`` maps names (e.g. "q_proj") to frozen bases (nn.Linear or weight); every
    projection is a :class:`FusedLoRA` child with its own adapter (PEFT names
    ``<name>.lora_A.weight`` / ``<name>.lora_B.weight``), seed and dropout mask, so
    ``group.q_proj(x)`` alone still works. ``forward(x)`` returns the projections' outputs in
    order. What the group adds: one Philox offset per call (one offset draw instead of one
    per projection), and backward sums the input gradient Σ_j dX_j inside the ⑤ GEMM
    epilogues (lf_grad_input_accum) instead of the per-projection elementwise adds autograd
    would run for an input read several times.
    """

    def __init__(
        self,
        projections: "dict[str, nn.Linear | torch.Tensor]",
        rank: int | Sequence[int],
        scaling: float | Sequence[float] | None = None,
        dropout_p: float | Sequence[float] = 0.0,
        *,
        alpha: float | None = None,
        seeds: Sequence[int] | None = None,
        init: str = "peft",
        dtype: torch.dtype = torch.float32,
        generator: torch.Generator | None = None,
        capturable: bool = False,
        dropout_rng: str | None = None,
    ):
        super().__init__()
        names = list(projections)
        if not names:
            raise ValidationError("FusedLoRAGroup needs at least one projection")
        J = len(names)

        def per(v, what):
            vs = list(v) if isinstance(v, (list, tuple)) else [v] * J
            if len(vs) != J:
                raise ValidationError(f"{what}: one value per projection ({J}), got {len(vs)}")
            return vs

        ranks, scalings, ps = per(rank, "rank"), per(scaling, "scaling"), per(dropout_p, "dropout_p")
        seeds = per(list(seeds) if seeds is not None else list(range(J)), "seeds")
        layers = {}
        for j, nm in enumerate(names):
            layers[nm] = FusedLoRA(projections[nm], ranks[j], scalings[j], ps[j], alpha=alpha, seed=seeds[j], init=init,
                                   dtype=dtype, generator=generator, capturable=capturable, dropout_rng=dropout_rng)
        self._adopt(layers, capturable, dropout_rng)

    @classmethod
    def from_layers(cls, layers: "dict[str, FusedLoRA]", capturable: bool | None = None,
                    dropout_rng: str | None = None) -> "FusedLoRAGroup":
        """Group existing FusedLoRA layers that read the same input (their parameters are
        shared, not copied)."""
        if not layers:
            raise ValidationError("FusedLoRAGroup needs at least one projection")
        first = next(iter(layers.values()))
        obj = cls.__new__(cls)
        nn.Module.__init__(obj)
        obj._adopt(dict(layers), first.capturable if capturable is None else capturable,
                   first.dropout_rng if dropout_rng is None else dropout_rng)
        return obj

    def _adopt(self, layers: "dict[str, FusedLoRA]", capturable: bool, dropout_rng: str) -> None:
        names = list(layers)
        self.names = names
        for nm in names:  # children under their own names: PEFT keys "<name>.lora_A.weight"
            if not nm.isidentifier():
                raise ValidationError(f"projection name {nm!r} must be a Python identifier")
            if not isinstance(layers[nm], FusedLoRA):
                raise ValidationError(f"projection {nm!r} must be a FusedLoRA layer")
            self.add_module(nm, layers[nm])
        ks = {self.proj(nm).in_features for nm in names}
        if len(ks) != 1:
            raise ValidationError(f"all projections of a group read the same input: in_features {sorted(ks)}")
        self.in_features = ks.pop()
        _init_capturable(self, capturable, self.proj(names[0]).base_weight.device, dropout_rng)
        self._offset = 0
        self._operands = ShadowOperands() if capturable else OperandCache(capacity=2 * len(names))
        cfgs = [self.proj(nm).config for nm in names]
        self._packed = pack_adapters(cfgs)
        self._has_dropout = any(c.dropout_p > 0 for c in cfgs)

    def proj(self, name: str) -> FusedLoRA:
        return self._modules[name]

    def next_offset(self) -> int:
        off = self._offset
        self._offset += 1
        return off

    def dropout_state(self) -> dict:
        return _dropout_state(self)

    def load_dropout_state(self, state: dict) -> None:
        _load_dropout_state(self, state)

    def invalidate_operands(self) -> None:
        self._operands.clear()

    def forward(self, x: torch.Tensor) -> tuple[torch.Tensor, ...]:
        from .functional import lora_group_fwd  # noqa: F401  (registers the operator)

        projs = [self._modules[nm] for nm in self.names]
        ws = [p.base_weight for p in projs]
        a = [p.lora_A.weight for p in projs]
        b = [p.lora_B.weight for p in projs]
        k = self.in_features
        x2, lead = _flatten_input(x, k)
        for j, p in enumerate(projs):
            _check_call(x2, ws[j], [a[j]], [b[j]], [self._packed[0][j]], k, p.out_features, None, None)
        if x2.shape[0] == 0:
            ys = [_EmptyBatchFn.apply(x2, w.shape[0], a_, b_) for w, a_, b_ in zip(ws, a, b)]
        else:
            off, off_dev = _step_offsets(self, x2.device, self._has_dropout)
            ys = torch.ops.lorafusion_b200.lora_group_fwd(
                x2, ws, a, b, [1] * len(ws), *self._packed, [], off, off_dev, self.training,
                _cache_handle(self._operands))[0]
        out = []
        for p, y in zip(projs, ys):
            y = y.reshape(lead + (p.out_features,))
            if p.base_bias is not None:
                y = y + p.base_bias.to(y.dtype)
            out.append(y)
        return tuple(out)


class FusedMultiLoRAGroup(nn.Module):
    """FusedMultiLoRA layers that read the same input (q/k/v, gate/up) as one module: every
    projection is a :class:`FusedMultiLoRA` child with its own adapter slots, seeds and
    masks, and all share the microbatch segment table. ``forward(x, segments)`` returns the
    projections' outputs in order; ②, ④ and ⑤ run as one launch each for the group where
    its shape allows (fused_multi_lora_group)."""

    def __init__(self, projections: "dict[str, nn.Linear | torch.Tensor]", adapters: Sequence[AdapterConfig], *,
                 seeds: Sequence[Sequence[int]] | None = None, init: str = "peft", dtype: torch.dtype = torch.float32,
                 generator: torch.Generator | None = None, capturable: bool = False, dropout_rng: str | None = None):
        super().__init__()
        names = list(projections)
        layers = {}
        for j, nm in enumerate(names):
            ads = list(adapters)
            if seeds is not None:
                ads = [AdapterConfig(a.rank, a.scaling, a.dropout_p, seed=sd) for a, sd in zip(ads, seeds[j])]
            layers[nm] = FusedMultiLoRA(projections[nm], ads, init=init, dtype=dtype, generator=generator,
                                        capturable=capturable, dropout_rng=dropout_rng)
        self._adopt(layers, capturable, dropout_rng)

    @classmethod
    def from_layers(cls, layers: "dict[str, FusedMultiLoRA]", capturable: bool | None = None,
                    dropout_rng: str | None = None) -> "FusedMultiLoRAGroup":
        """Group existing FusedMultiLoRA layers that read the same input (parameters shared)."""
        if not layers:
            raise ValidationError("FusedMultiLoRAGroup needs at least one projection")
        first = next(iter(layers.values()))
        obj = cls.__new__(cls)
        nn.Module.__init__(obj)
        obj._adopt(dict(layers), first.capturable if capturable is None else capturable,
                   first.dropout_rng if dropout_rng is None else dropout_rng)
        return obj

    def _adopt(self, layers: "dict[str, FusedMultiLoRA]", capturable: bool, dropout_rng: str) -> None:
        names = list(layers)
        if not names:
            raise ValidationError("FusedMultiLoRAGroup needs at least one projection")
        if len(names) > _lib.LF_MAX_GROUP:
            raise ValidationError(f"at most {_lib.LF_MAX_GROUP} projections per group, got {len(names)}")
        self.names = names
        for nm in names:
            if not nm.isidentifier():
                raise ValidationError(f"projection name {nm!r} must be a Python identifier")
            if not isinstance(layers[nm], FusedMultiLoRA):
                raise ValidationError(f"projection {nm!r} must be a FusedMultiLoRA layer")
            self.add_module(nm, layers[nm])
        ks = {self.proj(nm).in_features for nm in names}
        if len(ks) != 1:
            raise ValidationError(f"all projections of a group read the same input: in_features {sorted(ks)}")
        nslots = {len(self.proj(nm).adapters) for nm in names}
        if len(nslots) != 1:
            raise ValidationError("all projections of a group need the same adapter slots (one segment table)")
        self.in_features = ks.pop()
        _init_capturable(self, capturable, self.proj(names[0]).base_weight.device, dropout_rng)
        self._offset = 0
        self._operands = ShadowOperands() if capturable else OperandCache(capacity=2 * len(names))
        self._has_dropout = any(a.dropout_p > 0 for nm in names for a in self.proj(nm).adapters)

    def proj(self, name: str) -> "FusedMultiLoRA":
        return self._modules[name]

    def next_offset(self) -> int:
        off = self._offset
        self._offset += 1
        return off

    def dropout_state(self) -> dict:
        return _dropout_state(self)

    def load_dropout_state(self, state: dict) -> None:
        _load_dropout_state(self, state)

    def invalidate_operands(self) -> None:
        self._operands.clear()

    def forward(self, x: torch.Tensor, segments: Sequence[Segment]) -> tuple[torch.Tensor, ...]:
        from .functional import fused_multi_lora_group

        projs = [self._modules[nm] for nm in self.names]
        has_dropout = any(p.adapters[s_.adapter].dropout_p > 0 for p in projs for s_ in segments)
        off, off_dev = _step_offsets(self, projs[0].base_weight.device, has_dropout)
        ys = fused_multi_lora_group(
            x, [p.base_weight for p in projs], [[la.weight for la in p.lora_A] for p in projs],
            [[lb.weight for lb in p.lora_B] for p in projs], [p.adapters for p in projs], segments, offset=off,
            training=self.training, offset_dev=off_dev, operand_cache=self._operands)
        out = []
        for p, y in zip(projs, ys):
            if p.base is not None and p.base.bias is not None:
                y = y + p.base.bias.to(y.dtype)
            out.append(y)
        return tuple(out)
