"""LLaMa-style decoder stack whose seven linears per layer are FusedMultiLoRA layers.

This is the *caller* of the hot path for BASELINE.json configs[4] (C5: "LLaMa-3.1-8B 4
concurrent LoRA jobs, full decoder fwd+bwd step, bin-packed microbatches ... with dA/dB
allreduce"). The reference has no model code at all
(its runner replays a schedule, ls/runner.py); the paper's training system runs the
fused layers inside Megatron-LM. Here a microbatch is exactly what the
reference planner packs (ls/packing.py:41-98, serialised by ls/schedule.py:441-490 and
read by :mod:`.schedule`): segments of (adapter, global batch) rows, each a run of packed
samples padded to the adapter's multiple. Everything except the LoRA linears — token
embedding, RMSNorm, RoPE, causal varlen attention (flash-attn, per packed sample, so
samples and pad rows never attend to each other), SwiGLU, LM head and the loss — is stock
torch / library code and frozen: only the adapters train (W frozen).

``LoRADecoder(..., fused=False)`` builds the identical model with the unfused PEFT-style
torch projections (:func:`.baseline.unfused_multi_lora`) — the end-to-end baseline.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import Sequence

import torch
import torch.nn.functional as F
from torch import nn

from .baseline import unfused_multi_lora
from .errors import ValidationError
from .functional import refresh_stale_operand_shadows
from .modules import FusedMultiLoRA, FusedMultiLoRAGroup
from .plan import AdapterConfig, Segment

PROJECTIONS = ("q", "k", "v", "o", "gate", "up", "down")


@dataclass(frozen=True)
class DecoderShape:
    hidden: int = 4096
    heads: int = 32
    kv_heads: int = 8
    ffn: int = 14336
    layers: int = 32
    vocab: int = 128256
    rope_theta: float = 500000.0
    eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.hidden // self.heads

    def proj_shapes(self) -> dict[str, tuple[int, int]]:
        """(in_features k, out_features n) of every LoRA linear of one layer."""
        h, kv, f = self.hidden, self.kv_heads * self.head_dim, self.ffn
        return {"q": (h, h), "k": (h, kv), "v": (h, kv), "o": (h, h), "gate": (h, f), "up": (h, f), "down": (f, h)}

    def linear_flops(self, rows: int, rank_rows: Sequence[tuple[int, int]] = ()) -> float:
        """fwd+bwd FLOPs of the LoRA linears of the stack for ``rows`` packed rows:
        4kn per row (fwd + dgrad, W frozen) plus 6r(k+n) per (rank, rows) LoRA segment."""
        tot = 0.0
        for k, n in self.proj_shapes().values():
            tot += 4.0 * rows * k * n + sum(6.0 * L * r * (k + n) for r, L in rank_rows)
        return self.layers * tot


LLAMA31_8B = DecoderShape()


@dataclass
class PackedMicrobatch:
    """Device tensors of one packed microbatch (rows = Σ segment padded rows)."""

    tokens: torch.Tensor  # (m,) int64
    labels: torch.Tensor  # (m,) int64, -100 = no loss (pad rows, last token of a sample)
    positions: torch.Tensor  # (m,) int64, restart at 0 for every packed sequence
    cu_seqlens: torch.Tensor  # (nseq+1,) int32
    max_seqlen: int
    segments: list[Segment]
    raw_tokens: int

    @property
    def rows(self) -> int:
        return int(self.tokens.shape[0])


def pack_microbatch(mb, vocab: int, device, generator: torch.Generator | None = None) -> PackedMicrobatch:
    """Device tensors for a :class:`.schedule.MicrobatchPlan`: synthetic token ids (no
    dataset), positions restarting per packed sequence, next-token labels with no loss
    across a sequence boundary or on segment padding (pad rows carry token 0)."""
    seqs = [int(L) for L in mb.sequences]
    if not seqs or sum(seqs) != mb.rows or len(mb.segment_raw) != len(mb.segments):
        raise ValidationError("microbatch lacks its packed sequences (ingest it with schedule.microbatches_from_doc)")
    m = mb.rows
    cu = [0]
    for L in seqs:
        cu.append(cu[-1] + L)
    positions = torch.cat([torch.arange(L, dtype=torch.int64) for L in seqs])
    is_pad = torch.zeros(m, dtype=torch.bool)
    for seg, raw in zip(mb.segments, mb.segment_raw):
        is_pad[seg.row_start + int(raw):seg.row_end] = True
    tokens = torch.randint(0, vocab, (m,), generator=generator, dtype=torch.int64)
    tokens[is_pad] = 0
    labels = torch.roll(tokens, -1)
    labels[torch.tensor(cu[1:]) - 1] = -100  # no prediction across a sequence boundary
    labels[is_pad] = -100
    return PackedMicrobatch(tokens.to(device), labels.to(device), positions.to(device),
                            torch.tensor(cu, dtype=torch.int32, device=device), max(seqs),
                            list(mb.segments), int(mb.raw_tokens))


class RMSNorm(nn.Module):
    def __init__(self, dim: int, eps: float, device=None, dtype=torch.bfloat16):
        super().__init__()
        self.weight = nn.Parameter(torch.ones(dim, dtype=dtype, device=device), requires_grad=False)
        self.eps = eps

    def forward(self, x):
        return F.rms_norm(x, (x.shape[-1],), self.weight, self.eps)


class Rotary:
    """LLaMa RoPE tables indexed by per-row positions (positions restart per sample)."""

    def __init__(self, head_dim: int, theta: float, max_pos: int, device, dtype=torch.bfloat16):
        inv = 1.0 / (theta ** (torch.arange(0, head_dim, 2, device=device, dtype=torch.float32) / head_dim))
        t = torch.arange(max_pos, device=device, dtype=torch.float32)
        freqs = torch.outer(t, inv)
        self.cos = torch.cat([freqs.cos(), freqs.cos()], dim=-1).to(dtype)
        self.sin = torch.cat([freqs.sin(), freqs.sin()], dim=-1).to(dtype)

    def tables(self, positions: torch.Tensor):
        return self.cos[positions].unsqueeze(1), self.sin[positions].unsqueeze(1)


def _rotate_half(x):
    x1, x2 = x.chunk(2, dim=-1)
    return torch.cat((-x2, x1), dim=-1)


def apply_rope(q, k, cos, sin):
    return q * cos + _rotate_half(q) * sin, k * cos + _rotate_half(k) * sin


class TorchMultiLoRA(nn.Module):
    """The unfused baseline projection: frozen W plus per-adapter bf16 A/B driven by the
    per-segment torch loop (cuBLAS + elementwise), same parameters as FusedMultiLoRA."""

    def __init__(self, weight: torch.Tensor, adapters: Sequence[AdapterConfig], generator=None):
        super().__init__()
        dtype = weight.dtype
        self.register_buffer("weight", weight, persistent=False)
        self.adapters = list(adapters)
        n, k = weight.shape
        dev = weight.device
        self.lora_A = nn.ParameterList()
        self.lora_B = nn.ParameterList()
        for a in self.adapters:
            A = torch.empty(a.rank, k, device=dev).uniform_(-1 / math.sqrt(k), 1 / math.sqrt(k), generator=generator)
            B = torch.empty(n, a.rank, device=dev).normal_(0, 1 / math.sqrt(a.rank), generator=generator)
            self.lora_A.append(nn.Parameter(A.to(dtype)))
            self.lora_B.append(nn.Parameter(B.to(dtype)))

    def forward(self, x, segments):
        return unfused_multi_lora(x, self.weight, list(self.lora_A), list(self.lora_B), self.adapters, segments,
                                  training=self.training)


def varlen_attention_sdpa(q, k, v, cu_seqlens, scale=None):
    """Causal attention per packed sequence with torch SDPA (any dtype; the fp32 reference
    path of the tests), GQA by repeating k/v heads."""
    rep = q.shape[1] // k.shape[1]
    out = torch.empty_like(q)
    cu = cu_seqlens.tolist()
    for a, b in zip(cu[:-1], cu[1:]):
        qs = q[a:b].transpose(0, 1)
        ks = k[a:b].repeat_interleave(rep, dim=1).transpose(0, 1)
        vs = v[a:b].repeat_interleave(rep, dim=1).transpose(0, 1)
        out[a:b] = F.scaled_dot_product_attention(qs, ks, vs, is_causal=True, scale=scale).transpose(0, 1)
    return out


class DecoderLayer(nn.Module):
    def __init__(self, shape: DecoderShape, adapters: Sequence[AdapterConfig], layer_idx: int, fused: bool,
                 device, generator=None, dtype=torch.bfloat16, attention: str = "flash", capturable: bool = False):
        super().__init__()
        if fused and dtype != torch.bfloat16:
            raise ValidationError("the fused layers compute in bf16")
        self.shape = shape
        self.attention = attention
        self.ln1 = RMSNorm(shape.hidden, shape.eps, device, dtype)
        self.ln2 = RMSNorm(shape.hidden, shape.eps, device, dtype)
        self.proj = nn.ModuleDict()
        for i, (name, (k, n)) in enumerate(shape.proj_shapes().items()):
            w = (torch.randn(n, k, device=device, generator=generator) / math.sqrt(k)).to(dtype)
            # distinct dropout streams per (layer, projection, adapter)
            ads = [AdapterConfig(a.rank, a.scaling, a.dropout_p, seed=(a.seed * 1000003 + layer_idx * 7 + i) % 2**63)
                   for a in adapters]
            if fused:
                self.proj[name] = FusedMultiLoRA(w, ads, init="gaussian", generator=generator, capturable=capturable)
            else:
                self.proj[name] = TorchMultiLoRA(w, ads, generator=generator)
        # projections that read the same input run as shared-input groups (②/④/⑤ one launch
        # each); kept outside the module registry so parameter names and state dicts stay the
        # per-projection ones
        self._groups = None
        if fused and os.environ.get("LF_DECODER_GROUPS", "1") != "0":  # =0: per-projection calls (A/B)
            self._groups = (FusedMultiLoRAGroup.from_layers({nm: self.proj[nm] for nm in ("q", "k", "v")}),
                            FusedMultiLoRAGroup.from_layers({nm: self.proj[nm] for nm in ("gate", "up")}))

    def forward(self, h, mb: PackedMicrobatch, rope: Rotary):
        s = self.shape
        m, segs = h.shape[0], mb.segments
        x = self.ln1(h)
        if self._groups is not None:
            for grp in self._groups:  # not registered submodules: follow train() / eval() here
                grp.training = self.training
            q, k, v = self._groups[0](x, segs)
        else:
            q, k, v = (self.proj[nm](x, segs) for nm in ("q", "k", "v"))
        q = q.view(m, s.heads, s.head_dim)
        k = k.view(m, s.kv_heads, s.head_dim)
        v = v.view(m, s.kv_heads, s.head_dim)
        cos, sin = rope.tables(mb.positions)
        q, k = apply_rope(q, k, cos, sin)
        if self.attention == "flash":
            from flash_attn import flash_attn_varlen_func

            o = flash_attn_varlen_func(q, k, v, mb.cu_seqlens, mb.cu_seqlens, mb.max_seqlen, mb.max_seqlen,
                                       causal=True)
        else:
            o = varlen_attention_sdpa(q, k, v, mb.cu_seqlens)
        h = h + self.proj["o"](o.reshape(m, s.hidden), segs)
        x = self.ln2(h)
        if self._groups is not None:
            g, u = self._groups[1](x, segs)
        else:
            g, u = self.proj["gate"](x, segs), self.proj["up"](x, segs)
        return h + self.proj["down"](F.silu(g) * u, segs)


class LoRADecoder(nn.Module):
    """Embedding -> ``layers`` decoder layers -> RMSNorm -> LM head -> token cross-entropy;
    every base weight frozen, 7 multi-adapter LoRA linears per layer."""

    def __init__(self, shape: DecoderShape, adapters: Sequence[AdapterConfig], *, fused: bool = True, device=None,
                 generator=None, max_pos: int = 8192, dtype=torch.bfloat16, attention: str = "flash",
                 capturable: bool = False):
        super().__init__()
        self.shape = shape
        self.adapters = list(adapters)
        self.embed = nn.Embedding(shape.vocab, shape.hidden, device=device, dtype=dtype)
        self.embed.weight.requires_grad_(False)
        with torch.no_grad():
            self.embed.weight.normal_(0, 1.0, generator=generator)
        self.layers = nn.ModuleList(DecoderLayer(shape, adapters, i, fused, device, generator, dtype, attention,
                                                 capturable) for i in range(shape.layers))
        self.norm = RMSNorm(shape.hidden, shape.eps, device, dtype)
        self.head = (torch.randn(shape.vocab, shape.hidden, device=device, generator=generator) /
                     math.sqrt(shape.hidden)).to(dtype)
        self.rope = Rotary(shape.head_dim, shape.rope_theta, max_pos, device, dtype)

    def adapter_parameters(self) -> list[nn.Parameter]:
        return [p for p in self.parameters() if p.requires_grad]

    def forward(self, mb: PackedMicrobatch) -> torch.Tensor:
        if mb.max_seqlen > self.rope.cos.shape[0]:
            raise ValidationError(f"sequence of {mb.max_seqlen} rows exceeds the RoPE table ({self.rope.cos.shape[0]})")
        h = self.embed(mb.tokens)
        for layer in self.layers:
            h = layer(h, mb, self.rope)
        h = self.norm(h)
        logits = F.linear(h, self.head)
        return F.cross_entropy(logits.float(), mb.labels, ignore_index=-100, reduction="sum")


def train_step(model: LoRADecoder, microbatches: Sequence[PackedMicrobatch], reducer=None, optimizer=None):
    """One optimizer step of data-parallel multi-LoRA fine-tuning on this rank: fwd+bwd of
    every assigned microbatch (adapter gradients accumulate), the SUM all-reduce of the fp32
    adapter gradients (:class:`.dp.AdapterGradReducer`; the only cross-rank exchange,
    SURVEY.md §8(e)), then the optimizer step. Returns the summed loss (device tensor)."""
    total = None
    overlap = reducer is not None and bool(getattr(reducer, "_hooks", None))
    for i, mb in enumerate(microbatches):
        loss = model(mb)
        if overlap and i == len(microbatches) - 1:
            reducer.arm()  # buckets all-reduce as the last backward finalizes them
        loss.backward()
        total = loss.detach() if total is None else total + loss.detach()
    if reducer is not None:
        if overlap:
            reducer.wait()
        else:
            reducer.reduce()
    if optimizer is not None:
        optimizer.step()
        optimizer.zero_grad(set_to_none=True)
    return total


class GraphedTrainStep:
    """A training step whose per-microbatch forward+backward passes replay as CUDA graphs.

    One graph per microbatch (its shape and segments are baked in), all drawing from one
    memory pool — they replay in capture order, so each reuses the activation memory the
    previous one released and the peak stays that of one microbatch. The first graph
    writes the adapter gradients, the others accumulate into the same tensors, so the
    optimizer (eager, after the replays) must not reset ``.grad`` to None. The gradient
    all-reduce (``reducer.reduce()``) and the optimizer step run eagerly after the replays.
    The fused layers must be ``capturable`` (device-side Philox counters)."""

    def __init__(self, model: LoRADecoder, microbatches: Sequence[PackedMicrobatch], reducer=None, optimizer=None,
                 warmup: int = 2):
        self.model, self.reducer, self.optimizer = model, reducer, optimizer
        params = model.adapter_parameters()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(max(1, warmup)):
                for mb in microbatches:
                    model(mb).backward()
        torch.cuda.current_stream().wait_stream(side)
        for p in params:
            p.grad = None
        pool = torch.cuda.graph_pool_handle()
        self.graphs, self.losses = [], []
        for mb in microbatches:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=pool):
                loss = model(mb)
                loss.backward()
            self.graphs.append(g)
            self.losses.append(loss.detach())

    def __call__(self):
        refresh_stale_operand_shadows()
        for g in self.graphs:
            g.replay()
        if self.reducer is not None:
            self.reducer.reduce()
        if self.optimizer is not None:
            self.optimizer.step()
        total = self.losses[0]
        for l in self.losses[1:]:
            total = total + l
        return total
