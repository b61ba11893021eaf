"""Segment tables and per-call problem plans.

A microbatch is a sequence of *segments*: contiguous token rows that belong to one
(adapter, global batch) pair — lorasched's ``MicrobatchSegment`` (ls/packing.py:41-60),
whose rows are padded to the adapter's ``padding_multiple`` (ls/packing.py:30-32) and
ordered by (adapter, global batch) (ls/packing.py:251-258). Each segment gets its own
column block in a rank-concatenated low-rank dimension, so one fused launch handles
every adapter present: Ŝ and dŜ are (m x R) with each row non-zero only in its own
segment's block, A_cat (R x k) and B_cat (n x R) stack the segments' adapter weights.
A tile that straddles two segments (P = 64 < 128-row tiles) simply runs both blocks.

``LayerPlan`` owns everything one layer call needs on the device besides the tensors:
the C ``LfProblem`` (segment table by value), the 16-byte-per-128-row routing table
(ls/costmodel.py:23-26, 279-281) and a self-cleaning split-K workspace.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib
from .errors import ValidationError

RANK_ALIGN = 16  # one bf16 tcgen05 MMA-K step


def padded_rank(rank: int) -> int:
    """Adapter rank rounded up to the MMA-K granularity (16)."""
    return -(-int(rank) // RANK_ALIGN) * RANK_ALIGN


@dataclass(frozen=True)
class AdapterConfig:
    """Per-adapter hyper-parameters the kernels route on.

    Mirrors the fields of lorasched's AdapterSpec (ls/workload.py:25-48) that reach the
    FusedMultiLoRA lookup table: ``rank`` = lora_rank, ``scaling`` = Eq. 1
    alpha (PEFT convention alpha / r, see SPEC.md §1), ``dropout_p``, plus the dropout seed.
    """

    rank: int
    scaling: float = 2.0
    dropout_p: float = 0.0
    seed: int = 0

    def __post_init__(self):
        if int(self.rank) < 1:
            raise ValidationError(f"rank must be >= 1, got {self.rank}")
        if not math.isfinite(float(self.scaling)):
            raise ValidationError(f"scaling must be finite, got {self.scaling}")
        if not 0.0 <= float(self.dropout_p) < 1.0:
            raise ValidationError(f"dropout_p must be in [0, 1), got {self.dropout_p}")
        if not 0 <= int(self.seed) < 2**64:
            raise ValidationError(f"seed must be a 64-bit unsigned integer, got {self.seed}")

    @classmethod
    def from_adapter_spec(cls, spec, seed: int = 0) -> "AdapterConfig":
        """Build from a lorasched ``AdapterSpec``-like object (lora_rank, alpha, dropout_p)."""
        rank = int(spec.lora_rank)
        return cls(rank=rank, scaling=float(spec.alpha) / rank, dropout_p=float(spec.dropout_p), seed=seed)


@dataclass(frozen=True)
class Segment:
    """Token rows [row_start, row_end) of one (adapter slot, global batch) pair."""

    adapter: int
    row_start: int
    row_end: int
    batch: int = 0

    @property
    def rows(self) -> int:
        return self.row_end - self.row_start


def segments_from_lengths(adapters: Sequence[int], lengths: Sequence[int], batches: Sequence[int] | None = None,
                          start: int = 0) -> list[Segment]:
    """Consecutive segments of the given (padded) token lengths."""
    segs, row = [], start
    batches = list(batches) if batches is not None else [0] * len(adapters)
    for a, n, b in zip(adapters, lengths, batches):
        segs.append(Segment(int(a), row, row + int(n), int(b)))
        row += int(n)
    return segs


def split_segments(adapters: Sequence[AdapterConfig], segments: Sequence[Segment], m: int,
                   max_rank_total: int | None = None, max_segments: int | None = None,
                   share_blocks: bool = True) -> list[tuple[int, int, list]]:
    """Cut a microbatch whose segments exceed one launch's limits (rank-concat width R ≤
    LF_MAX_RANK_TOTAL, ≤ LF_MAX_SEGMENTS segments) into consecutive row ranges that each fit:
    [(row_start, row_end, segments)]. R counts each distinct adapter's padded rank once when
    its segments share a column block (``share_blocks``, LayerPlan's default), else once per
    segment (per-(adapter, batch) gradient slots). The ranges tile [0, m); rows in no segment
    stay with the range before them. One range when everything fits."""
    max_rank_total = max_rank_total or _lib.LF_MAX_RANK_TOTAL
    max_segments = max_segments or _lib.LF_MAX_SEGMENTS
    groups, cur, ranks, width = [], [], set(), 0
    for s in sorted(segments, key=lambda s_: s_.row_start):
        r = padded_rank(adapters[s.adapter].rank)
        if r > max_rank_total:
            raise ValidationError(f"adapter {s.adapter}: rank {adapters[s.adapter].rank} exceeds {max_rank_total}")
        grow = 0 if (share_blocks and s.adapter in ranks) else r
        if cur and (width + grow > max_rank_total or len(cur) >= max_segments):
            groups.append(cur)
            cur, ranks, width, grow = [], set(), 0, r
        cur.append(s)
        ranks.add(s.adapter)
        width += grow
    if not groups:
        return [(0, m, list(cur))]
    groups.append(cur)
    bounds = [0] + [g[0].row_start for g in groups[1:]] + [m]
    return [(bounds[i], bounds[i + 1], g) for i, g in enumerate(groups)]


def rank_layout(adapter_ranks: Sequence[int], segments: Sequence[Segment],
                share_blocks: bool = True) -> tuple[list[int], list[int], int]:
    """Column blocks of the rank-concat dimension: (col_start per segment, padded rank per
    segment, total width R). One block per adapter present — segments of the same adapter
    (two global batches in one microbatch) share it, their rows being disjoint — or, with
    ``share_blocks=False``, one per segment so dA/dB split per (adapter, batch) slot."""
    padded = [padded_rank(adapter_ranks[s.adapter]) for s in segments]
    col_starts, c, first = [], 0, {}
    for s, r in zip(segments, padded):
        if share_blocks and s.adapter in first:
            col_starts.append(first[s.adapter])
            continue
        first[s.adapter] = c
        col_starts.append(c)
        c += r
    return col_starts, padded, c


def validate_segments(segments: Sequence[Segment], m: int, num_adapters: int,
                      max_segments: int | None = _lib.LF_MAX_SEGMENTS) -> None:
    """Segments must be sorted, disjoint, inside [0, m) and name a valid adapter slot; at
    most ``max_segments`` of them per launch (None: no cap — a whole microbatch that
    fused_multi_lora then splits into launches)."""
    if max_segments is not None and len(segments) > max_segments:
        raise ValidationError(f"at most {max_segments} segments per launch, got {len(segments)}")
    prev = 0
    for i, s in enumerate(segments):
        if not 0 <= s.adapter < num_adapters:
            raise ValidationError(f"segment {i}: adapter slot {s.adapter} out of range [0, {num_adapters})")
        if s.row_start < prev or s.row_end < s.row_start or s.row_end > m:
            raise ValidationError(
                f"segment {i}: rows [{s.row_start}, {s.row_end}) must be sorted, disjoint and inside [0, {m})"
            )
        prev = s.row_end


def routing_table(segments: Sequence[Segment], col_starts: Sequence[int], ranks: Sequence[int], m: int) -> list[tuple]:
    """Host restatement of the device routing table (used for the tile-level cost
    accounting; the kernels consume the table lf_build_routes writes)."""
    out = []
    for t in range(-(-m // _lib.ROUTE_TILE_ROWS)):
        r0, r1 = t * _lib.ROUTE_TILE_ROWS, min(m, (t + 1) * _lib.ROUTE_TILE_ROWS)
        hit = [i for i, s in enumerate(segments) if s.row_start < s.row_end and s.row_start < r1 and s.row_end > r0]
        if not hit:
            out.append((0, -1, 0, 0))
        else:
            lo, hi = hit[0], hit[-1]
            out.append((lo, hi, min(col_starts[i] for i in hit), max(col_starts[i] + ranks[i] for i in hit)))
    return out


_WORKSPACES: dict[tuple[int, int], torch.Tensor] = {}
_ROUTES: dict[tuple, torch.Tensor] = {}
_ROUTES_MAX = 256


def workspace(device: torch.device, stream: "torch.cuda.Stream | int", nbytes: int) -> torch.Tensor:
    """Zero-initialised scratch owned per (device, stream). Kernels return it to zero."""
    sid = stream if isinstance(stream, int) else stream.cuda_stream
    key = (device.index if device.index is not None else torch.cuda.current_device(), sid)
    buf = _WORKSPACES.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.zeros(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)
        _WORKSPACES[key] = buf
    return buf


class LayerPlan:
    """Device-side plan of one fused LoRA layer call (forward and its backward)."""

    def __init__(
        self,
        m: int,
        k: int,
        n: int,
        adapters: Sequence[AdapterConfig],
        segments: Sequence[Segment],
        *,
        offset: int = 0,
        training: bool = True,
        keep_mask: torch.Tensor | None = None,
        device: torch.device | None = None,
        share_blocks: bool = True,
        offset_dev: torch.Tensor | None = None,
        row_base: int = 0,
    ):
        self.m, self.k, self.n = int(m), int(k), int(n)
        self.adapters = list(adapters)
        self.segments = list(segments)
        self.offset = int(offset)
        self.training = bool(training)
        validate_segments(self.segments, self.m, len(self.adapters))
        self.share_blocks = bool(share_blocks)
        self.col_starts, self.ranks, self.rank_total = rank_layout(
            [a.rank for a in self.adapters], self.segments, self.share_blocks)
        if self.rank_total > _lib.LF_MAX_RANK_TOTAL:
            raise ValidationError(
                f"sum of padded segment ranks {self.rank_total} exceeds {_lib.LF_MAX_RANK_TOTAL}; "
                "split the microbatch"
            )
        self.keep_mask = keep_mask
        if keep_mask is not None:
            if keep_mask.dtype != torch.uint8 or tuple(keep_mask.shape) != (self.m, self.k):
                raise ValidationError(f"keep_mask must be uint8 of shape ({self.m}, {self.k})")
            if not keep_mask.is_contiguous():
                raise ValidationError("keep_mask must be contiguous")
        self.device = device
        self.problem = _lib.LfProblem()
        p = self.problem
        p.m, p.k, p.n = self.m, self.k, self.n
        p.rank_total = self.rank_total
        p.num_segments = len(self.segments)
        for i, (s, c0, r) in enumerate(zip(self.segments, self.col_starts, self.ranks)):
            a = self.adapters[s.adapter]
            d = p.segments[i]
            d.row_start, d.row_end = s.row_start, s.row_end
            d.col_start, d.rank = c0, r
            d.scaling = float(a.scaling)
            d.dropout_p = float(a.dropout_p) if self.training else 0.0
            d.seed = int(a.seed) & (2**64 - 1)
            d.offset = self.offset & (2**64 - 1)
        p.keep_mask = keep_mask.data_ptr() if (keep_mask is not None and self.training) else None
        # microbatch row of this call's row 0 (Philox counters use absolute rows, SPEC.md §3)
        self.row_base = int(row_base)
        p.row_base = self.row_base
        # device-resident step counter added to the Philox offsets when the kernels run
        # (CUDA-graph replays then draw fresh masks); SPEC.md §3
        self.offset_dev = offset_dev
        if offset_dev is not None:
            if offset_dev.dtype != torch.int64 or offset_dev.numel() != 1 or not offset_dev.is_cuda:
                raise ValidationError("offset_dev must be a one-element int64 CUDA tensor")
            p.offset_dev = offset_dev.data_ptr()
        self.routes: torch.Tensor | None = None
        self._ws: torch.Tensor | None = None
        # ① writes the Philox keep mask bit-packed (m x k/8 bytes); ④/⑤ read it back
        self.needs_keep_bits = (self.training and keep_mask is None and
                                any(p.segments[i].dropout_p > 0 for i in range(p.num_segments)))
        self.keep_bits: torch.Tensor | None = None
        # optional bf16 copies of the adapter weights (lora_A list, lora_B list) kept by a
        # module in step with its fp32 master parameters; None = cast on every call
        self.weights_bf16: tuple | None = None
        # optional functional.OperandCache of the calling module (A_cat / B_cat reuse)
        self.operand_cache = None

    # -- derived ------------------------------------------------------------------
    @property
    def has_lora(self) -> bool:
        return len(self.segments) > 0

    @property
    def num_tiles(self) -> int:
        return -(-self.m // _lib.ROUTE_TILE_ROWS)

    def host_routes(self) -> list[tuple]:
        return routing_table(self.segments, self.col_starts, self.ranks, self.m)

    # -- device ---------------------------------------------------------------------
    def bind(self, device: torch.device, stream: torch.cuda.Stream | None = None,
             keep_bits: torch.Tensor | None = None) -> "LayerPlan":
        """Build the routing table and attach the workspace on ``device``/``stream``; the
        packed keep mask is ``keep_bits`` (the forward's, for the backward) or a new buffer."""
        self.device = device
        lib = _lib.load()
        dev_index = device.index if device.index is not None else torch._C._cuda_getDevice()
        sid = stream.cuda_stream if stream is not None else torch._C._cuda_getCurrentRawStream(dev_index)
        # the routing table depends only on the segment table: built once per (device,
        # stream, m, segments) and reused by every later call with the same microbatch layout
        key = (dev_index, sid, self.m,
               tuple((s.row_start, s.row_end) for s in self.segments), tuple(self.col_starts), tuple(self.ranks))
        cached = _ROUTES.get(key)
        fresh = cached is None
        if fresh:
            if len(_ROUTES) >= _ROUTES_MAX:
                _ROUTES.pop(next(iter(_ROUTES)))
            cached = torch.empty((max(self.num_tiles, 1), 4), dtype=torch.int32, device=device)
            _ROUTES[key] = cached
        self.routes = cached
        nbytes = _lib.workspace_bytes(self.m, self.rank_total)
        self._ws = workspace(device, sid, nbytes)
        self.problem.routes = self.routes.data_ptr()
        self.problem.workspace = self._ws.data_ptr()
        self.problem.workspace_bytes = self._ws.numel()
        if self.needs_keep_bits:
            if keep_bits is None or keep_bits.numel() == 0:
                keep_bits = torch.empty((self.m, self.k // 8), dtype=torch.uint8, device=device)
            self.keep_bits = keep_bits
            self.problem.keep_bits = self.keep_bits.data_ptr()
        if self.has_lora and fresh:
            from .functional import _call

            _call("build_routes", lib.lf_build_routes, ctypes.byref(self.problem), self.routes.data_ptr(),
                  ctypes.c_void_p(sid))
        return self

    def column_blocks(self) -> list[tuple[int, int, int]]:
        """(adapter, col_start, padded rank) of every distinct column block, in column order."""
        seen, out = set(), []
        for s, c0, r in zip(self.segments, self.col_starts, self.ranks):
            if c0 not in seen:
                seen.add(c0)
                out.append((s.adapter, c0, r))
        return sorted(out, key=lambda b: b[1])

    def gather_a(self, lora_a: Sequence[torch.Tensor]) -> torch.Tensor:
        """A_cat (R x k, bf16): each column block's adapter lora_A.weight, zero-padded to it."""
        blocks = []
        for adapter, _c0, r in self.column_blocks():
            a = lora_a[adapter].to(torch.bfloat16)
            if a.shape[0] != r:
                a = torch.nn.functional.pad(a, (0, 0, 0, r - a.shape[0]))
            blocks.append(a)
        return torch.cat(blocks, 0).contiguous() if len(blocks) > 1 else blocks[0].contiguous()

    def gather_b(self, lora_b: Sequence[torch.Tensor]) -> torch.Tensor:
        """B_cat (n x R, bf16): each column block's adapter lora_B.weight, zero-padded to it."""
        blocks = []
        for adapter, _c0, r in self.column_blocks():
            b = lora_b[adapter].to(torch.bfloat16)
            if b.shape[1] != r:
                b = torch.nn.functional.pad(b, (0, r - b.shape[1]))
            blocks.append(b)
        return torch.cat(blocks, 1).contiguous() if len(blocks) > 1 else blocks[0].contiguous()

    def adapter_grad_slices(self) -> list[tuple[int, int, int]]:
        """(adapter, col_start, rank) of every distinct column block: summing these into the
        adapter's dA/dB covers each block exactly once."""
        seen, out = set(), []
        for s, c0 in zip(self.segments, self.col_starts):
            if (s.adapter, c0) in seen:
                continue
            seen.add((s.adapter, c0))
            out.append((s.adapter, c0, self.adapters[s.adapter].rank))
        return out

    def segment_grad_slices(self) -> list[tuple[int, int, int, int]]:
        """(adapter, batch, col_start, rank) for routing dA/dB columns to (adapter, batch) slots
        (distinct per segment only when the plan was built with share_blocks=False)."""
        return [(s.adapter, s.batch, c0, self.adapters[s.adapter].rank)
                for s, c0 in zip(self.segments, self.col_starts)]
