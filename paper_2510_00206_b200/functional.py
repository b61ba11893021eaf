"""Functional FusedLoRA / FusedMultiLoRA (forward + backward through the sm_100a kernels).

Forward:  ① lf_dropout_down_fwd   Ŝ = s·(M⊙X)·Aᵀ
                               ② lf_base_fwd           Y = X·Wᵀ + Ŝ·Bᵀ   (one write of Y)
Backward:  ③ lf_grad_up            dŜ = s·dY·B, dB += dYᵀ·Ŝ   (one read of dY)
                               ④ lf_grad_down          dA += dŜᵀ·(M⊙X)
                               ⑤ lf_grad_input         dX = dY·W + M⊙(dŜ·A)       (one write of dX)

The two passes are registered as torch operators (``torch.ops.lorafusion_b200.lora_fwd`` /
``lora_bwd``) with fake (meta) implementations and an autograd formula,
so a FusedLoRA layer traces under ``torch.compile(fullgraph=True)`` without graph breaks
and recomputes correctly under ``torch.utils.checkpoint`` (the packed keep mask and Ŝ are
ordinary saved tensors). The operators take plain tensors and scalars: the adapter table
(ranks, scalings, dropout p, seeds) and the segment table (adapter, row_start, row_end,
batch) as flat lists; the host plan (LfProblem, routing table, workspace) is rebuilt from
them inside each operator. The base weight is frozen (LoRA fine-tuning); there is no CPU
path — tensors must live on a B200 and the shared library must be built, otherwise the call
raises.
"""
from __future__ import annotations

import ctypes
import itertools
import weakref
from typing import Callable, Optional, Sequence

import torch
from torch.optim.optimizer import register_optimizer_step_post_hook

from . import _lib
from .errors import ValidationError
from .plan import AdapterConfig, LayerPlan, Segment, rank_layout, split_segments, validate_segments
from .plan import workspace as group_workspace

_BF16 = torch.bfloat16
_NS = "lorafusion_b200"


def _ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None and t.numel() > 0 else 0)


def _stream(device: torch.device | None = None) -> ctypes.c_void_p:
    """The current torch stream of ``device`` as a raw cudaStream_t (cheap: no Stream object)."""
    idx = device.index if device is not None and device.index is not None else torch._C._cuda_getDevice()
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(idx))


class LaunchStats:
    """Counts kernel launches and (optionally) times each launcher with CUDA events on the
    launching stream. Install with ``set_launch_stats``; used by bench.py."""

    def __init__(self, timed: bool = False, external: bool = False):
        self.timed = timed
        self.external = external  # events recorded inside a CUDA-graph capture (timing per replay)
        self.launches: dict[str, int] = {}
        self.events: dict[str, list] = {}

    def _event(self):
        if self.external:
            return torch.cuda.Event(enable_timing=True, external=True)
        return torch.cuda.Event(enable_timing=True)

    def begin(self, name: str):
        self.launches[name] = self.launches.get(name, 0) + 1
        if not self.timed:
            return None
        ev = self._event()
        ev.record()
        return ev

    def end(self, name: str, start) -> None:
        if start is None:
            return
        ev = self._event()
        ev.record()
        self.events.setdefault(name, []).append((start, ev))

    # device kernels each C entry point launches (③ adds its split-K finalize kernel)
    KERNELS_PER_CALL = {"grad_up": 2}

    def total_launches(self) -> int:
        return sum(n * self.KERNELS_PER_CALL.get(k, 1) for k, n in self.launches.items())

    def durations_ms(self) -> dict[str, list[float]]:
        torch.cuda.synchronize()
        return {k: [a.elapsed_time(b) for a, b in v] for k, v in self.events.items()}


_STATS: LaunchStats | None = None


def set_launch_stats(stats: LaunchStats | None) -> None:
    global _STATS
    _STATS = stats


def _call(name: str, fn, *args) -> None:
    st = _STATS
    tok = st.begin(name) if st is not None else None
    rc = fn(*args)
    if st is not None:
        st.end(name, tok)
    _lib.check(rc, name)


def _check_operand(t: torch.Tensor, name: str, shape: tuple | None = None) -> None:
    if not isinstance(t, torch.Tensor):
        raise ValidationError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValidationError(f"{name} must be a CUDA tensor on a B200 (no CPU fallback)")
    if t.dtype != _BF16:
        raise ValidationError(f"{name} must be bfloat16, got {t.dtype}")
    if not t.is_contiguous():
        raise ValidationError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValidationError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


# --------------------------------------------------------------------------------------
# bf16 rank-concat operand cache
# --------------------------------------------------------------------------------------
# Adapter weights change in place: through the optimizer (torch's fused AdamW/SGD kernels
# leave the parameters' version counters untouched), through ``p.data`` or through external
# updaters (apex, Megatron's main->model copy). Every optimizer step therefore bumps a
# global weight generation (torch's global optimizer step post-hook) that is part of the
# cache key, next to the parameters' pointers and versions; updates outside any
# torch.optim.Optimizer must call ``invalidate_operand_caches()``.
_GENERATION = [0]


def invalidate_operand_caches(*_args, **_kwargs) -> None:
    """Forget every cached bf16 A_cat/B_cat and refresh every persistent bf16 operand copy
    (call after updating adapter weights outside a torch.optim optimizer step, e.g. through
    ``p.data``). Runs automatically after every optimizer step."""
    _GENERATION[0] += 1
    for sh in list(_SHADOW_SETS):
        sh.refresh_all()


_SHADOW_SETS: "weakref.WeakSet" = weakref.WeakSet()
register_optimizer_step_post_hook(invalidate_operand_caches)


class ShadowOperands:
    """Persistent bf16 rank-concat operands (A_cat (R,k), B_cat (n,R)) for ``capturable``
    modules: a CUDA graph reads them at fixed addresses, so no cast, pad or concatenation
    runs inside the graph. Each entry covers one column-block layout — one adapter
    (FusedLoRA) or several (FusedMultiLoRA: every block is an adapter's lora_A/lora_B cast
    into its columns; padding columns stay zero). They are refreshed in place — all of them
    in one multi-tensor copy per device — after every optimizer step (the global post-hook
    above), and by a lookup that sees a parameter's in-place version change; an update
    through ``p.data`` needs ``invalidate_operand_caches()`` (or the module's
    ``invalidate_operands()``)."""

    def __init__(self, capacity: int = 64):
        self.capacity = capacity
        self._d: dict = {}
        _SHADOW_SETS.add(self)

    def lookup(self, a: torch.Tensor, b: torch.Tensor, R: int) -> tuple[torch.Tensor, torch.Tensor] | None:
        """One adapter: A (r,k) / B (n,r) into columns [0, r) of R."""
        return self.lookup_blocks([(a, b, 0)], R)

    def lookup_blocks(self, blocks, R: int) -> tuple[torch.Tensor, torch.Tensor] | None:
        """``blocks``: (lora_A weight, lora_B weight, first column) per column block; R the
        total (padded) column count. None when the module's entry cap is reached."""
        key = (R,) + tuple((a.data_ptr(), b.data_ptr(), c0) for a, b, c0 in blocks)
        ent = self._d.get(key)
        if ent is None:
            # entries are never dropped: a captured graph may read them. Past the cap (layouts
            # churning, parameters moved) or first seen inside a capture, the caller gathers
            # per call instead.
            if len(self._d) >= self.capacity or torch.cuda.is_current_stream_capturing():
                return None  # (inside a capture: a new copy would be valid only after a replay)
            a0, b0 = blocks[0][0], blocks[0][1]
            a_cat = torch.zeros((R, a0.shape[1]), dtype=_BF16, device=a0.device)
            b_cat = torch.zeros((b0.shape[0], R), dtype=_BF16, device=b0.device)
            # piece: [A_cat rows, B_cat columns, weakref A, weakref B, A version, B version]
            pieces = [[a_cat[c0:c0 + a.shape[0]], b_cat[:, c0:c0 + a.shape[0]], weakref.ref(a), weakref.ref(b), -1, -1]
                      for a, b, c0 in blocks]
            ent = self._d[key] = (a_cat, b_cat, pieces)
        if any(pc[4] != a._version or pc[5] != b._version for pc, (a, b, _c) in zip(ent[2], blocks)):
            self._copy(ent[2])
        return ent[0], ent[1]

    @staticmethod
    def _copy(pieces) -> None:
        by_dev: dict = {}
        for pc in pieces:
            a, b = pc[2](), pc[3]()
            if a is None or b is None:
                continue
            dst, src = by_dev.setdefault(a.device, ([], []))
            dst += [pc[0], pc[1]]
            src += [a.detach(), b.detach()]
            pc[4], pc[5] = a._version, b._version
        with torch.no_grad():
            for dst, src in by_dev.values():
                torch._foreach_copy_(dst, src)

    def _pieces(self) -> list:
        return [pc for ent in self._d.values() for pc in ent[2]]

    def refresh_all(self) -> None:
        self._copy(self._pieces())

    def clear(self) -> None:
        """Re-copy every persistent operand (the addresses a captured graph reads stay put)."""
        self.refresh_all()

    def stale(self) -> list:
        """Pieces whose parameters changed in place since their last copy (host check)."""
        out = []
        for pc in self._pieces():
            a, b = pc[2](), pc[3]()
            if a is not None and b is not None and (pc[4] != a._version or pc[5] != b._version):
                out.append(pc)
        return out


def refresh_stale_operand_shadows() -> None:
    """Re-copy the persistent bf16 operands whose fp32 parameters changed in place (version
    counter) since their last copy — a host-side check, one multi-tensor copy only when
    something changed. GraphedStep.replay() calls it before every replay."""
    pcs = [pc for sh in list(_SHADOW_SETS) for pc in sh.stale()]
    if pcs:
        ShadowOperands._copy(pcs)


class OperandCache:
    """bf16 rank-concat operands (A_cat, B_cat) of a module, keyed by the column-block
    layout, the weight generation and the adapter parameters' pointers and in-place
    versions: every layer call between two optimizer steps that sees the same adapters
    reuses them instead of re-casting, padding and concatenating (a dozen small launches
    of host work per call)."""

    def __init__(self, capacity: int = 8):
        self.capacity = capacity
        self._d: dict = {}

    def get(self, key):
        return self._d.get(key)

    def put(self, key, value) -> None:
        if len(self._d) >= self.capacity:
            self._d.pop(next(iter(self._d)))
        self._d[key] = value

    def clear(self) -> None:
        self._d.clear()


# operators take an integer handle for the calling module's operand cache
_CACHES: "weakref.WeakValueDictionary[int, OperandCache | ShadowOperands]" = weakref.WeakValueDictionary()
_ids = itertools.count(1)


def _cache_handle(cache: "OperandCache | ShadowOperands | None") -> int:
    if cache is None:
        return 0
    h = getattr(cache, "_handle", None)
    if h is None:
        h = next(_ids)
        cache._handle = h
        _CACHES[h] = cache
    return h


def _own(t: torch.Tensor | None, inputs: Sequence[torch.Tensor], empty_shape, like: torch.Tensor) -> torch.Tensor:
    """An operator output that never aliases an input (gather_* returns a bf16 adapter weight
    itself when no cast or padding is needed)."""
    if t is None:
        return like.new_empty(empty_shape)
    if any(t.data_ptr() == i.data_ptr() for i in inputs):
        return t.clone()
    return t


def _rank_concat_operands(plan: LayerPlan, a: Sequence[torch.Tensor], b: Sequence[torch.Tensor], cache_id: int):
    cache = _CACHES.get(cache_id) if cache_id else None
    if isinstance(cache, ShadowOperands):
        hit = cache.lookup_blocks([(a[ad], b[ad], c0) for ad, c0, _r in plan.column_blocks()], plan.rank_total)
        if hit is not None:
            return hit
        cache = None
    key = None
    if cache is not None:
        blocks = plan.column_blocks()
        used = sorted({ad for ad, _, _ in blocks})
        key = (_GENERATION[0], tuple((ad, r) for ad, _, r in blocks),
               tuple((p.data_ptr(), p._version) for ad in used for p in (a[ad], b[ad])))
        hit = cache.get(key)
        if hit is not None:
            return hit
    blocks = plan.column_blocks()
    if len(blocks) == 1 and blocks[0][2] == a[blocks[0][0]].shape[0]:
        # one adapter, rank a multiple of 16: both casts in one multi-tensor launch
        ad = blocks[0][0]
        a_cat = torch.empty(a[ad].shape, dtype=_BF16, device=a[ad].device)
        b_cat = torch.empty(b[ad].shape, dtype=_BF16, device=b[ad].device)
        torch._foreach_copy_([a_cat, b_cat], [a[ad].detach(), b[ad].detach()])
    else:
        a_cat, b_cat = plan.gather_a(a), plan.gather_b(b)
    if cache is not None:
        cache.put(key, (a_cat, b_cat))
    return a_cat, b_cat


def _group_operands(a: Sequence[torch.Tensor], b: Sequence[torch.Tensor], ranks) -> tuple[list, list] | None:
    """bf16 copies of every projection's A and B in one multi-tensor cast (ranks multiples of
    16, no padding needed), or None."""
    if any(_padr(r) != r for r in ranks):
        return None
    acs = [torch.empty(t.shape, dtype=_BF16, device=t.device) for t in a]
    bcs = [torch.empty(t.shape, dtype=_BF16, device=t.device) for t in b]
    torch._foreach_copy_(acs + bcs, [t.detach() for t in a] + [t.detach() for t in b])
    return acs, bcs


# --------------------------------------------------------------------------------------
# dB column blocks -> contiguous per-adapter gradients
# --------------------------------------------------------------------------------------
def _gather_db_blocks(flat: torch.Tensor, specs) -> list[torch.Tensor]:
    """Contiguous (n, r) fp32 gradients of the column blocks ``specs`` = ((offset, n, R, c0,
    r), ...) of n x R row-major matrices inside ``flat``. dB_cat[:, c0:c0 + r] is a strided
    view, which autograd would copy into a contiguous .grad with one elementwise launch per
    adapter and projection (28 per C3 step): blocks spanning their whole rows stay views,
    the others are copied out by one lf_copy_column_blocks launch per call."""
    res: list = [None] * len(specs)
    part = []
    for i, (off, n, R, c0, r) in enumerate(specs):
        if c0 == 0 and r == R:
            res[i] = flat[off:off + n * R].view(n, R)
        else:
            part.append(i)
    if not part:
        return res
    out = torch.empty(sum(specs[i][1] * specs[i][4] for i in part), dtype=flat.dtype, device=flat.device)
    lib = _lib.load()
    st = _stream(flat.device)
    base, esz = flat.data_ptr(), flat.element_size()
    pos = 0
    for c in range(0, len(part), _lib.LF_MAX_COPY_BLOCKS):
        chunk = part[c:c + _lib.LF_MAX_COPY_BLOCKS]
        nb = len(chunk)
        src, dst = (ctypes.c_void_p * nb)(), (ctypes.c_void_p * nb)()
        rows, ld, col, wid = ((ctypes.c_int32 * nb)() for _ in range(4))
        for t, i in enumerate(chunk):
            off, n, R, c0, r = specs[i]
            src[t], dst[t] = base + off * esz, out.data_ptr() + pos * esz
            rows[t], ld[t], col[t], wid[t] = n, R, c0, r
            res[i] = out[pos:pos + n * r].view(n, r)
            pos += n * r
        _call("copy_column_blocks", lib.lf_copy_column_blocks, nb, src, rows, ld, col, wid, dst, st)
    return res


# --------------------------------------------------------------------------------------
# packed call description (what the operators take instead of Python objects)
# --------------------------------------------------------------------------------------
def _u64_to_i64(v: int) -> int:
    v = int(v) & (2**64 - 1)
    return v - 2**64 if v >= 2**63 else v


def pack_adapters(adapters: Sequence[AdapterConfig]) -> tuple[list[int], list[float], list[float], list[int]]:
    return ([int(a.rank) for a in adapters], [float(a.scaling) for a in adapters],
            [float(a.dropout_p) for a in adapters], [_u64_to_i64(a.seed) for a in adapters])


def pack_segments(segments: Sequence[Segment]) -> list[int]:
    return [v for s in segments for v in (int(s.adapter), int(s.row_start), int(s.row_end), int(s.batch))]


_DESC_CACHE: dict = {}


def _unpack(ranks, scalings, ps, seeds, segs) -> tuple[list[AdapterConfig], list[Segment]]:
    key = (tuple(ranks), tuple(scalings), tuple(ps), tuple(seeds), tuple(segs))
    hit = _DESC_CACHE.get(key)
    if hit is None:
        if len(_DESC_CACHE) >= 512:
            _DESC_CACHE.pop(next(iter(_DESC_CACHE)))
        adapters = [AdapterConfig(rank=r, scaling=s, dropout_p=p, seed=int(sd) & (2**64 - 1))
                    for r, s, p, sd in zip(ranks, scalings, ps, seeds)]
        segments = [Segment(*segs[i:i + 4]) for i in range(0, len(segs), 4)]
        hit = _DESC_CACHE[key] = (adapters, segments)
    return hit


def _rank_total(ranks, segs, share_blocks) -> int:
    segments = [Segment(*segs[i:i + 4]) for i in range(0, len(segs), 4)]
    return rank_layout(ranks, segments, share_blocks)[2]


def _needs_bits(ps, segs, keep_mask, training) -> bool:
    return bool(training and keep_mask is None and any(ps[segs[i]] > 0 for i in range(0, len(segs), 4)))


def _plan(x_rows, k, n, ranks, scalings, ps, seeds, segs, offset, offset_dev, keep_mask, training,
          share_blocks, row_base) -> LayerPlan:
    adapters, segments = _unpack(ranks, scalings, ps, seeds, segs)
    return LayerPlan(x_rows, k, n, adapters, segments, offset=offset, training=training, keep_mask=keep_mask,
                     share_blocks=share_blocks, offset_dev=offset_dev, row_base=row_base)


# --------------------------------------------------------------------------------------
# torch operators
# --------------------------------------------------------------------------------------
@torch.library.custom_op(f"{_NS}::lora_fwd", mutates_args=(), device_types="cuda")
def lora_fwd(x: torch.Tensor, w: torch.Tensor, a: list[torch.Tensor], b: list[torch.Tensor], ranks: list[int],
             scalings: list[float], ps: list[float], seeds: list[int], segs: list[int], offset: int,
             offset_dev: Optional[torch.Tensor], keep_mask: Optional[torch.Tensor], training: bool,
             share_blocks: bool, row_base: int,
             cache_id: int) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    """① + ②: returns (Y (m,n) bf16, Ŝ (m,R) bf16, packed keep mask (m,k/8) u8 or empty,
    A_cat (R,k) bf16, B_cat (n,R) bf16) — the rank-concat operands are saved for the
    backward, so it never re-casts the adapter weights."""
    lib = _lib.load()
    m, k = x.shape
    n = w.shape[0]
    plan = _plan(m, k, n, ranks, scalings, ps, seeds, segs, offset, offset_dev, keep_mask, training,
                 share_blocks, row_base)
    plan.bind(x.device)
    pp = ctypes.byref(plan.problem)
    st = _stream(x.device)
    y = torch.empty((m, n), dtype=_BF16, device=x.device)
    s_hat = torch.empty((m, plan.rank_total), dtype=_BF16, device=x.device)
    a_cat = b_cat = None
    if plan.has_lora:
        a_cat, b_cat = _rank_concat_operands(plan, a, b, cache_id)
        _call("dropout_down_fwd", lib.lf_dropout_down_fwd, pp, _ptr(x), _ptr(a_cat), _ptr(s_hat), st)
    _call("base_fwd", lib.lf_base_fwd, pp, _ptr(x), _ptr(w), _ptr(s_hat), _ptr(b_cat), _ptr(y), st)
    bits = plan.keep_bits if plan.keep_bits is not None else torch.empty((0,), dtype=torch.uint8, device=x.device)
    a_cat, b_cat = _own(a_cat, a, (0, k), x), _own(b_cat, b, (n, 0), x)
    return y, s_hat, bits, a_cat, b_cat


@lora_fwd.register_fake
def _lora_fwd_fake(x, w, a, b, ranks, scalings, ps, seeds, segs, offset, offset_dev, keep_mask, training,
                   share_blocks, row_base, cache_id):
    m, k = x.shape
    R = _rank_total(ranks, segs, share_blocks)
    bits = (x.new_empty((m, k // 8), dtype=torch.uint8) if _needs_bits(ps, segs, keep_mask, training)
            else x.new_empty((0,), dtype=torch.uint8))
    n = w.shape[0]
    ops = (x.new_empty((R, k)), x.new_empty((n, R))) if segs else (x.new_empty((0, k)), x.new_empty((n, 0)))
    return x.new_empty((m, n)), x.new_empty((m, R)), bits, *ops


@torch.library.custom_op(f"{_NS}::lora_bwd", mutates_args=(), device_types="cuda")
def lora_bwd(dy: torch.Tensor, x: torch.Tensor, w: torch.Tensor, a_cat: torch.Tensor, b_cat: torch.Tensor,
             s_hat: torch.Tensor, keep_bits: torch.Tensor, ranks: list[int], scalings: list[float], ps: list[float],
             seeds: list[int], segs: list[int], offset: int, offset_dev: Optional[torch.Tensor],
             keep_mask: Optional[torch.Tensor], training: bool, share_blocks: bool, row_base: int, cache_id: int,
             need_dx: bool) -> tuple[torch.Tensor, torch.Tensor]:
    """③ + ④ + ⑤: returns (dX (m,k) bf16 or empty, [dA_cat (R,k) | dB_cat (n,R)] fp32 flat —
    one buffer, one zero-fill)."""
    lib = _lib.load()
    m, k = x.shape
    n = w.shape[0]
    plan = _plan(m, k, n, ranks, scalings, ps, seeds, segs, offset, offset_dev, keep_mask, training,
                 share_blocks, row_base)
    plan.bind(dy.device, keep_bits=keep_bits)
    pp = ctypes.byref(plan.problem)
    st = _stream(dy.device)
    R = plan.rank_total
    ds = None
    # one zero-fill for both fp32 accumulators
    acc = torch.zeros(R * k + n * R, dtype=torch.float32, device=dy.device)
    da = acc[:R * k].view(R, k)
    db = acc[R * k:].view(n, R)
    if plan.has_lora:
        ds = torch.empty((m, R), dtype=_BF16, device=dy.device)
        _call("grad_up", lib.lf_grad_up, pp, _ptr(dy), _ptr(b_cat), _ptr(s_hat), _ptr(ds), _ptr(db), st)
        _call("grad_down", lib.lf_grad_down, pp, _ptr(x), _ptr(ds), _ptr(da), st)
    if need_dx:
        dx = torch.empty((m, k), dtype=_BF16, device=dy.device)
        _call("grad_input", lib.lf_grad_input, pp, _ptr(dy), _ptr(w), _ptr(ds), _ptr(a_cat), _ptr(dx), st)
    else:
        dx = torch.empty((0,), dtype=_BF16, device=dy.device)
    return dx, acc


@lora_bwd.register_fake
def _lora_bwd_fake(dy, x, w, a_cat, b_cat, s_hat, keep_bits, ranks, scalings, ps, seeds, segs, offset, offset_dev,
                   keep_mask, training, share_blocks, row_base, cache_id, need_dx):
    m, k = x.shape
    R = _rank_total(ranks, segs, share_blocks)
    dx = x.new_empty((m, k)) if need_dx else x.new_empty((0,))
    return dx, x.new_empty((R * k + w.shape[0] * R,), dtype=torch.float32)


_PLAN_ARGS = ("ranks", "scalings", "ps", "seeds", "segs", "offset", "offset_dev", "keep_mask", "training",
              "share_blocks", "row_base", "cache_id")


def _setup_context(ctx, inputs, output, mark: bool = True):
    x, w, a, b, *rest = inputs
    y, s_hat, bits, a_cat, b_cat = output
    if mark:
        ctx.mark_non_differentiable(s_hat, bits, a_cat, b_cat)
    # no zero tensors for the outputs nothing differentiates (Ŝ, keep bits, operands)
    ctx.set_materialize_grads(False)
    args = dict(zip(_PLAN_ARGS, rest))
    # the gradient of a non-tensor argument is None, except that an empty list (no segments)
    # flattens like a list of tensors and must come back as []
    ctx.none_grads = tuple([] if isinstance(v, list) and not v else None for v in rest)
    ctx.n_adapters = len(a)
    ctx.param_dtypes = [p.dtype for p in a] + [p.dtype for p in b]
    opt = [args.pop("offset_dev"), args.pop("keep_mask")]
    ctx.has_opt = [t is not None for t in opt]
    ctx.args = args
    ctx.save_for_backward(x, w, s_hat, bits, a_cat, b_cat, *[t for t in opt if t is not None])


def _backward(ctx, dy, _ds=None, _dbits=None, _da=None, _db=None):
    na = ctx.n_adapters
    x, w, s_hat, bits, a_cat, b_cat, *opt = ctx.saved_tensors
    offset_dev = opt.pop(0) if ctx.has_opt[0] else None
    keep_mask = opt.pop(0) if ctx.has_opt[1] else None
    A = ctx.args
    if dy is None:  # Y unused downstream (materialize_grads is off)
        dy = torch.zeros((x.shape[0], w.shape[0]), dtype=_BF16, device=x.device)
    dy = dy.to(_BF16).contiguous()
    need_dx = bool(ctx.needs_input_grad[0])
    dx, dacc = torch.ops.lorafusion_b200.lora_bwd(
        dy, x, w, a_cat, b_cat, s_hat, bits, A["ranks"], A["scalings"], A["ps"], A["seeds"], A["segs"],
        A["offset"], offset_dev, keep_mask, A["training"], A["share_blocks"], A["row_base"], A["cache_id"], need_dx)
    segs = A["segs"]
    segments = [Segment(*segs[i:i + 4]) for i in range(0, len(segs), 4)]
    col_starts, _, R = rank_layout(A["ranks"], segments, A["share_blocks"])
    k, n = x.shape[1], w.shape[0]
    da, db = dacc[:R * k].view(R, k), dacc[R * k:].view(n, R)
    sink = getattr(ctx, "sink", None)
    if sink is not None and segments:
        sink(_SinkLayout(A["ranks"], segments, col_starts), da, db)
    # route the rank-concat gradients back to each adapter's parameters (summing the
    # blocks of one adapter when its segments do not share one, e.g. per-batch slots)
    ga: list = [None] * na
    gb: list = [None] * na
    seen, blocks = set(), []
    for s, c0 in zip(segments, col_starts):
        if (s.adapter, c0) in seen:
            continue
        seen.add((s.adapter, c0))
        blocks.append((s.adapter, c0, A["ranks"][s.adapter]))
    b_parts = _gather_db_blocks(dacc, [(R * k, n, R, c0, r) for _ad, c0, r in blocks])
    for (ad, c0, r), b_part in zip(blocks, b_parts):
        a_part = da[c0:c0 + r]
        ga[ad] = a_part if ga[ad] is None else ga[ad] + a_part
        gb[ad] = b_part if gb[ad] is None else gb[ad] + b_part
    dts = ctx.param_dtypes
    ga = [g.to(dts[i]) if g is not None else None for i, g in enumerate(ga)]
    gb = [g.to(dts[na + i]) if g is not None else None for i, g in enumerate(gb)]
    return (dx if need_dx else None, None, ga, gb) + ctx.none_grads


torch.library.register_autograd(f"{_NS}::lora_fwd", _backward, setup_context=_setup_context)


# --------------------------------------------------------------------------------------
# shared-input groups: several LoRA linears reading the same X
# --------------------------------------------------------------------------------------
def _padr(r: int) -> int:
    return -(-int(r) // 16) * 16


def _group_split(nads, *flat):
    """Per-projection slices of flat per-(projection, adapter) lists."""
    out, pos = [], 0
    for n_ in nads:
        out.append(tuple(list(f[pos:pos + n_]) for f in flat))
        pos += n_
    return out


def _group_layout(m, nads, ranks, segs):
    """(segments, [(col_starts_j, R_j)]) of a group call: the projections share the segment
    table (none: one segment over all rows, adapter 0) and each lays out its own adapters."""
    segs = list(segs) if segs else [0, 0, m, 0]
    segments = [Segment(*segs[i:i + 4]) for i in range(0, len(segs), 4)]
    lays = []
    for (r_j,) in _group_split(nads, ranks):
        cs, _, R = rank_layout(r_j, segments, True)
        lays.append((cs, R))
    return segs, segments, lays


def _group_plan(j, x_rows, k, n, nads, ranks, scalings, ps, seeds, segs, offset, offset_dev,
                training) -> LayerPlan:
    r_j, s_j, p_j, sd_j = _group_split(nads, ranks, scalings, ps, seeds)[j]
    return _plan(x_rows, k, n, r_j, s_j, p_j, sd_j, segs, offset, offset_dev, None, training, True, 0)


@torch.library.custom_op(f"{_NS}::lora_group_fwd", mutates_args=(), device_types="cuda")
def lora_group_fwd(x: torch.Tensor, ws: list[torch.Tensor], a: list[torch.Tensor], b: list[torch.Tensor],
                   nads: list[int], ranks: list[int], scalings: list[float], ps: list[float], seeds: list[int],
                   segs: list[int], offset: int, offset_dev: Optional[torch.Tensor], training: bool,
                   cache_id: int) -> tuple[list[torch.Tensor], list[torch.Tensor], list[torch.Tensor],
                                           list[torch.Tensor], list[torch.Tensor]]:
    """① + ② of every projection j of a shared-input group (its own adapters — nads[j] of
    them, flat in a / b / ranks / … — seeds and dropout masks, one shared Philox offset and
    segment table): returns ([Y_j], [Ŝ_j], [packed keep mask_j or empty], [A_cat_j bf16],
    [B_cat_j bf16])."""
    lib = _lib.load()
    m, k = x.shape
    st = _stream(x.device)
    segs, _, _ = _group_layout(m, nads, ranks, segs)
    ys, shats, bits, acs, bcs, plans = [], [], [], [], [], []
    single = all(n_ == 1 for n_ in nads) and len(segs) == 4
    pre = _group_operands(a, b, ranks) if (single and not cache_id) else None  # one multi-tensor cast
    per = _group_split(nads, a, b)
    for j, w in enumerate(ws):  # ① per projection (own adapters, seeds and masks)
        plan = _group_plan(j, m, k, w.shape[0], nads, ranks, scalings, ps, seeds, segs, offset, offset_dev, training)
        plan.bind(x.device)
        if pre is not None:
            a_cat, b_cat = pre[0][j], pre[1][j]
        else:
            a_cat, b_cat = _rank_concat_operands(plan, per[j][0], per[j][1], cache_id)
        s_hat = torch.empty((m, plan.rank_total), dtype=_BF16, device=x.device)
        _call("dropout_down_fwd", lib.lf_dropout_down_fwd, ctypes.byref(plan.problem), _ptr(x), _ptr(a_cat),
              _ptr(s_hat), st)
        ys.append(torch.empty((m, w.shape[0]), dtype=_BF16, device=x.device))
        shats.append(s_hat)
        bits.append(plan.keep_bits if plan.keep_bits is not None
                    else torch.empty((0,), dtype=torch.uint8, device=x.device))
        acs.append(_own(a_cat, a, None, x))
        bcs.append(_own(b_cat, b, None, x))
        plans.append(plan)
    # ② for the whole group: one GEMM over the concatenated output columns (the library runs
    # the projections one by one where the group shape has no one-launch variant)
    J = len(ws)
    probs = (ctypes.POINTER(_lib.LfProblem) * J)(*[ctypes.pointer(pl.problem) for pl in plans])
    arr = lambda ts: (ctypes.c_void_p * J)(*[t_.data_ptr() for t_ in ts])  # noqa: E731
    _call("base_fwd", lib.lf_base_fwd_group, probs, J, _ptr(x), arr(ws), arr(shats), arr(bcs), arr(ys), st)
    return ys, shats, bits, acs, bcs


@lora_group_fwd.register_fake
def _lora_group_fwd_fake(x, ws, a, b, nads, ranks, scalings, ps, seeds, segs, offset, offset_dev, training, cache_id):
    m, k = x.shape
    segs, segments, lays = _group_layout(m, nads, ranks, segs)
    ys = [x.new_empty((m, w.shape[0])) for w in ws]
    shats = [x.new_empty((m, R)) for _, R in lays]
    bits = [x.new_empty((m, k // 8), dtype=torch.uint8) if _needs_bits(p_j, segs, None, training) else
            x.new_empty((0,), dtype=torch.uint8) for (p_j,) in _group_split(nads, ps)]
    acs = [x.new_empty((R, k)) for _, R in lays]
    bcs = [x.new_empty((w.shape[0], R)) for (_, R), w in zip(lays, ws)]
    return ys, shats, bits, acs, bcs


@torch.library.custom_op(f"{_NS}::lora_group_bwd", mutates_args=(), device_types="cuda")
def lora_group_bwd(dys: list[torch.Tensor], x: torch.Tensor, ws: list[torch.Tensor], acs: list[torch.Tensor],
                   bcs: list[torch.Tensor], shats: list[torch.Tensor], bits: list[torch.Tensor], nads: list[int],
                   ranks: list[int], scalings: list[float], ps: list[float], seeds: list[int], segs: list[int],
                   offset: int, offset_dev: Optional[torch.Tensor], training: bool, cache_id: int,
                   need_dx: bool) -> tuple[torch.Tensor, torch.Tensor]:
    """③ + ④ + ⑤ of every projection: returns (dX = Σ_j dX_j, [dA_cat_0 | dB_cat_0 | dA_cat_1 |
    dB_cat_1 ...] fp32 flat, one zero-fill for the whole group). ④ runs as one launch and ⑤
    as one GEMM over the concatenated reduction dims where the group allows it."""
    lib = _lib.load()
    m, k = x.shape
    st = _stream(x.device)
    segs, _, lays = _group_layout(m, nads, ranks, segs)
    dx = torch.empty((m, k) if need_dx else (0,), dtype=_BF16, device=x.device)
    sizes = [R * (k + w.shape[0]) for (_, R), w in zip(lays, ws)]
    dacc = torch.zeros(sum(sizes), dtype=torch.float32, device=x.device)
    plans, daccs, dss = [], [], []
    pos = 0
    for j, w in enumerate(ws):
        n = w.shape[0]
        plan = _group_plan(j, m, k, n, nads, ranks, scalings, ps, seeds, segs, offset, offset_dev, training)
        plan.bind(x.device, keep_bits=bits[j])
        acc = dacc[pos:pos + sizes[j]]
        pos += sizes[j]
        plans.append(plan)
        daccs.append(acc)
        dss.append(torch.empty((m, plan.rank_total), dtype=_BF16, device=x.device))
    J = len(ws)
    # ③ for the group in one launch: each projection keeps its split-K partials in its own
    # slice of the (self-cleaning, per-stream) workspace
    wsz = [-(-_lib.workspace_bytes(m, pl.rank_total) // 256) * 256 for pl in plans]
    buf = group_workspace(x.device, st.value or 0, sum(wsz))
    off = 0
    for pl, sz in zip(plans, wsz):
        pl.problem.workspace = buf.data_ptr() + off
        pl.problem.workspace_bytes = sz
        off += sz
    probs = (ctypes.POINTER(_lib.LfProblem) * J)(*[ctypes.pointer(pl.problem) for pl in plans])
    arr = lambda ts: (ctypes.c_void_p * J)(*[t_.data_ptr() for t_ in ts])  # noqa: E731
    _call("grad_up", lib.lf_grad_up_group, probs, J, arr(dys), arr(bcs), arr(shats), arr(dss),
          arr([acc[pl.rank_total * k:] for acc, pl in zip(daccs, plans)]), st)
    # ④ for all projections in one launch: each X tile leaves DRAM once
    _call("grad_down", lib.lf_grad_down_group, probs, J, _ptr(x), arr(dss), arr(daccs), st)
    if need_dx:  # ⑤: one GEMM over the concatenated reduction dims (dX written once), or per
        # projection where the group has no one-launch variant (the first writes dX, the others
        # add into it in their epilogues)
        _call("grad_input", lib.lf_grad_input_group, probs, J, arr(dys), arr(ws), arr(dss), arr(acs), _ptr(dx), st)
    return dx, dacc


@lora_group_bwd.register_fake
def _lora_group_bwd_fake(dys, x, ws, acs, bcs, shats, bits, nads, ranks, scalings, ps, seeds, segs, offset,
                         offset_dev, training, cache_id, need_dx):
    m, k = x.shape
    _, _, lays = _group_layout(m, nads, ranks, segs)
    dx = x.new_empty((m, k) if need_dx else (0,))
    return dx, x.new_empty((sum(R * (k + w.shape[0]) for (_, R), w in zip(lays, ws)),), dtype=torch.float32)


_GROUP_ARGS = ("nads", "ranks", "scalings", "ps", "seeds", "segs", "offset", "offset_dev", "training", "cache_id")


def _group_setup_context(ctx, inputs, output):
    x, ws, a, b, *rest = inputs
    ys, shats, bits, acs, bcs = output
    ctx.mark_non_differentiable(*shats, *bits, *acs, *bcs)
    ctx.set_materialize_grads(False)
    args = dict(zip(_GROUP_ARGS, rest))
    # non-tensor arguments get None, except an empty list (no segment table), which
    # flattens like a list of tensors and must come back as []
    ctx.none_grads = tuple([] if isinstance(v, list) and not v else None for v in rest)
    offset_dev = args.pop("offset_dev")
    ctx.has_off = offset_dev is not None
    ctx.J = len(ws)
    ctx.NA = len(a)
    ctx.param_dtypes = [p.dtype for p in a] + [p.dtype for p in b]
    ctx.args = args
    ctx.save_for_backward(x, *ws, *acs, *bcs, *shats, *bits, *([offset_dev] if ctx.has_off else []))


def _group_backward(ctx, gys, _gs=None, _gbits=None, _ga=None, _gb=None):
    J, NA = ctx.J, ctx.NA
    x, *rest = ctx.saved_tensors
    ws, acs, bcs = rest[:J], rest[J:2 * J], rest[2 * J:3 * J]
    shats, bits = rest[3 * J:4 * J], rest[4 * J:5 * J]
    offset_dev = rest[5 * J] if ctx.has_off else None
    A = ctx.args
    need_dx = bool(ctx.needs_input_grad[0])
    dys = [(g if g is not None else torch.zeros((x.shape[0], w.shape[0]), dtype=_BF16, device=x.device))
           .to(_BF16).contiguous() for g, w in zip(gys, ws)]
    dx, dacc = torch.ops.lorafusion_b200.lora_group_bwd(
        dys, x, list(ws), list(acs), list(bcs), list(shats), list(bits), A["nads"], A["ranks"], A["scalings"],
        A["ps"], A["seeds"], A["segs"], A["offset"], offset_dev, A["training"], A["cache_id"], need_dx)
    m, k = x.shape
    _, segments, lays = _group_layout(m, A["nads"], A["ranks"], A["segs"])
    # each projection's rank-concat gradients back to its adapters' parameters (a block per
    # adapter present in the segment table; absent adapters get no gradient)
    ga: list = [None] * NA
    gb: list = [None] * NA
    pos, base = 0, 0
    b_specs, b_slots = [], []
    for j, ((cs, R), w, (r_j,)) in enumerate(zip(lays, ws, _group_split(A["nads"], A["ranks"]))):
        n = w.shape[0]
        da = dacc[pos:pos + R * k].view(R, k)
        seen = set()
        for s_, c0 in zip(segments, cs):
            if s_.adapter in seen:
                continue
            seen.add(s_.adapter)
            i = base + s_.adapter
            r = r_j[s_.adapter]
            ga[i] = da[c0:c0 + r].to(ctx.param_dtypes[i])
            b_specs.append((pos + R * k, n, R, c0, r))
            b_slots.append(i)
        pos += R * (k + n)
        base += len(r_j)
    # every projection's dB blocks in one gather (contiguous per-adapter gradients)
    for i, g in zip(b_slots, _gather_db_blocks(dacc, b_specs)):
        gb[i] = g.to(ctx.param_dtypes[NA + i])
    return (dx if need_dx else None, [None] * J, ga, gb) + ctx.none_grads


torch.library.register_autograd(f"{_NS}::lora_group_fwd", _group_backward, setup_context=_group_setup_context)


def fused_lora_group(x: torch.Tensor, weights: Sequence[torch.Tensor], lora_a: Sequence[torch.Tensor],
                     lora_b: Sequence[torch.Tensor], adapters: Sequence[AdapterConfig], offset: int = 0,
                     training: bool = True, offset_dev: torch.Tensor | None = None,
                     operand_cache: OperandCache | None = None) -> list[torch.Tensor]:
    """Several LoRA linears that read the same input (q/k/v, gate/up): Y_j = X·W_jᵀ +
    s_j·dropout_j(X)·A_jᵀ·B_jᵀ, each with its own adapter, seed and mask (one Philox offset
    for the call). Same results as separate fused_lora calls up to bf16 rounding; ②, ④ and
    ⑤ run as one launch each for the group where its shape allows."""
    if not weights or len(weights) != len(lora_a) or len(weights) != len(lora_b) or len(weights) != len(adapters):
        raise ValidationError("fused_lora_group needs one weight, lora_a, lora_b and adapter per projection")
    return fused_multi_lora_group(x, weights, [[a_] for a_ in lora_a], [[b_] for b_ in lora_b],
                                  [[ad] for ad in adapters], None, offset, training, offset_dev, operand_cache)


def fused_multi_lora_group(x: torch.Tensor, weights: Sequence[torch.Tensor],
                           lora_a: Sequence[Sequence[torch.Tensor]], lora_b: Sequence[Sequence[torch.Tensor]],
                           adapters: Sequence[Sequence[AdapterConfig]], segments: Sequence[Segment] | None = None,
                           offset: int = 0, training: bool = True, offset_dev: torch.Tensor | None = None,
                           operand_cache: OperandCache | None = None) -> list[torch.Tensor]:
    """FusedMultiLoRA for projections that read the same input: projection j has its own
    adapter slots (lora_a[j][i], lora_b[j][i], adapters[j][i]: rank, scale, dropout, seed) and
    all share one microbatch segment table (None: every row to slot 0). Y_j equals
    fused_multi_lora(x, weights[j], lora_a[j], lora_b[j], adapters[j], segments) up to bf16
    rounding. A microbatch beyond one launch's limits (> 32 segments, rank-concat > 128) runs
    projection by projection through fused_multi_lora."""
    J = len(weights)
    if not J or len(lora_a) != J or len(lora_b) != J or len(adapters) != J:
        raise ValidationError("fused_multi_lora_group needs weights, lora_a, lora_b and adapters per projection")
    if J > _lib.LF_MAX_GROUP:
        raise ValidationError(f"at most {_lib.LF_MAX_GROUP} projections per group, got {J}")
    k = weights[0].shape[1]
    x2, lead = _flatten_input(x, k)
    m = x2.shape[0]
    segs_list = list(segments) if segments is not None else None
    nads, flat_a, flat_b, flat_ad = [], [], [], []
    for j, w in enumerate(weights):
        if w.shape[1] != k:
            raise ValidationError(f"weights[{j}] has in_features {w.shape[1]}, expected {k} (one shared input)")
        if len(lora_a[j]) != len(adapters[j]) or len(lora_b[j]) != len(adapters[j]) or not adapters[j]:
            raise ValidationError(f"projection {j}: one lora_a, lora_b and adapter per slot (at least one)")
        if segs_list is not None:
            validate_segments(segs_list, m, len(adapters[j]), max_segments=None)
        packed_j = pack_adapters(adapters[j])
        _check_call(x2, w, lora_a[j], lora_b[j], packed_j[0], k, w.shape[0], None, offset_dev)
        nads.append(len(adapters[j]))
        flat_a += list(lora_a[j])
        flat_b += list(lora_b[j])
        flat_ad += list(adapters[j])
    if m == 0 or segs_list == []:  # no rows, or no LoRA rows: the per-projection path
        return [fused_multi_lora(x, w, lora_a[j], lora_b[j], adapters[j], segs_list or [], offset, None, training,
                                 offset_dev=offset_dev) for j, w in enumerate(weights)]
    if segs_list is not None:
        fits = all(len(split_segments(adapters[j], segs_list, m)) == 1 for j in range(J))
        if not fits:  # beyond one launch: the per-projection path splits the microbatch
            return [fused_multi_lora(x, w, lora_a[j], lora_b[j], adapters[j], segs_list, offset, None, training,
                                     offset_dev=offset_dev, operand_cache=operand_cache)
                    for j, w in enumerate(weights)]
    packed = pack_adapters(flat_ad)
    segs = pack_segments(segs_list) if segs_list else []
    ys = torch.ops.lorafusion_b200.lora_group_fwd(
        x2, list(weights), flat_a, flat_b, nads, *packed, segs, int(offset), offset_dev, bool(training),
        _cache_handle(operand_cache))[0]
    return [y.reshape(lead + (y.shape[1],)) for y in ys]


class _SinkLayout:
    """What a gradient sink sees of a call: (adapter, batch, col_start, rank) per segment."""

    def __init__(self, ranks, segments, col_starts):
        self._rows = [(s.adapter, s.batch, c0, ranks[s.adapter]) for s, c0 in zip(segments, col_starts)]

    def segment_grad_slices(self) -> list[tuple[int, int, int, int]]:
        return list(self._rows)


class _SinkFn(torch.autograd.Function):
    """Autograd node of a call that carries a gradient sink: the same operators, with the
    sink kept on the node for the backward (eager only; a sink is a Python side effect)."""

    @staticmethod
    def forward(ctx, x, w, n_adapters, plan_args, sink, *params):
        a, b = list(params[:n_adapters]), list(params[n_adapters:])
        out = torch.ops.lorafusion_b200.lora_fwd(x, w, a, b, *plan_args)
        _setup_context(ctx, (x, w, a, b, *plan_args), out, mark=False)
        y = out[0]
        ctx.sink = sink
        return y

    @staticmethod
    def backward(ctx, dy):
        dx, _, ga, gb = _backward(ctx, dy)[:4]
        return (dx, None, None, None, None, *ga, *gb)


# --------------------------------------------------------------------------------------
# functional API
# --------------------------------------------------------------------------------------
class _EmptyBatchFn(torch.autograd.Function):
    """An empty batch (m = 0) like nn.Linear: an empty (0, n) output that stays on the
    autograd graph, so backward gives an empty dX and all-zero adapter gradients. Nothing is
    launched (there is no work)."""

    @staticmethod
    def forward(ctx, x, n: int, *params):
        ctx.x_shape = x.shape
        ctx.shapes = [(p.shape, p.dtype, p.device) for p in params]
        return x.new_empty((0, n))

    @staticmethod
    def backward(ctx, dy):
        dx = dy.new_empty(ctx.x_shape) if ctx.needs_input_grad[0] else None
        grads = [torch.zeros(sh, dtype=dt, device=dev) for sh, dt, dev in ctx.shapes]
        return (dx, None, *grads)


def _flatten_input(x: torch.Tensor, k: int) -> tuple[torch.Tensor, tuple]:
    if x.shape[-1] != k:
        raise ValidationError(f"input last dim {x.shape[-1]} != in_features {k}")
    lead = tuple(x.shape[:-1])
    x2 = x.reshape(-1, k)
    if x2.dtype != _BF16:
        raise ValidationError(f"input must be bfloat16, got {x2.dtype}")
    return x2.contiguous(), lead


def _check_frozen(weight: torch.Tensor) -> None:
    if weight.requires_grad:
        raise ValidationError(
            "the base weight must be frozen (requires_grad=False): FusedLoRA trains only the adapters"
        )


def _check_call(x2, weight, lora_a, lora_b, ranks, k, n, keep_mask, offset_dev) -> None:
    _check_operand(x2, "x")
    _check_operand(weight, "weight", (n, k))
    _check_frozen(weight)
    for i, (a, b) in enumerate(zip(lora_a, lora_b)):
        r = ranks[i]
        if tuple(a.shape) != (r, k):
            raise ValidationError(f"lora_a[{i}] must have shape ({r}, {k}), got {tuple(a.shape)}")
        if tuple(b.shape) != (n, r):
            raise ValidationError(f"lora_b[{i}] must have shape ({n}, {r}), got {tuple(b.shape)}")
        if not (a.is_cuda and b.is_cuda):
            raise ValidationError("adapter weights must be CUDA tensors")
    if keep_mask is not None:
        if keep_mask.dtype != torch.uint8 or tuple(keep_mask.shape) != (x2.shape[0], k):
            raise ValidationError(f"keep_mask must be uint8 of shape ({x2.shape[0]}, {k})")
        if not keep_mask.is_contiguous():
            raise ValidationError("keep_mask must be contiguous")
    if offset_dev is not None and (offset_dev.dtype != torch.int64 or offset_dev.numel() != 1 or not offset_dev.is_cuda):
        raise ValidationError("offset_dev must be a one-element int64 CUDA tensor")


def _apply(x2, weight, lora_a, lora_b, packed, segs, offset, offset_dev, keep_mask, training, share_blocks,
           row_base, cache_id, sink=None):
    ranks, scalings, ps, seeds = packed
    plan_args = (ranks, scalings, ps, seeds, segs, int(offset), offset_dev, keep_mask, bool(training),
                 bool(share_blocks), int(row_base), int(cache_id))
    if sink is not None:
        return _SinkFn.apply(x2, weight, len(lora_a), plan_args, sink, *lora_a, *lora_b)
    return torch.ops.lorafusion_b200.lora_fwd(x2, weight, list(lora_a), list(lora_b), *plan_args)[0]


def fused_lora(
    x: torch.Tensor,
    weight: torch.Tensor,
    lora_a: torch.Tensor,
    lora_b: torch.Tensor,
    scaling: float,
    dropout_p: float = 0.0,
    seed: int = 0,
    offset: int = 0,
    keep_mask: torch.Tensor | None = None,
    training: bool = True,
    offset_dev: torch.Tensor | None = None,
    operand_cache: OperandCache | None = None,
) -> torch.Tensor:
    """Y = X·Wᵀ + scaling·dropout(X)·Aᵀ·Bᵀ  (Eq. 1) on one adapter.

    x (..., k) bf16; weight (n, k) = nn.Linear.weight (frozen); lora_a (r, k) =
    lora_A.weight; lora_b (n, r) = lora_B.weight, in any float dtype (fp32 master weights
    are cast to the bf16 operands inside, gradients come back in their dtype). Dropout uses
    SPEC.md §3's Philox mask keyed by (seed, offset) unless ``keep_mask`` (uint8, m x k) is
    given. ``offset_dev``: one-element int64 CUDA tensor added to ``offset`` when the kernels
    run (CUDA graphs: a device-side step counter or an offset drawn from torch's RNG).
    """
    k = weight.shape[1]
    x2, lead = _flatten_input(x, k)
    m = x2.shape[0]
    n = weight.shape[0]
    adapter = AdapterConfig(rank=lora_a.shape[0], scaling=float(scaling), dropout_p=float(dropout_p), seed=int(seed))
    packed = pack_adapters([adapter])
    _check_call(x2, weight, [lora_a], [lora_b], packed[0], k, n, keep_mask, offset_dev)
    if m == 0:
        return _EmptyBatchFn.apply(x2, n, lora_a, lora_b).reshape(lead + (n,))
    y = _apply(x2, weight, [lora_a], [lora_b], packed, [0, 0, m, 0], offset, offset_dev, keep_mask, training, True,
               0, _cache_handle(operand_cache))
    return y.reshape(lead + (n,))


def fused_multi_lora(
    x: torch.Tensor,
    weight: torch.Tensor,
    lora_a: Sequence[torch.Tensor],
    lora_b: Sequence[torch.Tensor],
    adapters: Sequence[AdapterConfig],
    segments: Sequence[Segment],
    offset: int = 0,
    keep_mask: torch.Tensor | None = None,
    training: bool = True,
    grad_sink: Callable | None = None,
    offset_dev: torch.Tensor | None = None,
    operand_cache: OperandCache | None = None,
) -> torch.Tensor:
    """Mixed-adapter microbatch: rows of ``segments`` route to their adapter's A/B, scale
    and dropout; the frozen W is streamed once for all of them.

    ``grad_sink(layout, dA_cat, dB_cat)`` (optional, eager only) receives the fp32
    rank-concat gradients so a caller can keep per-(adapter, global batch) slots
    (``layout.segment_grad_slices()``); segments then get one column block each.
    """
    k = weight.shape[1]
    n = weight.shape[0]
    x2, lead = _flatten_input(x, k)
    if len(lora_a) != len(adapters) or len(lora_b) != len(adapters):
        raise ValidationError("lora_a, lora_b and adapters must have one entry per adapter slot")
    m = x2.shape[0]
    segments = list(segments)
    validate_segments(segments, m, len(adapters), max_segments=None)
    packed = pack_adapters(adapters)
    _check_call(x2, weight, lora_a, lora_b, packed[0], k, n, keep_mask, offset_dev)
    if m == 0:
        return _EmptyBatchFn.apply(x2, n, *lora_a, *lora_b).reshape(lead + (n,))
    share = grad_sink is None
    cache_id = _cache_handle(operand_cache)
    # a microbatch beyond one launch's limits (R > 128 or > 32 segments) runs as several
    # consecutive row ranges; Philox keeps absolute rows (row_base), so masks are unchanged
    parts = split_segments(adapters, segments, m, share_blocks=share) if segments else [(0, m, [])]
    ys = []
    for r0, r1, segs in parts:
        local = [Segment(s_.adapter, s_.row_start - r0, s_.row_end - r0, s_.batch) for s_ in segs]
        xp = x2[r0:r1] if len(parts) > 1 else x2
        km = None if keep_mask is None else (keep_mask[r0:r1] if len(parts) > 1 else keep_mask)
        ys.append(_apply(xp, weight, lora_a, lora_b, packed, pack_segments(local), offset, offset_dev, km, training,
                         share, r0, cache_id, grad_sink))
    y = ys[0] if len(ys) == 1 else torch.cat(ys, 0)
    return y.reshape(lead + (n,))


def dropout_keep_mask(m: int, k: int, adapters: Sequence[AdapterConfig], segments: Sequence[Segment],
                      offset: int = 0, device: torch.device | str = "cuda") -> torch.Tensor:
    """The SPEC.md §3 keep mask (uint8, m x k) the kernels regenerate, materialised on device."""
    plan = LayerPlan(m, k, 8, adapters, segments, offset=offset)
    keep = torch.empty((m, k), dtype=torch.uint8, device=device)
    _lib.check(_lib.load().lf_dropout_mask(ctypes.byref(plan.problem), _ptr(keep), _stream()), "dropout_mask")
    return keep
