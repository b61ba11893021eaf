"""Functional FusedLoRA / FusedMultiLoRA (forward + backward through the sm_100a kernels).

Forward:  ① lf_dropout_down_fwd   Ŝ = s·(M⊙X)·Aᵀ
                               ② lf_base_fwd           Y = X·Wᵀ + Ŝ·Bᵀ   (one write of Y)
Backward:  ③ lf_grad_up            dŜ = s·dY·B, dB += dYᵀ·Ŝ   (one read of dY)
                               ④ lf_grad_down          dA += dŜᵀ·(M⊙X)
                               ⑤ lf_grad_input         dX = dY·W + M⊙(dŜ·A)       (one write of dX)

The base weight is frozen (LoRA fine-tuning); there is no CPU path — tensors must live on
a B200 and the shared library must be built, otherwise the call raises.
"""
from __future__ import annotations

import ctypes
from typing import Callable, Sequence

import torch

from . import _lib
from .errors import ValidationError
from .plan import AdapterConfig, LayerPlan, Segment, split_segments, validate_segments

_BF16 = torch.bfloat16


def _ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _stream(device: torch.device | None = None) -> ctypes.c_void_p:
    """The current torch stream of ``device`` as a raw cudaStream_t (cheap: no Stream object)."""
    idx = device.index if device is not None and device.index is not None else torch._C._cuda_getDevice()
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(idx))


class LaunchStats:
    """Counts kernel launches and (optionally) times each launcher with CUDA events on the
    launching stream. Install with ``set_launch_stats``; used by bench.py."""

    def __init__(self, timed: bool = False):
        self.timed = timed
        self.launches: dict[str, int] = {}
        self.events: dict[str, list] = {}

    def begin(self, name: str):
        self.launches[name] = self.launches.get(name, 0) + 1
        if not self.timed:
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        return ev

    def end(self, name: str, start) -> None:
        if start is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.events.setdefault(name, []).append((start, ev))

    # device kernels each C entry point launches (① and ③ add the split-K finalize kernel)
    KERNELS_PER_CALL = {"grad_up": 2}  # ③ + its split-K finalize; ① finalizes in-kernel

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


class OperandCache:
    """bf16 rank-concat operands (A_cat, B_cat) of a module, keyed by the column-block
    layout and the in-place versions of the adapter parameters: every layer call between
    two optimizer steps that sees the same adapters reuses them instead of re-casting,
    padding and concatenating (a dozen small launches of host work per call)."""

    def __init__(self, capacity: int = 8):
        self.capacity = capacity
        self._d: dict = {}

    def get(self, key):
        return self._d.get(key)

    def put(self, key, value) -> None:
        if len(self._d) >= self.capacity:
            self._d.pop(next(iter(self._d)))
        self._d[key] = value


def _rank_concat_operands(plan: LayerPlan, params, n_adapters: int):
    cache: OperandCache | None = plan.operand_cache
    key = None
    if cache is not None:
        blocks = plan.column_blocks()
        used = sorted({a for a, _, _ in blocks})
        key = (tuple((a, r) for a, _, r in blocks),
               tuple((p.data_ptr(), p._version) for a in used for p in (params[a], params[n_adapters + a])))
        hit = cache.get(key)
        if hit is not None:
            return hit
    # bf16 operand copies: the module's cached shadows when given, else cast here
    shadows = plan.weights_bf16
    a_cat = plan.gather_a(shadows[0] if shadows else params[:n_adapters])
    b_cat = plan.gather_b(shadows[1] if shadows else params[n_adapters:])
    if cache is not None:
        cache.put(key, (a_cat, b_cat))
    return a_cat, b_cat


class _FusedLoRAFn(torch.autograd.Function):
    """Autograd node over the five kernels.

    Inputs: x (m,k) bf16, w (n,k) bf16 frozen, the plan, an optional per-slot gradient sink,
    then the adapter parameters lora_A[0..a) and lora_B[0..a) in their own dtype (fp32
    master weights are cast to the bf16 rank-concat operands inside, outside autograd, so
    their gradients come back in fp32 without a bf16 round trip)."""

    @staticmethod
    def forward(ctx, x, w, plan: LayerPlan, grad_sink, n_adapters: int, *params):
        lib = _lib.load()
        m, k, n, R = plan.m, plan.k, plan.n, plan.rank_total
        pp = ctypes.byref(plan.problem)
        y = torch.empty((m, n), dtype=_BF16, device=x.device)
        s_hat = a_cat = b_cat = None
        st = _stream(x.device)
        if plan.has_lora:
            a_cat, b_cat = _rank_concat_operands(plan, params, n_adapters)
            s_hat = torch.empty((m, R), dtype=_BF16, device=x.device)
            _call("dropout_down_fwd", lib.lf_dropout_down_fwd, pp, _ptr(x), _ptr(a_cat), _ptr(s_hat), st)
        _call("base_fwd", lib.lf_base_fwd, pp, _ptr(x), _ptr(w), _ptr(s_hat), _ptr(b_cat), _ptr(y), st)
        ctx.plan = plan
        ctx.grad_sink = grad_sink
        ctx.n_adapters = n_adapters
        ctx.param_dtypes = [p.dtype for p in params]
        ctx.save_for_backward(x, w, a_cat, b_cat, s_hat)
        return y

    @staticmethod
    def backward(ctx, dy):
        lib = _lib.load()
        plan: LayerPlan = ctx.plan
        x, w, a_cat, b_cat, s_hat = ctx.saved_tensors
        m, k, n, R = plan.m, plan.k, plan.n, plan.rank_total
        dy = dy.to(_BF16).contiguous()
        pp = ctypes.byref(plan.problem)
        da = db = ds = None
        st = _stream(dy.device)
        if plan.has_lora:
            ds = torch.empty((m, R), dtype=_BF16, device=dy.device)
            # one zero-fill for both fp32 accumulators
            acc = torch.zeros(R * k + n * R, dtype=torch.float32, device=dy.device)
            da = acc[:R * k].view(R, k)
            db = acc[R * k:].view(n, R)
            _call("grad_up", lib.lf_grad_up, pp, _ptr(dy), _ptr(b_cat), _ptr(s_hat), _ptr(ds), _ptr(db), st)
            _call("grad_down", lib.lf_grad_down, pp, _ptr(x), _ptr(ds), _ptr(da), st)
        dx = None
        if ctx.needs_input_grad[0]:
            dx = torch.empty((m, k), dtype=_BF16, device=dy.device)
            _call("grad_input", lib.lf_grad_input, pp, _ptr(dy), _ptr(w), _ptr(ds), _ptr(a_cat), _ptr(dx), st)
        if ctx.grad_sink is not None and plan.has_lora:
            ctx.grad_sink(plan, da, db)
        # route the rank-concat gradients back to each adapter's parameters (summing the
        # segments that share an adapter, e.g. two global batches in one microbatch)
        na = ctx.n_adapters
        ga: list = [None] * na
        gb: list = [None] * na
        if plan.has_lora:
            for adapter, c0, r in plan.adapter_grad_slices():
                a_part, b_part = da[c0:c0 + r], db[:, c0:c0 + r]
                ga[adapter] = a_part if ga[adapter] is None else ga[adapter] + a_part
                gb[adapter] = b_part if gb[adapter] is None else gb[adapter] + b_part
        dts = ctx.param_dtypes
        ga = [g.to(dts[i]) if g is not None else None for i, g in enumerate(ga)]
        gb = [g.to(dts[na + i]) if g is not None else None for i, g in enumerate(gb)]
        return (dx, None, None, None, None, *ga, *gb)


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
    weights_bf16: tuple | None = None,
    offset_dev: torch.Tensor | None = None,
    operand_cache: OperandCache | None = None,
) -> torch.Tensor:
    """Y = X·Wᵀ + scaling·dropout(X)·Aᵀ·Bᵀ  (Eq. 1) on one adapter.

    x (..., k) bf16; weight (n, k) = nn.Linear.weight (frozen); lora_a (r, k) =
    lora_A.weight; lora_b (n, r) = lora_B.weight. Dropout uses SPEC.md §3's Philox mask
    keyed by (seed, offset) unless ``keep_mask`` (uint8, m x k) is given.
    ``weights_bf16 = (a_bf16, b_bf16)``: bf16 copies of fp32 master weights kept current by
    the caller (the modules refresh them when the parameters change); default: cast here.
    ``offset_dev``: one-element int64 CUDA tensor added to ``offset`` when the kernels run
    (CUDA-graph capture: advance it on the device between replays).
    """
    k = weight.shape[1]
    x2, lead = _flatten_input(x, k)
    m = x2.shape[0]
    adapter = AdapterConfig(rank=lora_a.shape[0], scaling=float(scaling), dropout_p=float(dropout_p), seed=int(seed))
    plan = LayerPlan(m, k, weight.shape[0], [adapter], [Segment(0, 0, m)] if m > 0 else [], offset=offset,
                     training=training, keep_mask=keep_mask, offset_dev=offset_dev)
    if weights_bf16 is not None:
        plan.weights_bf16 = ([weights_bf16[0]], [weights_bf16[1]])
    plan.operand_cache = operand_cache
    return _run(x2, weight, [lora_a], [lora_b], plan, lead, None)


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
    weights_bf16: tuple | None = None,
    offset_dev: torch.Tensor | None = None,
    operand_cache: OperandCache | None = None,
) -> torch.Tensor:
    """Mixed-adapter microbatch: rows of ``segments`` route to their adapter's A/B, scale
    and dropout; the frozen W is streamed once for all of them.

    ``grad_sink(plan, dA_cat, dB_cat)`` (optional) receives the fp32 rank-concat gradients
    so a caller can keep per-(adapter, global batch) slots (plan.segment_grad_slices()).
    """
    k = weight.shape[1]
    x2, lead = _flatten_input(x, k)
    if len(lora_a) != len(adapters) or len(lora_b) != len(adapters):
        raise ValidationError("lora_a, lora_b and adapters must have one entry per adapter slot")
    m = x2.shape[0]
    validate_segments(list(segments), m, len(adapters))
    # a microbatch beyond one launch's limits (R > 128 or > 32 segments) runs as several
    # consecutive row ranges; Philox keeps absolute rows (row_base), so masks are unchanged
    parts = split_segments(adapters, segments, m) if segments else [(0, m, [])]
    ys = []
    for r0, r1, segs in parts:
        local = [Segment(s_.adapter, s_.row_start - r0, s_.row_end - r0, s_.batch) for s_ in segs]
        plan = LayerPlan(r1 - r0, k, weight.shape[0], adapters, local, offset=offset, training=training,
                         keep_mask=None if keep_mask is None else keep_mask[r0:r1],
                         share_blocks=grad_sink is None, offset_dev=offset_dev, row_base=r0)
        if weights_bf16 is not None:
            plan.weights_bf16 = (list(weights_bf16[0]), list(weights_bf16[1]))
        plan.operand_cache = operand_cache
        ys.append(_run(x2[r0:r1] if len(parts) > 1 else x2, weight, lora_a, lora_b, plan, (r1 - r0,), grad_sink))
    y = ys[0] if len(ys) == 1 else torch.cat(ys, 0)
    return y.reshape(lead + (weight.shape[0],))


def _run(x2, weight, lora_a, lora_b, plan: LayerPlan, lead, grad_sink):
    _check_operand(x2, "x")
    _check_operand(weight, "weight", (plan.n, plan.k))
    _check_frozen(weight)
    for i, (a, b) in enumerate(zip(lora_a, lora_b)):
        r = plan.adapters[i].rank
        if tuple(a.shape) != (r, plan.k):
            raise ValidationError(f"lora_a[{i}] must have shape ({r}, {plan.k}), got {tuple(a.shape)}")
        if tuple(b.shape) != (plan.n, r):
            raise ValidationError(f"lora_b[{i}] must have shape ({plan.n}, {r}), got {tuple(b.shape)}")
        if not (a.is_cuda and b.is_cuda):
            raise ValidationError("adapter weights must be CUDA tensors")
    if plan.m == 0:
        return _EmptyBatchFn.apply(x2, plan.n, *lora_a, *lora_b).reshape(lead + (plan.n,))
    plan.bind(x2.device)
    y = _FusedLoRAFn.apply(x2, weight, plan, grad_sink, len(lora_a), *lora_a, *lora_b)
    return y.reshape(lead + (plan.n,))


def dropout_keep_mask(m: int, k: int, adapters: Sequence[AdapterConfig], segments: Sequence[Segment],
                      offset: int = 0, device: torch.device | str = "cuda") -> torch.Tensor:
    """The SPEC.md §3 keep mask (uint8, m x k) the kernels regenerate, materialised on device."""
    plan = LayerPlan(m, k, 8, adapters, segments, offset=offset)
    keep = torch.empty((m, k), dtype=torch.uint8, device=device)
    _lib.check(_lib.load().lf_dropout_mask(ctypes.byref(plan.problem), _ptr(keep), _stream()), "dropout_mask")
    return keep
