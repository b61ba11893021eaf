"""The drop-in boundary under the ways PEFT/HF training drives a LoRA linear (needs a B200):
torch operators + torch.compile, activation checkpointing, fused optimizers, biases and
microbatches beyond one launch's limits."""
from __future__ import annotations

import pytest
import torch
import torch.utils.checkpoint as ckpt

from paper_2510_00206_b200 import AdapterConfig, FusedLoRA, FusedMultiLoRA, Segment, segments_from_lengths

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _rel(a, b):
    a, b = a.detach().float(), b.detach().float()
    return float((a - b).norm() / b.norm().clamp_min(1e-12))


def _layer(seed=0, k=512, n=384, r=16, p=0.1, **kw):
    g = torch.Generator(device=DEV).manual_seed(seed)
    w = (torch.randn(n, k, device=DEV, generator=g) / k**0.5).to(torch.bfloat16)
    return FusedLoRA(w, rank=r, scaling=2.0, dropout_p=p, seed=5, init="gaussian", generator=g, **kw)


def _grads(layer):
    return [p.grad.clone() for p in (layer.lora_A.weight, layer.lora_B.weight)]


def _same_step(got, want):
    """(Y, dX, dA, dB): Y bit-identical; dX, dA, dB within reduction-order noise — ③ and ④
    accumulate split-K partials with red.global.add, whose order is not fixed, so dŜ can
    round to a neighbouring bf16 and dA/dB differ in the last fp32 bits."""
    assert torch.equal(got[0], want[0])
    assert _rel(got[1], want[1]) < 1e-3
    for g_, w_ in zip(got[2:], want[2:]):
        assert _rel(g_, w_) < 1e-4


def test_ops_are_registered_with_fake_impls():
    """the two passes are torch operators with meta implementations."""
    assert hasattr(torch.ops.lorafusion_b200, "lora_fwd") and hasattr(torch.ops.lorafusion_b200, "lora_bwd")
    from torch._subclasses.fake_tensor import FakeTensorMode

    with FakeTensorMode():
        x = torch.empty(300, 256, dtype=torch.bfloat16, device=DEV)
        w = torch.empty(128, 256, dtype=torch.bfloat16, device=DEV)
        a = [torch.empty(8, 256, device=DEV), torch.empty(32, 256, device=DEV)]
        b = [torch.empty(128, 8, device=DEV), torch.empty(128, 32, device=DEV)]
        y, s, bits, a_cat, b_cat = torch.ops.lorafusion_b200.lora_fwd(
            x, w, a, b, [8, 32], [2.0, 1.0], [0.1, 0.0], [1, 2], [0, 0, 100, 0, 1, 100, 300, 0], 0, None, None, True,
            True, 0, 0)
        assert y.shape == (300, 128) and s.shape == (300, 48) and bits.shape == (300, 32)
        assert a_cat.shape == (48, 256) and b_cat.shape == (128, 48)


@pytest.mark.parametrize("reentrant", [False, True], ids=["non_reentrant", "reentrant"])
def test_activation_checkpointing_redraws_the_same_mask(reentrant):
    """torch.utils.checkpoint restores torch's RNG state before recomputing, and the default
    dropout offsets come from torch's CUDA generator: Y and every gradient are identical
    with and without checkpointing."""
    layer = _layer()
    x0 = torch.randn(640, 512, device=DEV).to(torch.bfloat16)
    dy = torch.randn(640, 384, device=DEV).to(torch.bfloat16)
    outs = []
    for use_ckpt in (False, True):
        torch.manual_seed(123)
        x = x0.clone().requires_grad_(True)
        layer.lora_A.weight.grad = layer.lora_B.weight.grad = None
        if use_ckpt:
            y = ckpt.checkpoint(lambda t: layer(t) * 1.0, x, use_reentrant=reentrant)
        else:
            y = layer(x) * 1.0
        y.backward(dy)
        outs.append((y.detach(), x.grad.clone(), *_grads(layer)))
    _same_step(outs[1], outs[0])
    # and a second forward draws a different mask (fresh offset per forward)
    torch.manual_seed(123)
    layer(x0)
    y2 = layer(x0)
    assert not torch.equal(y2, outs[0][0])


def test_torch_compile_fullgraph_matches_eager():
    """FusedLoRA traces into one graph (custom ops + fake impls + registered autograd): no
    graph break under fullgraph=True, and the compiled fwd+bwd equals eager."""
    layer = _layer(seed=1, capturable=True, dropout_rng="counter")
    x0 = torch.randn(512, 512, device=DEV).to(torch.bfloat16)
    dy = torch.randn(512, 384, device=DEV).to(torch.bfloat16)

    def run(fn):
        x = x0.clone().requires_grad_(True)
        layer.lora_A.weight.grad = layer.lora_B.weight.grad = None
        with torch.no_grad():
            layer.step_counter.zero_()
        y = fn(x)
        y.backward(dy)
        return (y.detach(), x.grad.clone(), *_grads(layer))

    eager = run(layer)
    compiled = torch.compile(layer, backend="aot_eager", fullgraph=True)
    got = run(compiled)
    _same_step(got, eager)


def test_operand_cache_sees_fused_optimizer_updates():
    """AdamW(fused=True) updates parameters without bumping their version counters: the
    cached bf16 operands must still be refreshed after every optimizer step."""
    layer = _layer(seed=2, p=0.0)
    fresh = _layer(seed=2, p=0.0, capturable=True)  # no operand cache: re-casts every call
    opt = torch.optim.AdamW(layer.parameters(), lr=1e-2, fused=True)
    x = torch.randn(256, 512, device=DEV).to(torch.bfloat16)
    for _ in range(3):
        y = layer(x)
        y.float().square().mean().backward()
        v0 = layer.lora_A.weight._version
        opt.step()
        opt.zero_grad()
        assert layer.lora_A.weight._version == v0  # the case the version key alone misses
        with torch.no_grad():
            fresh.lora_A.weight.copy_(layer.lora_A.weight)
            fresh.lora_B.weight.copy_(layer.lora_B.weight)
        assert torch.equal(layer(x), fresh(x))
    # updates outside any optimizer: explicit invalidation
    with torch.no_grad():
        layer.lora_B.weight.data.mul_(3.0)
        fresh.lora_B.weight.copy_(layer.lora_B.weight)
    layer.invalidate_operands()
    assert torch.equal(layer(x), fresh(x))


def test_linear_bias_stays_frozen_and_keeps_bf16():
    base = torch.nn.Linear(256, 128, bias=True, device=DEV, dtype=torch.bfloat16)
    base.bias.data = base.bias.data.float()  # an fp32 bias must not promote the output
    layer = FusedLoRA(base, rank=8, init="gaussian")
    x = torch.randn(64, 256, device=DEV).to(torch.bfloat16)
    y = layer(x)
    assert y.dtype == torch.bfloat16 and not base.bias.requires_grad
    ref = (x.float() @ base.weight.float().T + base.bias.float() +
           4.0 * (x.float() @ layer.lora_A.weight.bfloat16().float().T) @ layer.lora_B.weight.bfloat16().float().T)
    assert _rel(y, ref) < 1e-2


def test_module_with_more_than_32_segments_splits():
    """A microbatch of 40 segments runs as several launches (the whole-microbatch
    check no longer rejects it); results equal the per-segment torch reference."""
    from paper_2510_00206_b200 import unfused_multi_lora

    ads = [AdapterConfig(8, 2.0, 0.0, 1), AdapterConfig(16, 1.0, 0.0, 2)]
    segs = segments_from_lengths([i % 2 for i in range(40)], [16] * 40, batches=[i // 2 for i in range(40)])
    g = torch.Generator(device=DEV).manual_seed(3)
    w = (torch.randn(192, 256, device=DEV, generator=g) / 16).to(torch.bfloat16)
    layer = FusedMultiLoRA(w, ads, init="gaussian", generator=g)
    x = torch.randn(640, 256, device=DEV, generator=g).to(torch.bfloat16).requires_grad_(True)
    y = layer(x, segs)
    ref = unfused_multi_lora(x.detach(), w, [a.weight.bfloat16() for a in layer.lora_A],
                             [b.weight.bfloat16() for b in layer.lora_B], ads, segs)
    assert _rel(y, ref) < 1e-2
    y.float().sum().backward()
    assert x.grad is not None and all(p.grad is not None for p in layer.parameters() if p.requires_grad)


def test_slot_grads_split_unshared_blocks():
    """track_slot_grads gives each (adapter, batch) segment its own column block: three
    rank-64 global batches (192 columns) are split into launches that fit."""
    g = torch.Generator(device=DEV).manual_seed(4)
    w = (torch.randn(128, 256, device=DEV, generator=g) / 16).to(torch.bfloat16)
    ads = [AdapterConfig(64, 1.0, 0.1, 7)]
    layer = FusedMultiLoRA(w, ads, init="gaussian", generator=g, track_slot_grads=True)
    segs = [Segment(0, 0, 128, 0), Segment(0, 128, 256, 1), Segment(0, 256, 384, 2)]
    x = torch.randn(384, 256, device=DEV, generator=g).to(torch.bfloat16)
    layer(x, segs).float().square().mean().backward()
    total_a = sum(layer.slot_grads[(0, bt)][0] for bt in range(3))
    total_b = sum(layer.slot_grads[(0, bt)][1] for bt in range(3))
    torch.testing.assert_close(total_a, layer.lora_A[0].weight.grad, rtol=1e-5, atol=1e-6)
    torch.testing.assert_close(total_b, layer.lora_B[0].weight.grad, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("p,ranks,kv", [(0.0, [16, 8, 16], 128), (0.1, [16, 8, 16], 128), (0.1, [64, 16, 32], 128),
                                       (0.0, [16, 8, 16], 256), (0.1, [64, 16, 32], 256)],
                         ids=["p0", "p01", "p01_r64", "p0_onegemm", "p01_r64_onegemm"])
def test_group_matches_separate_projections(p, ranks, kv):
    """FusedLoRAGroup (q/k/v sharing X) = three FusedLoRA layers at the same Philox offset:
    identical outputs, the same dX as autograd's sum of the three input gradients up to bf16
    rounding (the group's ⑤ is one GEMM over the concatenated reduction dims — dX rounded once
    instead of per projection), same dA/dB (④ runs as one launch for the group). kv = 256:
    whole 256-column tiles, so ② also runs as one GEMM over the concatenated outputs
    (lf_base_fwd_group); kv = 128 exercises its per-projection fallback."""
    from paper_2510_00206_b200 import FusedLoRAGroup

    g = torch.Generator(device=DEV).manual_seed(11)
    k = 512
    bases = {nm: (torch.randn(n, k, device=DEV, generator=g) / k**0.5).to(torch.bfloat16)
             for nm, n in (("q_proj", 512), ("k_proj", kv), ("v_proj", kv))}
    grp = FusedLoRAGroup(bases, rank=ranks, scaling=[2.0, 1.0, 0.5], dropout_p=[p, p, 0.0], seeds=[3, 4, 5],
                         init="gaussian", generator=g, dropout_rng="counter")
    x0 = torch.randn(640, k, device=DEV, generator=g).to(torch.bfloat16)
    dys = [torch.randn(640, n.shape[0], device=DEV, generator=g).to(torch.bfloat16) for n in bases.values()]
    grp._offset = 7
    x = x0.clone().requires_grad_(True)
    ys = grp(x)
    torch.autograd.backward(ys, dys)
    got = [(y.detach(), grp.proj(nm).lora_A.weight.grad.clone(), grp.proj(nm).lora_B.weight.grad.clone())
           for y, nm in zip(ys, grp.names)]
    dx_group = x.grad.clone()
    xs = x0.clone().requires_grad_(True)
    for j, nm in enumerate(grp.names):
        layer = grp.proj(nm)
        layer.lora_A.weight.grad = layer.lora_B.weight.grad = None
        layer.dropout_rng = "counter"
        layer._offset = 7
        y = layer(xs)
        y.backward(dys[j])
        assert torch.equal(y, got[j][0])
        # dA/dB: the same fp32 products summed in another split-K partition (one ④ launch for
        # the group vs one per projection; red.global.add order) — reduction-order noise only
        assert _rel(layer.lora_A.weight.grad, got[j][1]) < 1e-4 and _rel(layer.lora_B.weight.grad, got[j][2]) < 1e-4
    # one rounding of the summed input gradient (group) vs three bf16 dX_j added in bf16
    # (autograd): bf16-level differences only (SPEC.md §5 tolerance)
    assert _rel(dx_group, xs.grad) < 4e-3


def test_group_compiles_fullgraph():
    from paper_2510_00206_b200 import FusedLoRAGroup

    g = torch.Generator(device=DEV).manual_seed(12)
    bases = {nm: (torch.randn(256, 256, device=DEV, generator=g) / 16).to(torch.bfloat16) for nm in ("gate", "up")}
    grp = FusedLoRAGroup(bases, rank=16, dropout_p=0.1, init="gaussian", generator=g, capturable=True,
                         dropout_rng="counter")
    x0 = torch.randn(384, 256, device=DEV, generator=g).to(torch.bfloat16)

    def run(fn):
        x = x0.clone().requires_grad_(True)
        for p_ in grp.parameters():
            p_.grad = None
        with torch.no_grad():
            grp.step_counter.zero_()
        y1, y2 = fn(x)
        (y1.float() * y2.float()).sum().backward()
        return y1.detach(), x.grad.clone(), grp.gate.lora_A.weight.grad.clone()

    eager = run(grp)
    got = run(torch.compile(grp, backend="aot_eager", fullgraph=True))
    assert torch.equal(got[0], eager[0]) and _rel(got[1], eager[1]) < 1e-3 and _rel(got[2], eager[2]) < 1e-4


@pytest.mark.parametrize("m,k,ns,wide", [(8192, 4096, (4096, 1024, 1024), ""), (2048, 1024, (2048, 512, 512), "0")],
                         ids=["c2_qkv", "small_narrow_tiles"])
def test_group_one_gemm_vs_fp32_torch(m, k, ns, wide):
    """The shared-input group at a full BASELINE C2 q/k/v size through lf_base_fwd_group (one
    GEMM over N = 6144 — 256 x 512 tiles) and lf_grad_input_group (one GEMM over K = 6144 with
    three masked LoRA terms entering the accumulator in turn) against a torch fp32
    restatement of Eq. 1 on the kernels' own keep masks: rel-Fro <= 4e-3 (SPEC.md §5)."""
    import os
    import subprocess
    import sys

    if wide:  # the 256 x 256 group tiles: another process (LF_WIDE is read once)
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        r = subprocess.run([sys.executable, "-c", f"import tests.test_api_gpu as t; t._group_vs_fp32({m}, {k}, {ns})"],
                           cwd=root, env=dict(os.environ, LF_WIDE=wide), capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
        return
    _group_vs_fp32(m, k, ns)


def _group_vs_fp32(m, k, ns, p=0.1):
    from paper_2510_00206_b200 import AdapterConfig, Segment, dropout_keep_mask, fused_lora_group

    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device=DEV).manual_seed(21)
    x = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16).requires_grad_(True)
    ws = [(torch.randn(n, k, device=DEV, generator=g) / k**0.5).to(torch.bfloat16) for n in ns]
    As = [((torch.rand(16, k, device=DEV, generator=g) * 2 - 1) / k**0.5).requires_grad_(True) for _ in ns]
    Bs = [(torch.randn(n, 16, device=DEV, generator=g) / 4).requires_grad_(True) for n in ns]
    dys = [torch.randn(m, n, device=DEV, generator=g).to(torch.bfloat16) for n in ns]
    ads = [AdapterConfig(16, 2.0, p if j < 2 else 0.0, 40 + j) for j in range(len(ns))]
    ys = fused_lora_group(x, ws, As, Bs, ads, offset=5)
    torch.autograd.backward(ys, dys)
    rel = lambda g_, r_: float((g_.float() - r_).norm() / r_.norm())  # noqa: E731
    dx_ref = torch.zeros(m, k, device=DEV)
    errs = {}
    for j, (w, a, b, dy, ad) in enumerate(zip(ws, As, Bs, dys, ads)):
        keep = dropout_keep_mask(m, k, [ad], [Segment(0, 0, m)], offset=5, device=DEV).float()
        sc = ad.scaling / (1.0 - ad.dropout_p)
        ab, bb = a.detach().bfloat16().float(), b.detach().bfloat16().float()
        xm = x.detach().float() * keep
        s = ((xm @ ab.T) * sc).bfloat16().float()
        errs[f"y{j}"] = rel(ys[j].detach(), x.detach().float() @ w.float().T + s @ bb.T)
        ds = ((dy.float() @ bb) * sc).bfloat16().float()
        errs[f"dA{j}"] = rel(a.grad, ds.T @ xm)
        errs[f"dB{j}"] = rel(b.grad, dy.float().T @ s)
        dx_ref += dy.float() @ w.float() + keep * (ds @ ab)
        del xm, keep
    errs["dx"] = rel(x.grad, dx_ref)
    assert all(v < 4e-3 for v in errs.values()), errs


@pytest.mark.parametrize("ranks,ps", [((8, 16, 32, 64), (0.0, 0.05, 0.1, 0.1)), ((8, 16), (0.1, 0.0))],
                         ids=["c3_like", "rsum_small"])
def test_multi_lora_group_matches_separate_layers(ranks, ps):
    """FusedMultiLoRAGroup (q/k/v sharing X, 4 or 2 adapter slots each, one segment table) =
    three FusedMultiLoRA layers at the same Philox offset: identical Y (the group GEMM's LoRA
    K-range covers each projection's whole rank-concat width — zero off-segment columns add
    exact zeros), dA/dB up to reduction order, dX up to bf16 rounding. rsum_small: the
    accumulators of all three fit one ④ launch; c3_like (R = 128 each): ④ per projection."""
    from paper_2510_00206_b200 import FusedMultiLoRAGroup, segments_from_lengths

    g = torch.Generator(device=DEV).manual_seed(13)
    k = 512
    bases = {nm: (torch.randn(n, k, device=DEV, generator=g) / k**0.5).to(torch.bfloat16)
             for nm, n in (("q_proj", 512), ("k_proj", 256), ("v_proj", 256))}
    ads = [AdapterConfig(r, 2.0 / (i + 1), p_, seed=50 + i) for i, (r, p_) in enumerate(zip(ranks, ps))]
    seeds = [[100 * j + i for i in range(len(ads))] for j in range(3)]
    grp = FusedMultiLoRAGroup(bases, ads, seeds=seeds, init="gaussian", generator=g, dropout_rng="counter")
    lens = [200, 184, 128, 128][:len(ads)]
    segs = segments_from_lengths(list(range(len(ads))), lens)
    m = sum(lens)
    x0 = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16)
    dys = [torch.randn(m, b_.shape[0], device=DEV, generator=g).to(torch.bfloat16) for b_ in bases.values()]
    grp._offset = 3
    x = x0.clone().requires_grad_(True)
    ys = grp(x, segs)
    torch.autograd.backward(ys, dys)
    dx_group = x.grad.clone()
    got = [(y.detach(), [la.weight.grad.clone() for la in grp.proj(nm).lora_A],
            [lb.weight.grad.clone() for lb in grp.proj(nm).lora_B]) for y, nm in zip(ys, grp.names)]
    xs = x0.clone().requires_grad_(True)
    for j, nm in enumerate(grp.names):
        layer = grp.proj(nm)
        for p_ in layer.parameters():
            p_.grad = None
        layer.dropout_rng = "counter"
        layer._offset = 3
        y = layer(xs, segs)
        y.backward(dys[j])
        assert torch.equal(y, got[j][0])
        for ga, gl in zip(got[j][1] + got[j][2], [la.weight.grad for la in layer.lora_A] +
                          [lb.weight.grad for lb in layer.lora_B]):
            assert _rel(gl, ga) < 1e-4
    assert _rel(dx_group, xs.grad) < 4e-3


@pytest.mark.parametrize("grouped", [False, True], ids=["layer", "group"])
def test_capturable_multi_lora_step_has_no_operand_or_grad_copies(grouped):
    """A capturable multi-adapter step (ranks 8/16/32/64: padded and full blocks) reads the
    persistent rank-concat operands and gathers every dB column block in one index_select:
    after the first call the fwd+bwd launches no cast, pad, cat or strided-copy kernels, and
    its outputs and gradients equal the non-capturable layer's bit for bit."""
    from torch.profiler import ProfilerActivity, profile

    from paper_2510_00206_b200 import FusedMultiLoRAGroup

    g = torch.Generator(device=DEV).manual_seed(21)
    k = 256
    ads = [AdapterConfig(r, 2.0, 0.0, seed=i + 1) for i, r in enumerate((8, 16, 32, 64))]
    segs = segments_from_lengths([0, 1, 2, 3], [128, 256, 128, 128])
    m = 640
    names = ("q", "k") if grouped else ("q",)
    bases = {nm: (torch.randn(n, k, device=DEV, generator=g) / 16).to(torch.bfloat16) for nm, n in zip(names, (384, 128))}
    caps = {nm: FusedMultiLoRA(w, ads, init="gaussian", generator=g, capturable=True) for nm, w in bases.items()}
    refs = {nm: FusedMultiLoRA(w, ads, init="gaussian") for nm, w in bases.items()}
    with torch.no_grad():
        for nm in names:
            for pr, pc in zip(refs[nm].parameters(), caps[nm].parameters()):
                pr.copy_(pc)
    mod = FusedMultiLoRAGroup.from_layers(caps) if grouped else caps["q"]
    ref = FusedMultiLoRAGroup.from_layers(refs) if grouped else refs["q"]
    x = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16)
    dys = [torch.randn(m, w.shape[0], device=DEV, generator=g).to(torch.bfloat16) for w in bases.values()]

    def step(layer):
        for p_ in layer.parameters():
            p_.grad = None
        ys = layer(x, segs)
        ys = ys if isinstance(ys, tuple) else (ys,)
        torch.autograd.backward(ys, dys)
        return ys

    step(mod)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ys = step(mod)
        torch.cuda.synchronize()
    names_run = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    bad = [nm_ for nm_ in names_run if any(t in nm_ for t in ("copy_kernel", "CatArray", "bfloat16_copy"))]
    assert not bad, bad
    ys_ref = step(ref)
    for y, yr in zip(ys, ys_ref):
        assert torch.equal(y, yr)
    for pc, pr in zip(mod.parameters(), ref.parameters()):
        assert pc.grad.is_contiguous()
        assert torch.equal(pc.grad, pr.grad)


def test_copy_column_blocks_matches_slicing():
    """lf_copy_column_blocks (through functional._gather_db_blocks): vectorised blocks (widths
    and offsets multiples of 4), scalar ones (width 3, column 5) and whole-row blocks (views,
    no copy) all equal the torch slices, over several matrices of one flat buffer."""
    from paper_2510_00206_b200.functional import _gather_db_blocks

    g = torch.Generator(device=DEV).manual_seed(4)
    flat = torch.randn(300 * 128 + 77 * 48 + 9 * 16, device=DEV, generator=g)
    specs = [(0, 300, 128, 0, 8), (0, 300, 128, 16, 64), (0, 300, 128, 5, 3), (300 * 128, 77, 48, 32, 16),
             (300 * 128 + 77 * 48, 9, 16, 0, 16)]
    got = _gather_db_blocks(flat, specs)
    for (off, n, R, c0, r), t in zip(specs, got):
        ref = flat[off:off + n * R].view(n, R)[:, c0:c0 + r]
        assert t.is_contiguous() and torch.equal(t, ref)
    assert got[-1].data_ptr() == flat[300 * 128 + 77 * 48:].data_ptr()  # whole rows: a view


def test_copy_column_blocks_more_blocks_than_one_launch_holds():
    """More than LF_MAX_COPY_BLOCKS blocks in one call: copied in several launches, each
    block still equal to its torch slice."""
    from paper_2510_00206_b200 import _lib
    from paper_2510_00206_b200.functional import _gather_db_blocks

    g = torch.Generator(device=DEV).manual_seed(6)
    n, R = 96, 128
    flat = torch.randn(n * R, device=DEV, generator=g)
    specs = [(0, n, R, (8 * i) % 120, 8) for i in range(_lib.LF_MAX_COPY_BLOCKS + 6)]
    got = _gather_db_blocks(flat, specs)
    for (off, n_, R_, c0, r), t in zip(specs, got):
        assert torch.equal(t, flat[off:off + n_ * R_].view(n_, R_)[:, c0:c0 + r])
