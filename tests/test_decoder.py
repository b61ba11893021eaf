"""C5 caller of the hot path: packing of planner microbatches and the LoRA decoder stack.

CPU: sequence/label/position packing from the lorasched-planned C5 schedule
(tests/golden/schedule_c5.json, made by tests/golden/make_c5_schedule.py).
GPU: a tiny decoder whose 7 linears per layer are FusedMultiLoRA layers agrees with the
same model built from the unfused torch projections (loss and every adapter gradient).
"""
from __future__ import annotations

import json
import math
import os

import pytest
import torch

from paper_2510_00206_b200 import AdapterConfig, Segment
from paper_2510_00206_b200 import decoder as D
from paper_2510_00206_b200 import schedule as sched
from paper_2510_00206_b200.errors import ValidationError
from paper_2510_00206_b200.schedule import MicrobatchPlan

HERE = os.path.dirname(os.path.abspath(__file__))
C5 = json.load(open(os.path.join(HERE, "golden", "schedule_c5.json")))


def test_c5_schedule_adapters_and_capacity():
    ids, cfgs = sched.adapters_from_doc(C5)
    assert [c.rank for c in cfgs] == [8, 16, 32, 64]
    assert [c.dropout_p for c in cfgs] == [0.0, 0.05, 0.1, 0.1]
    assert all(c.scaling == 2.0 for c in cfgs)
    mbs = sched.microbatches_from_doc(C5)
    assert len(mbs) >= 8 and all(mb.rows <= C5["capacity"] for mb in mbs)
    assert all(sum(mb.sequences) == mb.rows for mb in mbs)


def test_pack_microbatch_labels_positions_padding():
    mbs = sched.microbatches_from_doc(C5)
    for mb in mbs[:6]:
        pm = D.pack_microbatch(mb, 1000, "cpu", torch.Generator().manual_seed(0))
        assert pm.rows == mb.rows and pm.raw_tokens == mb.raw_tokens
        cu = pm.cu_seqlens.tolist()
        assert cu[0] == 0 and cu[-1] == mb.rows and pm.max_seqlen == max(mb.sequences)
        for a, b in zip(cu[:-1], cu[1:]):
            assert pm.positions[a:b].tolist() == list(range(b - a))
            assert pm.labels[b - 1] == -100  # never predict across a boundary
            assert torch.equal(pm.labels[a:b - 1][pm.labels[a:b - 1] != -100],
                               pm.tokens[a + 1:b][pm.labels[a:b - 1] != -100])
        for seg, raw in zip(mb.segments, mb.segment_raw):
            pad = slice(seg.row_start + raw, seg.row_end)
            assert (pm.tokens[pad] == 0).all() and (pm.labels[pad] == -100).all()
        # every non-pad, non-final row has a loss target
        n_loss = int((pm.labels != -100).sum())
        n_seq_real = len(mb.sequences) - sum(1 for s, r in zip(mb.segments, mb.segment_raw) if r < s.rows)
        assert n_loss == mb.raw_tokens - n_seq_real


def test_pack_microbatch_rejects_plans_without_sequences():
    mb = MicrobatchPlan(0, 0, (Segment(0, 0, 64),), 64, 64)
    with pytest.raises(ValidationError):
        D.pack_microbatch(mb, 100, "cpu")


def test_linear_flops_counts_lora_terms():
    s = D.DecoderShape(hidden=64, heads=2, kv_heads=1, ffn=128, layers=3, vocab=10)
    base = s.linear_flops(10)
    assert base == 3 * sum(4 * 10 * k * n for k, n in s.proj_shapes().values())
    extra = s.linear_flops(10, [(8, 10)]) - base
    assert extra == 3 * sum(6 * 10 * 8 * (k + n) for k, n in s.proj_shapes().values())


TINY = D.DecoderShape(hidden=256, heads=4, kv_heads=2, ffn=512, layers=2, vocab=512)


def _tiny_plan():
    segs = (Segment(0, 0, 192, 0), Segment(1, 192, 320, 0), Segment(2, 320, 448, 0))
    return MicrobatchPlan(0, 0, segs, 448, 440, (100, 92, 128, 60, 60, 8), (192, 128, 120))


def _copy_weights(dst, src, n_adapters):
    """dst <- src (frozen weights and adapter weights), casting to dst's dtypes."""
    with torch.no_grad():
        dst.embed.weight.copy_(src.embed.weight)
        dst.head.copy_(src.head)
        for ld, ls in zip(dst.layers, src.layers):
            for nm in D.PROJECTIONS:
                pd, ps = ld.proj[nm], ls.proj[nm]
                wd = pd.base_weight if hasattr(pd, "base_weight") else pd.weight
                ws = ps.base_weight if hasattr(ps, "base_weight") else ps.weight
                wd.copy_(ws)
                for a in range(n_adapters):
                    for dl, sl in ((pd.lora_A[a], ps.lora_A[a]), (pd.lora_B[a], ps.lora_B[a])):
                        dt = dl.weight if hasattr(dl, "weight") else dl
                        st = sl.weight if hasattr(sl, "weight") else sl
                        dt.copy_(st)


def _adapter_grads(model, n_adapters):
    out = []
    for layer in model.layers:
        for nm in D.PROJECTIONS:
            pr = layer.proj[nm]
            for a in range(n_adapters):
                for p in (pr.lora_A[a], pr.lora_B[a]):
                    g = (p.weight if hasattr(p, "weight") else p).grad
                    assert g is not None
                    out.append(g.float())
    return out


@pytest.mark.gpu
def test_tiny_decoder_fused_as_accurate_as_unfused_torch():
    """Fused bf16 decoder and the unfused bf16 torch decoder, both against an fp32 torch
    decoder with the same (bf16-representable) weights: the fused adapter gradients are no
    further from fp32 than the unfused bf16 path's, tensor by tensor."""
    dev = torch.device("cuda", 0)
    adapters = [AdapterConfig(8, 2.0, 0.0, 1), AdapterConfig(16, 2.0, 0.0, 2), AdapterConfig(32, 1.5, 0.0, 3)]
    na = len(adapters)
    fused = D.LoRADecoder(TINY, adapters, fused=True, device=dev,
                          generator=torch.Generator(device=dev).manual_seed(0), max_pos=512)
    with torch.no_grad():  # bf16-representable fp32 masters, so every model starts identical
        for p in fused.adapter_parameters():
            p.copy_(p.to(torch.bfloat16).float())
    ref_bf16 = D.LoRADecoder(TINY, adapters, fused=False, device=dev, max_pos=512,
                             generator=torch.Generator(device=dev).manual_seed(1))
    ref_f32 = D.LoRADecoder(TINY, adapters, fused=False, device=dev, max_pos=512, dtype=torch.float32,
                            attention="sdpa", generator=torch.Generator(device=dev).manual_seed(2))
    _copy_weights(ref_bf16, fused, na)
    _copy_weights(ref_f32, fused, na)
    pm = D.pack_microbatch(_tiny_plan(), TINY.vocab, dev, torch.Generator().manual_seed(3))
    losses = [float(D.train_step(m, [pm])) for m in (fused, ref_bf16, ref_f32)]
    torch.cuda.synchronize()
    assert all(math.isfinite(v) for v in losses)
    assert abs(losses[0] - losses[2]) <= 1e-2 * abs(losses[2]), losses
    g_f, g_b, g_32 = (_adapter_grads(m, na) for m in (fused, ref_bf16, ref_f32))
    e_f = [float((a - c).norm() / c.norm()) for a, c in zip(g_f, g_32)]
    e_b = [float((b - c).norm() / c.norm()) for b, c in zip(g_b, g_32)]
    med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
    print("adapter grads vs fp32: fused median %.2e max %.2e | unfused bf16 median %.2e max %.2e"
          % (med(e_f), max(e_f), med(e_b), max(e_b)))
    assert med(e_f) <= 1.25 * med(e_b) + 2e-3
    assert all(ef <= 2.0 * eb + 1e-2 for ef, eb in zip(e_f, e_b))


# two runs of the same step differ in fp32 red.add order, which can flip the bf16 rounding of
# a stored dŜ element and move whole gradient rows by one ulp: SPEC.md §5's end-to-end bound
GRAD_RTOL = 4e-3


@pytest.mark.gpu
def test_graphed_train_step_matches_eager():
    """GraphedTrainStep (per-microbatch CUDA graphs sharing one pool) gives the eager step's
    losses and accumulated adapter gradients (p = 0, so no mask-stream difference)."""
    dev = torch.device("cuda", 0)
    adapters = [AdapterConfig(8, 2.0, 0.0, 1), AdapterConfig(16, 2.0, 0.0, 2), AdapterConfig(32, 1.5, 0.0, 3)]
    mk = lambda cap: D.LoRADecoder(TINY, adapters, fused=True, device=dev, max_pos=512, capturable=cap,  # noqa: E731
                                   generator=torch.Generator(device=dev).manual_seed(0))
    eager, graphed = mk(False), mk(True)
    mbs = [D.pack_microbatch(_tiny_plan(), TINY.vocab, dev, torch.Generator().manual_seed(s)) for s in (3, 4)]
    loss_e = D.train_step(eager, mbs)
    step = D.GraphedTrainStep(graphed, mbs, warmup=1)
    loss_g = step()
    torch.cuda.synchronize()
    assert abs(float(loss_g) - float(loss_e)) <= 1e-3 * abs(float(loss_e))
    for pe, pg in zip(eager.adapter_parameters(), graphed.adapter_parameters()):
        assert pg.grad is not None
        rel = float((pg.grad - pe.grad).norm() / pe.grad.norm().clamp_min(1e-12))
        assert rel < GRAD_RTOL, rel
    # a second replay overwrites (first graph) and re-accumulates: same gradients again
    step()
    torch.cuda.synchronize()
    for pe, pg in zip(eager.adapter_parameters(), graphed.adapter_parameters()):
        rel = float((pg.grad - pe.grad).norm() / pe.grad.norm().clamp_min(1e-12))
        assert rel < GRAD_RTOL, rel
