"""CUDA-graph capture of fused LoRA steps (capturable=True: device-side Philox step counter).

A captured forward+backward replays with the same results as the eager path at the same
Philox offset, and each replay draws a fresh dropout mask (SPEC.md §3)."""
from __future__ import annotations

import pytest
import torch

from paper_2510_00206_b200 import AdapterConfig, FusedLoRA, FusedMultiLoRA, segments_from_lengths
from paper_2510_00206_b200.graphs import GraphedStep

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _close(a, b, tol=2e-3):
    a, b = a.detach().float(), b.detach().float()
    return float((a - b).norm() / b.norm().clamp_min(1e-12)) <= tol


def test_graphed_fused_lora_matches_eager_offset_and_redraws_mask():
    g = torch.Generator(device=DEV).manual_seed(0)
    m, k, n, r = 640, 512, 384, 16
    w = (torch.randn(n, k, device=DEV, generator=g) / k**0.5).to(torch.bfloat16)
    x = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16).requires_grad_(True)
    dy = torch.randn(m, n, device=DEV, generator=g).to(torch.bfloat16)
    cap = FusedLoRA(w, rank=r, scaling=2.0, dropout_p=0.1, seed=9, init="gaussian", capturable=True, dropout_rng="counter",
                    generator=torch.Generator(device=DEV).manual_seed(1))
    ref = FusedLoRA(w, rank=r, scaling=2.0, dropout_p=0.1, seed=9, init="gaussian", dropout_rng="counter",
                    generator=torch.Generator(device=DEV).manual_seed(1))

    def step():
        cap.lora_A.weight.grad = cap.lora_B.weight.grad = x.grad = None
        y = cap(x)
        y.backward(dy)
        return y.detach()

    graphed = GraphedStep(step, warmup=3)  # warm-up runs offsets 1..3; capture runs nothing
    outs = []
    for _ in range(2):
        y = graphed.replay()
        torch.cuda.synchronize()
        outs.append((y.clone(), cap.lora_A.weight.grad.clone(), cap.lora_B.weight.grad.clone(), x.grad.clone()))
    assert int(cap.step_counter.item()) == 5
    # eager, host offsets 4 and 5 = the two replays
    for i, off in enumerate((4, 5)):
        ref._offset = off
        x.grad = None
        ref.lora_A.weight.grad = ref.lora_B.weight.grad = None
        y = ref(x)
        y.backward(dy)
        torch.cuda.synchronize()
        got = outs[i]
        assert _close(got[0], y) and _close(got[1], ref.lora_A.weight.grad) and _close(got[2], ref.lora_B.weight.grad)
        assert _close(got[3], x.grad)
    # a fresh mask per replay: the two dA differ well beyond accumulation-order noise
    assert not _close(outs[0][1], outs[1][1], tol=5e-2)


def test_graphed_multi_lora_replays_track_weight_updates():
    """capturable multi-adapter layers read persistent bf16 rank-concat copies of the fp32
    master weights: an in-place update between replays is re-copied before the next replay."""
    g = torch.Generator(device=DEV).manual_seed(2)
    m, k, n = 768, 256, 256
    w = (torch.randn(n, k, device=DEV, generator=g) / k**0.5).to(torch.bfloat16)
    ads = [AdapterConfig(8, 2.0, 0.0, 1), AdapterConfig(32, 1.0, 0.0, 2)]
    layer = FusedMultiLoRA(w, ads, init="gaussian", capturable=True, generator=g)
    x = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16)
    segs = segments_from_lengths([0, 1], [320, 448])
    dy = torch.randn(m, n, device=DEV, generator=g).to(torch.bfloat16)

    def step():
        for p in layer.parameters():
            p.grad = None
        y = layer(x, segs)
        y.backward(dy)
        return y.detach()

    graphed = GraphedStep(step)
    y0 = graphed.replay().clone()
    with torch.no_grad():
        layer.lora_B[1].weight.mul_(3.0)
    y1 = graphed.replay().clone()
    eager = layer(x, segs).detach()
    torch.cuda.synchronize()
    assert not _close(y1, y0, tol=1e-2)
    assert _close(y1, eager)


def test_graphed_fused_lora_sees_optimizer_and_inplace_updates():
    """Capturable FusedLoRA reads persistent bf16 operand copies inside the graph; they are
    refreshed by every optimizer step (fused AdamW included: no version bump) and, before a
    replay, for parameters changed in place."""
    g = torch.Generator(device=DEV).manual_seed(5)
    m, k, n = 512, 256, 384
    w = (torch.randn(n, k, device=DEV, generator=g) / 16).to(torch.bfloat16)
    cap = FusedLoRA(w, rank=16, dropout_p=0.0, init="gaussian", capturable=True, generator=g)
    ref = FusedLoRA(w, rank=16, dropout_p=0.0, init="gaussian")
    x = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16)
    opt = torch.optim.AdamW(cap.parameters(), lr=1e-2, fused=True)

    def step():
        y = cap(x)
        y.float().square().mean().backward()
        return y.detach()

    graphed = GraphedStep(step, warmup=2)

    def check():
        y = graphed.replay()
        with torch.no_grad():
            ref.lora_A.weight.copy_(cap.lora_A.weight)
            ref.lora_B.weight.copy_(cap.lora_B.weight)
            ref.invalidate_operands()
            assert torch.equal(y, ref(x))

    check()
    for _ in range(2):
        opt.step()  # post-hook refreshes the copies
        opt.zero_grad(set_to_none=False)
        check()
    with torch.no_grad():
        cap.lora_B.weight.mul_(2.0)  # in place: version bump, refreshed before the replay
    check()


def test_graphed_multi_lora_sees_optimizer_updates_bitwise():
    """Capturable FusedMultiLoRA (ranks 8 / 32 / 16: padded and unpadded column blocks) reads
    persistent rank-concat copies inside the graph — no cast, pad or concatenation per call —
    refreshed by every optimizer step and by invalidate_operands(); the graphed step matches
    a non-capturable layer with the same weights bit for bit."""
    g = torch.Generator(device=DEV).manual_seed(9)
    m, k, n = 640, 256, 384
    w = (torch.randn(n, k, device=DEV, generator=g) / 16).to(torch.bfloat16)
    ads = [AdapterConfig(8, 2.0, 0.0, 1), AdapterConfig(32, 1.0, 0.0, 2), AdapterConfig(16, 0.5, 0.0, 3)]
    cap = FusedMultiLoRA(w, ads, init="gaussian", capturable=True, generator=g)
    ref = FusedMultiLoRA(w, ads, init="gaussian")
    x = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16)
    segs = segments_from_lengths([0, 1, 2], [128, 256, 256])
    opt = torch.optim.AdamW(cap.parameters(), lr=1e-2, fused=True)

    def step():
        y = cap(x, segs)
        y.float().square().mean().backward()
        return y.detach()

    graphed = GraphedStep(step, warmup=2)

    def check():
        y = graphed.replay()
        with torch.no_grad():
            for pr, pc in zip(ref.parameters(), cap.parameters()):
                pr.copy_(pc)
            ref.invalidate_operands()
            assert torch.equal(y, ref(x, segs))

    check()
    for _ in range(2):
        opt.step()
        opt.zero_grad(set_to_none=False)
        check()
    with torch.no_grad():
        cap.lora_A[0].weight.data.mul_(-1.0)  # through .data: no version bump
    cap.invalidate_operands()
    check()


def test_capture_with_a_layout_first_seen_inside_the_graph():
    """A capturable multi-adapter layer whose column-block layout is first seen during a
    capture gathers its operands inside the graph (no persistent copy is created mid-capture)
    and the replay equals the eager layer; a later eager call creates the persistent copy."""
    g = torch.Generator(device=DEV).manual_seed(12)
    m, k, n = 512, 256, 256
    w = (torch.randn(n, k, device=DEV, generator=g) / 16).to(torch.bfloat16)
    ads = [AdapterConfig(8, 2.0, 0.0, 1), AdapterConfig(32, 1.0, 0.0, 2)]
    layer = FusedMultiLoRA(w, ads, init="gaussian", capturable=True, generator=g)
    x = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16)
    warm_segs = segments_from_lengths([1], [m])  # layout {adapter 1}
    new_segs = segments_from_lengths([0, 1], [256, 256])  # layout {0, 1}: first seen in the capture
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side), torch.no_grad():
        layer(x, warm_segs)
    torch.cuda.current_stream().wait_stream(side)
    n_before = len(layer._operands._d)
    graph = torch.cuda.CUDAGraph()
    with torch.no_grad(), torch.cuda.graph(graph):
        y = layer(x, new_segs)
    assert len(layer._operands._d) == n_before  # nothing persistent created inside the capture
    graph.replay()
    with torch.no_grad():
        ref = layer(x, new_segs)
    torch.cuda.synchronize()
    assert torch.equal(y, ref)
    assert len(layer._operands._d) == n_before + 1
