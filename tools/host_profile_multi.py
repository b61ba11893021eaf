"""cProfile of the FusedMultiLoRA host path (4 adapters, 5 segments): where the enqueue time goes.

    python tools/host_profile_multi.py
"""
from __future__ import annotations

import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2510_00206_b200 import AdapterConfig, FusedMultiLoRA, Segment

    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    m, k, n = 8192, 4096, 4096
    w = (torch.randn(n, k, device=dev, generator=g) / 64).to(torch.bfloat16)
    ads = [AdapterConfig(8, 2.0, 0.0, 1), AdapterConfig(16, 2.0, 0.05, 2), AdapterConfig(32, 2.0, 0.1, 3),
           AdapterConfig(64, 2.0, 0.1, 4)]
    layer = FusedMultiLoRA(w, ads, init="gaussian", generator=g)
    segs = [Segment(0, 0, 1600), Segment(1, 1600, 4000), Segment(1, 4000, 6144, 1), Segment(2, 6144, 6464),
            Segment(3, 6464, 8192)]
    x = torch.randn(m, k, device=dev, generator=g).to(torch.bfloat16).requires_grad_(True)
    dy = torch.randn(m, n, device=dev, generator=g).to(torch.bfloat16)

    def step():
        for p in layer.parameters():
            p.grad = None
        x.grad = None
        layer(x, segs).backward(dy)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(50):
        step()
    print(f"host enqueue per fwd+bwd: {(time.perf_counter() - t) / 50 * 1e6:.0f} us")
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        step()
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
