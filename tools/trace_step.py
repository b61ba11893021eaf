"""GPU timeline of one bench step (torch.profiler / CUPTI): every kernel with its duration
and the idle gap before it, grouped per kernel name.

    python tools/trace_step.py [--config c2]
"""
from __future__ import annotations

import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--unfused", action="store_true")
    ap.add_argument("--graph", action="store_true", help="profile one replay of the step captured as a CUDA graph")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench

    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(0)
    m = bench.tokens_per_gpu(args.config)
    layers, inputs, grads = bench.build_layers(args.config, m, 16, 0.1, dev, gen, capturable=args.graph)
    if args.unfused:
        base = bench.unfused_base(args.config, layers)
        step = lambda: bench.unfused_step(args.config, base, inputs, grads, 0.1)  # noqa: E731
    else:
        def step():
            bench.zero_grads(layers, inputs)
            bench.fused_step(args.config, layers, inputs, grads, 1)
    if args.graph:
        from paper_2510_00206_b200.graphs import GraphedStep

        step = GraphedStep(step, warmup=3).replay
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    import time

    # CPU issue time per step (no sync inside) vs GPU time per step
    t = time.perf_counter()
    for _ in range(10):
        step()
    cpu_issue = (time.perf_counter() - t) / 10
    torch.cuda.synchronize()
    gpu = (time.perf_counter() - t) / 10
    print(f"CPU issue time per step {cpu_issue * 1e3:.3f} ms, wall per step (10 steps, one sync) {gpu * 1e3:.3f} ms")
    import cProfile
    import pstats

    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        step()
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    kern = [e for e in evs if not e.name.startswith("Memcpy") and not e.name.startswith("Memset")] or evs
    t0 = kern[0].time_range.start
    t1 = max(e.time_range.end for e in kern)
    busy = sum(e.time_range.end - e.time_range.start for e in kern)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    prev_end = t0
    for e in kern:
        gap = max(0.0, e.time_range.start - prev_end)
        a = agg[e.name[:60] if "elementwise" not in e.name else e.name[e.name.find("<"):][:150]]
        a[0] += 1
        a[1] += e.time_range.end - e.time_range.start
        a[2] += gap
        prev_end = max(prev_end, e.time_range.end)
    print(f"step span {(t1 - t0) / 1e3:.3f} ms, kernel busy {busy / 1e3:.3f} ms, idle {(t1 - t0 - busy) / 1e3:.3f} ms, "
          f"{len(kern)} kernels")
    for name, (cnt, dur, gap) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{cnt:4d} x  busy {dur / 1e3:8.3f} ms  gaps-before {gap / 1e3:7.3f} ms  {name}")


if __name__ == "__main__":
    main()
