"""Host (Python + C ABI) enqueue cost vs device time of one FusedLoRA fwd+bwd step.

    python tools/host_overhead.py [--m 2048 --k 4096 --n 4096]

A step is host-bound when enqueue_us >= device_us: the GPU then idles between kernels.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=2048)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--p", type=float, default=0.1)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--profile", action="store_true", help="cProfile the fused arm's host path")
    args = ap.parse_args()
    import torch

    from paper_2510_00206_b200 import FusedLoRA, unfused_lora

    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    w = (torch.randn(args.n, args.k, device=dev, generator=g) / args.k**0.5).to(torch.bfloat16)
    layer = FusedLoRA(w, rank=16, scaling=2.0, dropout_p=args.p, seed=1, init="gaussian", generator=g)
    x = torch.randn(args.m, args.k, device=dev, generator=g).to(torch.bfloat16).requires_grad_(True)
    dy = torch.randn(args.m, args.n, device=dev, generator=g).to(torch.bfloat16)
    a = layer.lora_A.weight.detach().to(torch.bfloat16).requires_grad_(True)
    b = layer.lora_B.weight.detach().to(torch.bfloat16).requires_grad_(True)

    def fused():
        for p_ in layer.parameters():
            p_.grad = None
        x.grad = None
        layer(x).backward(dy)

    def unfused():
        a.grad = b.grad = x.grad = None
        unfused_lora(x, w, a, b, 2.0, args.p).backward(dy)

    if args.profile:
        import cProfile
        import pstats

        for _ in range(5):
            fused()
        torch.cuda.synchronize()
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(args.iters):
            fused()
        pr.disable()
        torch.cuda.synchronize()
        pstats.Stats(pr).sort_stats("tottime").print_stats(30)
        return
    for name, fn in (("fused", fused), ("unfused", unfused)):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            fn()
        t_enq = time.perf_counter() - t0
        e1.record()
        torch.cuda.synchronize()
        t_all = time.perf_counter() - t0
        # device time with a host-free stream: enqueue far ahead first (blocking wait kernel)
        print(json.dumps({"arm": name, "m": args.m, "k": args.k, "n": args.n,
                          "enqueue_us": round(t_enq / args.iters * 1e6, 1),
                          "wall_us": round(t_all / args.iters * 1e6, 1),
                          "event_us": round(e0.elapsed_time(e1) / args.iters * 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
