"""Minimal driver for ncu: a few fwd+bwd calls of one FusedLoRA layer.

    ncu --set full -k regex:lf_ -s <skip> -c <n> -o gpurun_out/prof python tools/profile_layer.py --m 8192 --k 4096 --n 4096

Warm-up iterations come first so `-s` can skip them.
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--r", type=int, default=16)
    ap.add_argument("--p", type=float, default=0.1)
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    import torch

    from paper_2510_00206_b200 import FusedLoRA

    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    w = (torch.randn(args.n, args.k, generator=g, device=dev) / args.k**0.5).to(torch.bfloat16)
    layer = FusedLoRA(w, rank=args.r, scaling=2.0, dropout_p=args.p, seed=1, init="gaussian").to(dev)
    x = torch.randn(args.m, args.k, generator=g, device=dev).to(torch.bfloat16).requires_grad_(True)
    dy = torch.randn(args.m, args.n, generator=g, device=dev).to(torch.bfloat16)
    for _ in range(args.iters):
        y = layer(x)
        y.backward(dy)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
