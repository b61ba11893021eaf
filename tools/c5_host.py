"""Host enqueue time vs device time of one C5 decoder microbatch (is the decoder host-bound?).

    python tools/c5_host.py [--layers 4]
"""
from __future__ import annotations

import argparse
import dataclasses
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--fused", action=argparse.BooleanOptionalAction, default=True)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2510_00206_b200 import decoder as D

    dev = torch.device("cuda")
    shape = dataclasses.replace(D.LLAMA31_8B, layers=args.layers)
    adapters, chosen, assign = bench.c5_microbatches(1, 1)
    pm = D.pack_microbatch(chosen[0], shape.vocab, dev, torch.Generator().manual_seed(0))
    model = D.LoRADecoder(shape, adapters, fused=args.fused, device=dev,
                          generator=torch.Generator(device=dev).manual_seed(1))
    for _ in range(3):
        D.train_step(model, [pm])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        D.train_step(model, [pm])
    t_enq = (time.perf_counter() - t0) / 5
    e1.record()
    torch.cuda.synchronize()
    t_all = (time.perf_counter() - t0) / 5
    print(f"fused={args.fused} layers={args.layers} rows={pm.rows}: host enqueue {t_enq * 1e3:.1f} ms, "
          f"wall {t_all * 1e3:.1f} ms, device {e0.elapsed_time(e1) / 5:.1f} ms per microbatch")


if __name__ == "__main__":
    main()
