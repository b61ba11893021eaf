"""Per-launcher microbenchmark through the C ABI (CUDA events, rotating inputs > L2).

    python tools/kbench.py --m 8192 --k 4096 --n 4096 --r 16 --p 0.1 [--bits]

Prints one JSON line per launcher: µs per call, algorithmic GB/s (memory-bound kernels)
or TFLOP/s (GEMMs).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--r", type=int, default=16)
    ap.add_argument("--p", type=float, default=0.1)
    ap.add_argument("--bits", action="store_true", help="① writes packed keep bits, ④/⑤ read them")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default="")
    ap.add_argument("--rounds", type=int, default=1, help="repeat the kernel list (A/B interleaving under the power cap)")
    ap.add_argument("--power", action="store_true", help="sample SM clock and board power (NVML) per timed loop")
    ap.add_argument("--graph", action="store_true",
                    help="capture the timed loop as one CUDA graph (GPU time without the per-call host cost)")
    args = ap.parse_args()
    import torch

    from paper_2510_00206_b200 import _lib

    lib = _lib.load()
    dev = torch.device("cuda")
    m, k, n, r = args.m, args.k, args.n, args.r
    R = -(-r // 16) * 16
    nbuf = max(2, int(-(-300e6 // (2 * m * max(k, n)))))  # > L2 worth of activations
    g = torch.Generator(device=dev).manual_seed(0)
    X = [torch.randn(m, k, device=dev, generator=g).to(torch.bfloat16) for _ in range(nbuf)]
    DY = [torch.randn(m, n, device=dev, generator=g).to(torch.bfloat16) for _ in range(nbuf)]
    W = (torch.randn(n, k, device=dev, generator=g) / k**0.5).to(torch.bfloat16)
    A = (torch.randn(R, k, device=dev, generator=g) / k**0.5).to(torch.bfloat16)
    B = (torch.randn(n, R, device=dev, generator=g) / 4).to(torch.bfloat16)
    S = torch.randn(m, R, device=dev, generator=g).to(torch.bfloat16)
    DS = torch.randn(m, R, device=dev, generator=g).to(torch.bfloat16)
    Y = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    DX = torch.empty(m, k, device=dev, dtype=torch.bfloat16)
    DA = torch.zeros(R, k, device=dev)
    DB = torch.zeros(n, R, device=dev)
    p = _lib.LfProblem()
    p.m, p.k, p.n, p.rank_total, p.num_segments = m, k, n, R, 1
    s = p.segments[0]
    s.row_start, s.row_end, s.col_start, s.rank, s.scaling, s.dropout_p, s.seed, s.offset = 0, m, 0, R, 2.0, args.p, 5, 1
    routes = torch.empty((-(-m // 128), 4), dtype=torch.int32, device=dev)
    ws = torch.zeros(_lib.workspace_bytes(m, R), dtype=torch.uint8, device=dev)
    bits = torch.zeros((m, k // 8), dtype=torch.uint8, device=dev)
    p.routes, p.workspace, p.workspace_bytes = routes.data_ptr(), ws.data_ptr(), ws.numel()
    if args.bits:
        p.keep_bits = bits.data_ptr()
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    pp = ctypes.byref(p)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.lf_build_routes(pp, P(routes), st), "routes")
    launches = {
        "dropout_down_fwd": (lambda i: lib.lf_dropout_down_fwd(pp, P(X[i]), P(A), P(S), st),
                             "gbs", 2 * m * k + 2 * k * R + 2 * m * R),
        "base_fwd": (lambda i: lib.lf_base_fwd(pp, P(X[i]), P(W), P(S), P(B), P(Y), st),
                     "tflops", 2 * m * k * n + 2 * m * R * n),
        "grad_up": (lambda i: lib.lf_grad_up(pp, P(DY[i]), P(B), P(S), P(DS), P(DB), st),
                    "gbs", 2 * (m * n + R * n + m * R) + 2 * m * R + 4 * R * n),
        "grad_down": (lambda i: lib.lf_grad_down(pp, P(X[i]), P(DS), P(DA), st), "gbs", 2 * (m * k + m * R) + 4 * k * R),
        "grad_input": (lambda i: lib.lf_grad_input(pp, P(DY[i]), P(W), P(DS), P(A), P(DX), st),
                       "tflops", 2 * m * n * k + 2 * m * R * k),
    }
    BITS2 = torch.empty((m, k // 8), dtype=torch.uint8, device=dev)
    launches["keep_bits"] = (lambda i: lib.lf_keep_bits(pp, P(BITS2), st), "gbs", m * k // 8)
    side = torch.cuda.Stream(dev)
    s2 = ctypes.c_void_p(side.cuda_stream)
    fork, join = torch.cuda.Event(), torch.cuda.Event()

    def gemm_with_bits(i, gemm):
        """the input-free keep-bits generator on a side stream underneath a GEMM"""
        main = torch.cuda.current_stream()
        fork.record(main)
        side.wait_event(fork)
        rc = lib.lf_keep_bits(pp, P(BITS2), s2)
        rc = rc or gemm(i)
        join.record(side)
        main.wait_event(join)
        return rc

    def dgrad_with_graddown(i):
        """④ on a side stream concurrently with ⑤ (both only need dŜ)"""
        main = torch.cuda.current_stream()
        fork.record(main)
        side.wait_event(fork)
        rc = lib.lf_grad_down(pp, P(X[i]), P(DS), P(DA), s2)
        rc = rc or launches["grad_input"][0](i)
        join.record(side)
        main.wait_event(join)
        return rc

    launches["overlap_dgrad_graddown"] = (dgrad_with_graddown, "tflops", 2 * m * n * k + 2 * m * R * k)
    launches["overlap_fwd_bits"] = (lambda i: gemm_with_bits(i, launches["base_fwd"][0]), "tflops",
                                    2 * m * k * n + 2 * m * R * n)
    launches["overlap_dgrad_bits"] = (lambda i: gemm_with_bits(i, launches["grad_input"][0]), "tflops",
                                      2 * m * n * k + 2 * m * R * k)
    OUT = torch.empty_like(X[0])
    launches["torch_copy_x"] = (lambda i: (OUT.copy_(X[i]), 0)[1], "gbs", 4 * m * k)
    launches["torch_sum_x"] = (lambda i: (X[i].sum(dtype=torch.float32), 0)[1], "gbs", 2 * m * k)
    WT = W.t()
    launches["cublas_fwd"] = (lambda i: (torch.mm(X[i], WT, out=Y), 0)[1], "tflops", 2 * m * k * n)
    launches["cublas_dgrad"] = (lambda i: (torch.mm(DY[i], W, out=DX), 0)[1], "tflops", 2 * m * k * n)
    # ① once so packed bits exist for ④/⑤
    _lib.check(lib.lf_dropout_down_fwd(pp, P(X[0]), P(A), P(S), st), "down")
    sampler = _NvmlSampler() if args.power else None
    order = [nm for nm in launches if not args.only or nm in args.only.split(",")]
    if args.only:
        order = [nm for nm in args.only.split(",") if nm in launches]
    for rnd, name in [(rr, nm) for rr in range(args.rounds) for nm in order]:
        fn, unit, work = launches[name]
        for i in range(3):
            _lib.check(fn(i % nbuf), name)
        torch.cuda.synchronize()
        graph = None
        if args.graph and not name.startswith("overlap"):
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
                for i in range(args.iters):
                    fn(i % nbuf)
            st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            graph.replay()
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if sampler:
            sampler.start()
        e0.record()
        if graph is not None:
            graph.replay()
        else:
            for i in range(args.iters):
                fn(i % nbuf)
        e1.record()
        torch.cuda.synchronize()
        extra = sampler.stop() if sampler else {}
        us = e0.elapsed_time(e1) * 1e3 / args.iters
        val = work / (us * 1e-6) / (1e9 if unit == "gbs" else 1e12)
        print(json.dumps({"kernel": name, "m": m, "k": k, "n": n, "r": R, "p": args.p, "bits": args.bits,
                          "round": rnd, "us": round(us, 2), unit: round(val, 1), **extra}), flush=True)


class _NvmlSampler:
    """SM clock (MHz) and board power (W) sampled every 5 ms on a thread while a loop runs."""

    def __init__(self):
        import pynvml

        pynvml.nvmlInit()
        self.nv = pynvml
        import torch

        self.h = pynvml.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(0).uuid))

    def start(self):
        import threading

        self.samples, self.run = [], True
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def _loop(self):
        import time

        while self.run:
            self.samples.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                 self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0))
            time.sleep(0.005)

    def stop(self) -> dict:
        self.run = False
        self.t.join()
        if not self.samples:
            return {}
        clk = sorted(c for c, _ in self.samples)
        pw = sorted(p for _, p in self.samples)
        return {"sm_mhz": clk[len(clk) // 2], "power_w": round(pw[len(pw) // 2], 1), "samples": len(clk)}


if __name__ == "__main__":
    main()
