"""Shared-input group GEMMs through the C ABI: lf_base_fwd_group / lf_grad_input_group against
the per-projection launches, CUDA-graph timed (one graph per variant, interleaved rounds).

    python tools/grp_bench.py --m 8192 --k 4096 --ns 4096,1024,1024 --p 0.1
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
    ap.add_argument("--ns", default="4096,1024,1024")
    ap.add_argument("--p", type=float, default=0.1)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--only", default="", help="comma-separated variants (e.g. dgrad_group)")
    args = ap.parse_args()
    import torch

    from paper_2510_00206_b200 import _lib

    lib = _lib.load()
    dev = torch.device("cuda")
    m, k, R = args.m, args.k, 16
    ns = [int(v) for v in args.ns.split(",")]
    J = len(ns)
    g = torch.Generator(device=dev).manual_seed(0)
    X = torch.randn(m, k, device=dev, generator=g).to(torch.bfloat16)
    W = [(torch.randn(n, k, device=dev, generator=g) / k**0.5).to(torch.bfloat16) for n in ns]
    A = [(torch.randn(R, k, device=dev, generator=g) / k**0.5).to(torch.bfloat16) for _ in ns]
    B = [(torch.randn(n, R, device=dev, generator=g) / 4).to(torch.bfloat16) for n in ns]
    S = [torch.randn(m, R, device=dev, generator=g).to(torch.bfloat16) for _ in ns]
    DY = [torch.randn(m, n, device=dev, generator=g).to(torch.bfloat16) for n in ns]
    Y = [torch.empty(m, n, device=dev, dtype=torch.bfloat16) for n in ns]
    DX = torch.empty(m, k, device=dev, dtype=torch.bfloat16)
    keep = []
    probs = []
    for j, n in enumerate(ns):
        p = _lib.LfProblem()
        p.m, p.k, p.n, p.rank_total, p.num_segments = m, k, n, R, 1
        s = p.segments[0]
        s.row_start, s.row_end, s.col_start, s.rank, s.scaling, s.dropout_p, s.seed, s.offset = 0, m, 0, R, 2.0, args.p, 5 + j, 1
        routes = torch.empty((-(-m // 128), 4), dtype=torch.int32, device=dev)
        ws = torch.zeros(_lib.workspace_bytes(m, R), dtype=torch.uint8, device=dev)
        bits = torch.zeros((m, k // 8), dtype=torch.uint8, device=dev)
        p.routes, p.workspace, p.workspace_bytes, p.keep_bits = routes.data_ptr(), ws.data_ptr(), ws.numel(), bits.data_ptr()
        keep += [routes, ws, bits]
        probs.append(p)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for j, p in enumerate(probs):
        routes = keep[3 * j]
        _lib.check(lib.lf_build_routes(ctypes.byref(p), P(routes), st), "routes")
        _lib.check(lib.lf_dropout_down_fwd(ctypes.byref(p), P(X), P(A[j]), P(S[j]), st), "down")  # keep bits
    pp = (ctypes.POINTER(_lib.LfProblem) * J)(*[ctypes.pointer(p) for p in probs])
    arr = lambda ts: (ctypes.c_void_p * J)(*[t.data_ptr() for t in ts])  # noqa: E731

    def fwd_sep(s_):
        for j, p in enumerate(probs):
            _lib.check(lib.lf_base_fwd(ctypes.byref(p), P(X), P(W[j]), P(S[j]), P(B[j]), P(Y[j]), s_), "fwd")

    def fwd_grp(s_):
        _lib.check(lib.lf_base_fwd_group(pp, J, P(X), arr(W), arr(S), arr(B), arr(Y), s_), "fwd_group")

    def dg_sep(s_):
        for j, p in enumerate(probs):
            f = lib.lf_grad_input if j == 0 else lib.lf_grad_input_accum
            _lib.check(f(ctypes.byref(p), P(DY[j]), P(W[j]), P(S[j]), P(A[j]), P(DX), s_), "dgrad")

    def dg_grp(s_):
        _lib.check(lib.lf_grad_input_group(pp, J, arr(DY), arr(W), arr(S), arr(A), P(DX), s_), "dgrad_group")

    variants = {"fwd_separate": fwd_sep, "fwd_group": fwd_grp, "dgrad_separate": dg_sep, "dgrad_group": dg_grp}
    if args.only:
        variants = {k_: v_ for k_, v_ in variants.items() if k_ in args.only.split(",")}
    flops = {"fwd": 2 * m * k * sum(ns), "dgrad": 2 * m * k * sum(ns)}
    graphs = {}
    for name, fn in variants.items():
        fn(st)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            s2 = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            for _ in range(args.iters):
                fn(s2)
        graphs[name] = gr
    for rnd in range(args.rounds):
        for name, gr in graphs.items():
            gr.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gr.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / args.iters
            print(json.dumps({"variant": name, "m": m, "k": k, "ns": ns, "p": args.p, "round": rnd, "us": round(us, 1),
                              "tflops": round(flops[name.split("_")[0]] / (us * 1e-6) / 1e12, 1)}), flush=True)


if __name__ == "__main__":
    main()
