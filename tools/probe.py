"""Kernel-by-kernel GPU probe: runs each launcher in isolation against the oracle and
prints one JSON line per case (errors instead of assertions), each case in its own
subprocess so a trapped kernel cannot take the others down.

    python tools/probe.py            # all cases
    python tools/probe.py --case down
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CASES = {
    # name: (m, k, n, ranks, lengths, ps)
    "plain": (256, 512, 512, (), (), ()),
    "plain_odd": (200, 136, 264, (), (), ()),
    "single_p0": (256, 512, 384, (16,), (256,), (0.0,)),
    "single_p1": (256, 512, 384, (16,), (256,), (0.1,)),
    "single_r32": (384, 256, 512, (32,), (384,), (0.0,)),
    "single_odd": (130, 72, 200, (8,), (130,), (0.1,)),
    "multi4": (1024, 512, 512, (8, 16, 32, 64), (448, 304, 176, 96), (0.0, 0.05, 0.1, 0.1)),
    "multi_gap": (640, 256, 256, (16, 16), (100, 300), (0.1, 0.0)),
    "c1": (2048, 4096, 4096, (16,), (2048,), (0.1,)),
}


def run_case(name: str) -> dict:
    import numpy as np
    import torch

    import harness as H
    from oracle import lora as olora
    from paper_2510_00206_b200 import _lib

    m, k, n, ranks, lengths, ps = CASES[name]
    case = H.Case(m, k, n, ranks, lengths, tuple(2.0 for _ in ranks), ps, tuple(1234 + i for i in range(len(ranks))))
    x, w, dy, a_list, b_list = H.make_inputs(case)
    res = {"case": name}
    lib = _lib.load()
    dev = torch.device("cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    if not ranks:
        p, routes, ws, R = H.make_problem(case, dev)
        xd, wd, dyd = x.to(dev), w.to(dev), dy.to(dev)
        y = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
        dx = torch.empty((m, k), dtype=torch.bfloat16, device=dev)
        _lib.check(lib.lf_base_fwd(ctypes.byref(p), P(xd), P(wd), None, None, P(y), st), "base_fwd")
        torch.cuda.synchronize()
        ref = (x.float() @ w.float().T)
        res["y_relfro"] = olora.rel_fro(y.float().cpu().numpy(), ref.numpy())
        _lib.check(lib.lf_grad_input(ctypes.byref(p), P(dyd), P(wd), None, None, P(dx), st), "grad_input")
        torch.cuda.synchronize()
        ref = (dy.float() @ w.float())
        res["dx_relfro"] = olora.rel_fro(dx.float().cpu().numpy(), ref.numpy())
        return res
    a_cat, b_cat = H.cat_weights(case, a_list, b_list)
    t0 = time.time()
    o = H.run_oracle(case, x, w, dy, a_cat, b_cat)
    res["oracle_s"] = round(time.time() - t0, 2)
    # routes + mask
    segs, R = H.oracle_segments(case)
    from oracle import routing as orouting
    ref_routes = orouting.routes([(s.row_start, s.row_end) for s in segs], [(s.col_start, s.rank) for s in segs], m)
    p, routes, ws, R = H.make_problem(case, dev)
    _lib.check(lib.lf_build_routes(ctypes.byref(p), P(routes), st), "routes")
    keep = torch.empty((m, k), dtype=torch.uint8, device=dev)
    _lib.check(lib.lf_dropout_mask(ctypes.byref(p), P(keep), st), "mask")
    torch.cuda.synchronize()
    res["routes_exact"] = bool(np.array_equal(routes.cpu().numpy(), ref_routes))
    res["mask_exact"] = bool(np.array_equal(keep.cpu().numpy(), o["keep"]))
    out = H.run_device(case, x, w, dy, a_cat, b_cat)
    for key in ("s_hat", "y", "ds", "db", "da", "dx"):
        res[key + "_relfro"] = olora.rel_fro(out[key], o[key])
    res["ws_clean"] = out["ws_clean"]
    if any(p > 0 for p in ps):  # packed-mask path: ① writes bits, ④/⑤ read them
        out = H.run_device(case, x, w, dy, a_cat, b_cat, use_bits=True)
        for key in ("s_hat", "da", "dx"):
            res[key + "_bits_relfro"] = olora.rel_fro(out[key], o[key])
    # module API end to end (autograd, fp32 master adapter weights)
    if len(ranks) == 1 and lengths[0] == m:
        from paper_2510_00206_b200 import fused_lora

        xd = x.to(dev).requires_grad_(True)
        a = a_list[0].to(dev).float().requires_grad_(True)
        b = b_list[0].to(dev).float().requires_grad_(True)
        y = fused_lora(xd, w.to(dev), a, b, 2.0, ps[0], seed=case.seeds[0], offset=case.offset)
        y.backward(dy.to(dev))
        torch.cuda.synchronize()
        r0 = ranks[0]
        res["api_y_relfro"] = olora.rel_fro(y.detach().float().cpu().numpy(), o["y"])
        res["api_dx_relfro"] = olora.rel_fro(xd.grad.float().cpu().numpy(), o["dx"])
        res["api_da_relfro"] = olora.rel_fro(a.grad.cpu().numpy(), o["da"][:r0])
        res["api_db_relfro"] = olora.rel_fro(b.grad.cpu().numpy(), o["db"][:, :r0])
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default=None)
    ap.add_argument("--timeout", type=int, default=120)
    args = ap.parse_args()
    if args.case:
        try:
            print(json.dumps(run_case(args.case)), flush=True)
        except Exception as e:  # report, do not hide
            print(json.dumps({"case": args.case, "error": f"{type(e).__name__}: {e}"[:2000]}), flush=True)
            sys.exit(1)
        return
    for name in CASES:
        try:
            r = subprocess.run([sys.executable, __file__, "--case", name], capture_output=True, text=True,
                               timeout=args.timeout)
            line = (r.stdout.strip().splitlines() or [""])[-1]
            print(line if line else json.dumps({"case": name, "rc": r.returncode, "stderr": r.stderr[-1500:]}),
                  flush=True)
        except subprocess.TimeoutExpired:
            print(json.dumps({"case": name, "error": "timeout"}), flush=True)


if __name__ == "__main__":
    main()
