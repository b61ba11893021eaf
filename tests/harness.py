"""Shared test harness: seeded inputs, the oracle, and direct C-ABI runs of each kernel."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from oracle import lora as olora
from oracle import philox as ophilox
from oracle import routing as orouting


@dataclass
class Case:
    m: int
    k: int
    n: int
    ranks: tuple  # adapter rank per segment
    lengths: tuple  # rows per segment
    scalings: tuple
    ps: tuple
    seeds: tuple
    offset: int = 7
    gap_rows: int = 0  # rows after the last segment that belong to no adapter


def make_inputs(case: Case, seed: int = 0):
    """Seeded bf16 inputs (SURVEY.md §8(d) distributions), as float32 numpy bf16-exact arrays."""
    g = torch.Generator().manual_seed(seed)
    m, k, n = case.m, case.k, case.n
    x = torch.randn(m, k, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, generator=g) / k**0.5).to(torch.bfloat16)
    dy = torch.randn(m, n, generator=g).to(torch.bfloat16)
    a_list, b_list = [], []
    for r in case.ranks:
        a_list.append(((torch.rand(r, k, generator=g) * 2 - 1) / k**0.5).to(torch.bfloat16))
        b_list.append((torch.randn(n, r, generator=g) / r**0.5).to(torch.bfloat16))
    return x, w, dy, a_list, b_list


def oracle_segments(case: Case):
    segs, row, col = [], 0, 0
    for r, L, s, p, sd in zip(case.ranks, case.lengths, case.scalings, case.ps, case.seeds):
        rp = orouting.pad_rank(r)
        segs.append(olora.OracleSegment(row, row + L, col, rp, s, p, sd))
        row += L
        col += rp
    return segs, col


def cat_weights(case: Case, a_list, b_list):
    """A_cat (R,k) / B_cat (n,R) with zero padding of each block to a multiple of 16."""
    a_blocks, b_blocks = [], []
    for r, a, b in zip(case.ranks, a_list, b_list):
        rp = orouting.pad_rank(r)
        a_blocks.append(torch.nn.functional.pad(a.float(), (0, 0, 0, rp - r)))
        b_blocks.append(torch.nn.functional.pad(b.float(), (0, rp - r)))
    return torch.cat(a_blocks, 0).to(torch.bfloat16), torch.cat(b_blocks, 1).to(torch.bfloat16)


def oracle_keep(case: Case, segs):
    class _A:
        def __init__(self, p, seed):
            self.dropout_p, self.seed = p, seed

    adapters = [_A(s.dropout_p, s.seed) for s in segs]
    return ophilox.keep_mask(case.m, case.k, [(i, s.row_start, s.row_end) for i, s in enumerate(segs)], adapters,
                             case.offset)


def run_oracle(case: Case, x, w, dy, a_cat, b_cat, keep=None):
    segs, _ = oracle_segments(case)
    if keep is None:
        keep = oracle_keep(case, segs)
    xf, wf, dyf = x.float().numpy(), w.float().numpy(), dy.float().numpy()
    af, bf = a_cat.float().numpy(), b_cat.float().numpy()
    y, s_hat = olora.forward(xf, wf, af, bf, segs, keep)
    dx, da, db, ds = olora.backward(dyf, xf, wf, af, bf, s_hat, segs, keep)
    return dict(y=y, s_hat=s_hat, dx=dx, da=da, db=db, ds=ds, keep=keep)


def make_problem(case: Case, device, keep_mask=None, use_bits=False):
    from paper_2510_00206_b200 import _lib

    segs, R = oracle_segments(case)
    p = _lib.LfProblem()
    p.m, p.k, p.n = case.m, case.k, case.n
    p.rank_total = R
    p.num_segments = len(segs)
    for i, s in enumerate(segs):
        d = p.segments[i]
        d.row_start, d.row_end, d.col_start, d.rank = s.row_start, s.row_end, s.col_start, s.rank
        d.scaling, d.dropout_p, d.seed, d.offset = s.scaling, s.dropout_p, s.seed, case.offset
    routes = torch.empty((-(-case.m // 128), 4), dtype=torch.int32, device=device)
    ws = torch.zeros(_lib.workspace_bytes(case.m, R) + 4096, dtype=torch.uint8, device=device)
    p.routes = routes.data_ptr()
    p.workspace = ws.data_ptr()
    p.workspace_bytes = ws.numel()
    p.keep_mask = keep_mask.data_ptr() if keep_mask is not None else None
    bits = None
    if use_bits:
        bits = torch.full((case.m, case.k // 8), 0xAA, dtype=torch.uint8, device=device)
        p.keep_bits = bits.data_ptr()
    p._bits_ref = bits  # keep alive
    return p, routes, ws, R


def run_device(case: Case, x, w, dy, a_cat, b_cat, keep_mask=None, device="cuda", use_bits=False):
    """Run all five launchers through the C ABI; returns every intermediate on the host."""
    from paper_2510_00206_b200 import _lib

    lib = _lib.load()
    dev = torch.device(device)
    p, routes, ws, R = make_problem(case, dev, keep_mask, use_bits)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    xd, wd, dyd = x.to(dev).contiguous(), w.to(dev).contiguous(), dy.to(dev).contiguous()
    ad, bd = a_cat.to(dev).contiguous(), b_cat.to(dev).contiguous()
    m, k, n = case.m, case.k, case.n
    s_hat = torch.full((m, R), float("nan"), dtype=torch.bfloat16, device=dev)
    y = torch.full((m, n), float("nan"), dtype=torch.bfloat16, device=dev)
    ds = torch.full((m, R), float("nan"), dtype=torch.bfloat16, device=dev)
    db = torch.zeros((n, R), dtype=torch.float32, device=dev)
    da = torch.zeros((R, k), dtype=torch.float32, device=dev)
    dx = torch.full((m, k), float("nan"), dtype=torch.bfloat16, device=dev)
    pp = ctypes.byref(p)
    _lib.check(lib.lf_build_routes(pp, P(routes), st), "routes")
    _lib.check(lib.lf_dropout_down_fwd(pp, P(xd), P(ad), P(s_hat), st), "down")
    _lib.check(lib.lf_base_fwd(pp, P(xd), P(wd), P(s_hat), P(bd), P(y), st), "base_fwd")
    _lib.check(lib.lf_grad_up(pp, P(dyd), P(bd), P(s_hat), P(ds), P(db), st), "grad_up")
    _lib.check(lib.lf_grad_down(pp, P(xd), P(ds), P(da), st), "grad_down")
    _lib.check(lib.lf_grad_input(pp, P(dyd), P(wd), P(ds), P(ad), P(dx), st), "grad_input")
    torch.cuda.synchronize()
    ws_clean = bool((ws == 0).all().item())
    out = dict(y=y, s_hat=s_hat, ds=ds, db=db, da=da, dx=dx, routes=routes)
    out = {kk: v.float().cpu().numpy() if v.dtype != torch.int32 else v.cpu().numpy() for kk, v in out.items()}
    out["ws_clean"] = ws_clean
    return out


def assert_within_ulps(got, ref, name, ulps=1.0):
    """Stored bf16 intermediates (Ŝ, dŜ): within `ulps` bf16 ulp of the oracle — the fp32
    accumulation order of a kernel may flip the final rounding, never more."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (name, got.shape, ref.shape)
    assert np.isfinite(got).all(), f"{name}: non-finite values"
    # absolute floor for values born of cancellation: fp32-vs-fp64 summation error of the
    # terms is ~2^-24 of their magnitude, far below 2^-12 of the tensor's rms
    rms = float(np.sqrt(np.mean(ref**2))) if ref.size else 0.0
    tol = ulps * np.maximum(olora.bf16_ulp(ref), olora.bf16_ulp(got)) + 2.0**-12 * rms + 1e-30
    bad = np.abs(got - ref) > tol
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(f"{name}: {int(bad.sum())}/{bad.size} elements differ by more than {ulps} bf16 ulp; "
                             f"first {idx.tolist()} got {[got[tuple(i)] for i in idx]} "
                             f"ref {[ref[tuple(i)] for i in idx]}")


def check_chain(out, ref, x, w, dy, a_cat, b_cat, keep, tag):
    """SPEC.md §5 parity of all five kernels.

    Each kernel is checked against the oracle applied to the SAME inputs the kernel saw
    (so a legitimate one-ulp flip of a stored bf16 intermediate upstream cannot fail a
    downstream check), and the whole chain end to end against the pure oracle."""
    xf, wf, dyf = x.float().numpy(), w.float().numpy(), dy.float().numpy()
    af, bf = a_cat.float().numpy(), b_cat.float().numpy()
    assert_within_ulps(out["s_hat"], ref["s_hat"], f"{tag}:s_hat")  # ①
    assert_within_ulps(out["ds"], ref["ds"], f"{tag}:ds")  # ③ (dŜ)
    y_given = olora.base_forward(xf, wf, out["s_hat"], bf)  # ② on the device Ŝ
    assert_close_bf16(out["y"], y_given, f"{tag}:y")
    dx_g, da_g, db_g = olora.grads_given(dyf, xf, wf, af, out["s_hat"], out["ds"], keep)
    assert_close_bf16(out["db"], db_g, f"{tag}:db")  # ③ (dB)
    assert_close_bf16(out["da"], da_g, f"{tag}:da")  # ④
    assert_close_bf16(out["dx"], dx_g, f"{tag}:dx")  # ⑤
    for key in ("y", "dx", "da", "db", "s_hat", "ds"):  # end to end vs the pure oracle
        rf = olora.rel_fro(out[key], ref[key])
        assert rf <= 4e-3, f"{tag}:{key} end-to-end relative Frobenius error {rf:.3e}"


def assert_close_bf16(got, ref, name, rel_elem=2.0**-7, rel_rms=2.0**-7, rel_fro=4e-3):
    """SPEC.md §5 float tolerance: elementwise |g-o| <= rel_elem*|o| + rel_rms*rms(o),
    and ||g-o||_F / ||o||_F <= rel_fro."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    assert got.shape == ref.shape, (name, got.shape, ref.shape)
    assert np.isfinite(got).all(), f"{name}: non-finite values"
    rms = float(np.sqrt(np.mean(ref**2))) if ref.size else 0.0
    err = np.abs(got - ref)
    bound = rel_elem * np.abs(ref) + rel_rms * rms + 1e-30
    bad = err > bound
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(
            f"{name}: {int(bad.sum())}/{bad.size} elements out of tolerance; first {idx.tolist()} "
            f"got {[got[tuple(i)] for i in idx]} ref {[ref[tuple(i)] for i in idx]}"
        )
    rf = olora.rel_fro(got, ref)
    assert rf <= rel_fro, f"{name}: relative Frobenius error {rf:.3e} > {rel_fro:.1e}"


def assert_chain_close(got, ref, name):
    """End-to-end (module API) tolerance: the chained kernels may carry a one-ulp flip of a
    stored bf16 intermediate (Ŝ, dŜ) into whole output rows, so the elementwise bound is
    looser than the per-kernel one; the relative Frobenius bound of SPEC.md §5 still holds."""
    assert_close_bf16(got, ref, name, rel_elem=2.0**-5, rel_rms=2.0**-5, rel_fro=4e-3)
