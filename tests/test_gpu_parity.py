"""Parity of the sm_100a kernels with the CPU oracle (SPEC.md §5 tolerances), through the
C ABI and through the public module/functional API. Needs a B200."""
from __future__ import annotations

import ctypes
import glob
import os
import zlib

import numpy as np
import pytest
import torch

import tests.harness as H
from oracle import lora as olora
from oracle import philox as ophilox
from oracle import routing as orouting

pytestmark = pytest.mark.gpu

DEV = "cuda"


def _lib():
    from paper_2510_00206_b200 import _lib

    return _lib


def _check_all(out, ref, inputs, tag):
    x, w, dy, a_cat, b_cat = inputs
    H.check_chain(out, ref, x, w, dy, a_cat, b_cat, ref["keep"], tag)


CASES = {
    "single_r16_p0": H.Case(256, 512, 384, (16,), (256,), (2.0,), (0.0,), (11,)),
    "single_r16_p01": H.Case(256, 512, 384, (16,), (256,), (2.0,), (0.1,), (12,)),
    "single_r8_odd": H.Case(130, 72, 200, (8,), (130,), (2.0,), (0.1,), (13,)),
    "single_r32": H.Case(384, 256, 520, (32,), (384,), (0.5,), (0.05,), (14,)),
    "single_r64": H.Case(200, 1024, 256, (64,), (200,), (1.0,), (0.1,), (15,)),
    "one_row": H.Case(1, 64, 64, (16,), (1,), (2.0,), (0.5,), (16,)),
    "multi4_aligned": H.Case(1024, 512, 512, (8, 16, 32, 64), (448, 304, 176, 96), (2.0,) * 4,
                             (0.0, 0.05, 0.1, 0.1), (1, 2, 3, 4)),
    "multi4_straddle_p64": H.Case(1088, 256, 264, (8, 16, 32, 64), (320, 448, 192, 128), (2.0, 1.0, 0.5, 2.0),
                                  (0.1, 0.0, 0.1, 0.2), (5, 6, 7, 8)),
    "rows_without_adapter": H.Case(640, 256, 256, (16, 16), (100, 300), (2.0, 2.0), (0.1, 0.0), (9, 10)),
    "c1": H.Case(2048, 4096, 4096, (16,), (2048,), (2.0,), (0.1,), (1234,)),
    # stream-K CTAs of ① / ④ wrap their stage rings while crossing from a p = 0 segment into
    # a p > 0 one (the masked-barrier protocol must not depend on the tile)
    "mixed_p_wrap": H.Case(4096, 4096, 128, (16, 32), (1920, 2176), (2.0, 1.0), (0.0, 0.1), (31, 32)),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("use_bits", [False, True], ids=["philox", "packed"])
def test_kernels_match_oracle(name, use_bits):
    case = CASES[name]
    x, w, dy, a_list, b_list = H.make_inputs(case, seed=zlib.crc32(name.encode()) % 1000)
    a_cat, b_cat = H.cat_weights(case, a_list, b_list)
    ref = H.run_oracle(case, x, w, dy, a_cat, b_cat)
    out = H.run_device(case, x, w, dy, a_cat, b_cat, use_bits=use_bits)
    _check_all(out, ref, (x, w, dy, a_cat, b_cat), name)
    segs, _ = H.oracle_segments(case)
    r_ref = orouting.routes([(s.row_start, s.row_end) for s in segs], [(s.col_start, s.rank) for s in segs], case.m)
    assert np.array_equal(out["routes"], r_ref)
    assert out["ws_clean"], "split-K workspace must be returned to zero"


@pytest.mark.parametrize("name", sorted(CASES))
def test_dropout_mask_bit_exact(name):
    case = CASES[name]
    L = _lib()
    p, routes, ws, R = H.make_problem(case, torch.device(DEV))
    keep = torch.empty((case.m, case.k), dtype=torch.uint8, device=DEV)
    L.check(L.load().lf_dropout_mask(ctypes.byref(p), ctypes.c_void_p(keep.data_ptr()), None), "mask")
    segs, _ = H.oracle_segments(case)
    assert np.array_equal(keep.cpu().numpy(), H.oracle_keep(case, segs))


@pytest.mark.parametrize("name", ["multi4_straddle_p64", "single_r8_odd", "c1"])
def test_keep_bits_generator_matches_oracle(name):
    """lf_keep_bits (the input-free packed-mask generator) == packbits(oracle keep mask) on
    every dropout row."""
    case = CASES[name]
    L = _lib()
    p, routes, ws, R = H.make_problem(case, torch.device(DEV))
    bits = torch.full((case.m, case.k // 8), 0x5A, dtype=torch.uint8, device=DEV)
    L.check(L.load().lf_keep_bits(ctypes.byref(p), ctypes.c_void_p(bits.data_ptr()), None), "keep_bits")
    segs, _ = H.oracle_segments(case)
    keep = H.oracle_keep(case, segs)
    got = np.unpackbits(bits.cpu().numpy(), axis=1, bitorder="little")[:, :case.k]
    for s in segs:
        rows = slice(s.row_start, s.row_end)
        assert np.array_equal(got[rows], keep[rows]), s


def test_packed_bits_written_by_forward_match_oracle():
    case = CASES["multi4_straddle_p64"]
    x, w, dy, a_list, b_list = H.make_inputs(case)
    a_cat, b_cat = H.cat_weights(case, a_list, b_list)
    L = _lib()
    lib = L.load()
    p, routes, ws, R = H.make_problem(case, torch.device(DEV), use_bits=True)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    xd, ad = x.to(DEV), a_cat.to(DEV)
    s_hat = torch.empty((case.m, R), dtype=torch.bfloat16, device=DEV)
    L.check(lib.lf_build_routes(ctypes.byref(p), P(routes), None), "routes")
    L.check(lib.lf_dropout_down_fwd(ctypes.byref(p), P(xd), P(ad), P(s_hat), None), "down")
    bits = p._bits_ref.cpu().numpy()
    segs, _ = H.oracle_segments(case)
    keep = H.oracle_keep(case, segs)
    for s in segs:
        if s.dropout_p == 0:
            continue
        rows = slice(s.row_start, s.row_end)
        unpacked = np.unpackbits(bits[rows], axis=1, bitorder="little")[:, :case.k]
        assert np.array_equal(unpacked, keep[rows])


def test_explicit_keep_mask():
    case = CASES["single_r16_p01"]
    x, w, dy, a_list, b_list = H.make_inputs(case)
    a_cat, b_cat = H.cat_weights(case, a_list, b_list)
    rng = np.random.default_rng(0)
    keep = (rng.random((case.m, case.k)) > 0.3).astype(np.uint8)
    ref = H.run_oracle(case, x, w, dy, a_cat, b_cat, keep=keep)
    out = H.run_device(case, x, w, dy, a_cat, b_cat, keep_mask=torch.from_numpy(keep).to(DEV))
    _check_all(out, ref, (x, w, dy, a_cat, b_cat), "explicit")


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "numeric_*.npz"))),
                         ids=os.path.basename)
def test_golden_vectors(path):
    """Committed oracle vectors: exact bf16 inputs, bit-exact mask, outputs within tolerance."""
    d = np.load(path)
    f = lambda k: torch.from_numpy(olora.from_bf16_bits(d[k])).to(torch.bfloat16)
    st = d["seg_table"]
    sp = d["seg_params"]
    m, k = d["x"].shape
    n = d["w"].shape[0]
    used = int(st[-1, 1])
    lengths = tuple(int(r1 - r0) for r0, r1, _, _ in st)
    case = H.Case(m, k, n, tuple(int(r) for r in st[:, 3]), lengths, tuple(float(v) for v in sp[:, 0]),
                  tuple(float(v) for v in sp[:, 1]), tuple(int(v) for v in d["seg_seeds"]), int(d["offset"][0]),
                  m - used)
    inputs = (f("x"), f("w"), f("dy"), f("a_cat"), f("b_cat"))
    out = H.run_device(case, *inputs)
    ref = {kk: olora.from_bf16_bits(d[kk]) for kk in ("y", "s_hat", "dx", "ds")}
    ref.update(da=d["da"], db=d["db"], keep=d["keep"])
    _check_all(out, ref, inputs, os.path.basename(path))


def test_module_api_fused_lora_matches_oracle():
    from paper_2510_00206_b200 import FusedLoRA

    case = H.Case(512, 256, 384, (16,), (512,), (2.0,), (0.1,), (21,))
    x, w, dy, a_list, b_list = H.make_inputs(case)
    layer = FusedLoRA(w.to(DEV), rank=16, scaling=2.0, dropout_p=0.1, seed=21, dropout_rng="counter").to(DEV)
    with torch.no_grad():
        layer.lora_A.weight.copy_(a_list[0].float())
        layer.lora_B.weight.copy_(b_list[0].float())
    layer._offset = case.offset
    xd = x.to(DEV).requires_grad_(True)
    y = layer(xd)
    y.backward(dy.to(DEV))
    a_cat, b_cat = H.cat_weights(case, a_list, b_list)
    ref = H.run_oracle(case, x, w, dy, a_cat, b_cat)
    H.assert_chain_close(y.detach().float().cpu().numpy(), ref["y"], "api:y")
    H.assert_chain_close(xd.grad.float().cpu().numpy(), ref["dx"], "api:dx")
    H.assert_chain_close(layer.lora_A.weight.grad.cpu().numpy(), ref["da"], "api:dA")
    H.assert_chain_close(layer.lora_B.weight.grad.cpu().numpy(), ref["db"], "api:dB")
    assert layer._offset == case.offset + 1
    # eval: no dropout, no offset advance
    layer.eval()
    with torch.no_grad():
        y2 = layer(xd)
    case0 = H.Case(512, 256, 384, (16,), (512,), (2.0,), (0.0,), (21,))
    ref0 = H.run_oracle(case0, x, w, dy, a_cat, b_cat)
    H.assert_chain_close(y2.float().cpu().numpy(), ref0["y"], "api:eval_y")


def test_empty_batch_like_nn_linear():
    """m = 0 (e.g. a (2, 0, k) batch): an empty output that stays on the autograd graph, an
    empty dX and all-zero adapter gradients — what nn.Linear / PEFT give; nothing launches."""
    from paper_2510_00206_b200 import FusedLoRA

    w = torch.randn(384, 256, device=DEV).to(torch.bfloat16)
    layer = FusedLoRA(w, rank=16, scaling=2.0, dropout_p=0.1, seed=3).to(DEV)
    x = torch.empty(2, 0, 256, device=DEV, dtype=torch.bfloat16, requires_grad=True)
    y = layer(x)
    assert y.shape == (2, 0, 384) and y.requires_grad
    y.sum().backward()
    assert x.grad is not None and x.grad.shape == x.shape
    for p in (layer.lora_A.weight, layer.lora_B.weight):
        assert p.grad is not None and p.grad.shape == p.shape and not p.grad.any()


def test_module_api_multi_lora_slots():
    from paper_2510_00206_b200 import AdapterConfig, FusedMultiLoRA, segments_from_lengths

    case = CASES["multi4_straddle_p64"]
    x, w, dy, a_list, b_list = H.make_inputs(case)
    ads = [AdapterConfig(r, s, p, sd) for r, s, p, sd in zip(case.ranks, case.scalings, case.ps, case.seeds)]
    layer = FusedMultiLoRA(w.to(DEV), ads, track_slot_grads=True, dropout_rng="counter").to(DEV)
    with torch.no_grad():
        for i in range(4):
            layer.lora_A[i].weight.copy_(a_list[i].float())
            layer.lora_B[i].weight.copy_(b_list[i].float())
    layer._offset = case.offset
    segs = segments_from_lengths([0, 1, 2, 3], case.lengths, batches=[7, 7, 7, 7])
    xd = x.to(DEV).requires_grad_(True)
    y = layer(xd, segs)
    y.backward(dy.to(DEV))
    a_cat, b_cat = H.cat_weights(case, a_list, b_list)
    ref = H.run_oracle(case, x, w, dy, a_cat, b_cat)
    H.assert_chain_close(y.detach().float().cpu().numpy(), ref["y"], "multi:y")
    H.assert_chain_close(xd.grad.float().cpu().numpy(), ref["dx"], "multi:dx")
    oseg, _ = H.oracle_segments(case)
    for i, s in enumerate(oseg):
        r = case.ranks[i]
        H.assert_chain_close(layer.lora_A[i].weight.grad.cpu().numpy(), ref["da"][s.col_start:s.col_start + r],
                            f"multi:dA{i}")
        H.assert_chain_close(layer.lora_B[i].weight.grad.cpu().numpy(), ref["db"][:, s.col_start:s.col_start + r],
                            f"multi:dB{i}")
        ga, gb = layer.slot_grads[(i, 7)]
        assert torch.equal(ga, layer.lora_A[i].weight.grad) and torch.equal(gb, layer.lora_B[i].weight.grad)


def test_same_adapter_two_batches_keeps_separate_slots():
    """lorasched can put two global batches of one adapter in a microbatch (SURVEY §7 hard
    part 6): their gradients land in separate (adapter, batch) slots and sum in .grad."""
    from paper_2510_00206_b200 import AdapterConfig, FusedMultiLoRA, Segment

    torch.manual_seed(0)
    w = (torch.randn(256, 128) / 11).to(torch.bfloat16).to(DEV)
    layer = FusedMultiLoRA(w, [AdapterConfig(16, 2.0, 0.0, 1)], init="gaussian", track_slot_grads=True).to(DEV)
    x = torch.randn(384, 128, device=DEV).to(torch.bfloat16).requires_grad_(True)
    segs = [Segment(0, 0, 128, 0), Segment(0, 128, 384, 1)]
    y = layer(x, segs)
    y.backward(torch.randn_like(y))
    g0a, g0b = layer.slot_grads[(0, 0)]
    g1a, g1b = layer.slot_grads[(0, 1)]
    torch.testing.assert_close(g0a + g1a, layer.lora_A[0].weight.grad, rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(g0b + g1b, layer.lora_B[0].weight.grad, rtol=1e-5, atol=1e-5)
    assert not torch.allclose(g0a, g1a)


def test_shared_adapter_blocks_non_adjacent_vs_oracle():
    """Default FusedMultiLoRA: segments of one adapter share its column block, also when
    they are not adjacent (a0 | a1 | a0); checked against the oracle on that layout."""
    from paper_2510_00206_b200 import AdapterConfig, FusedMultiLoRA, Segment

    m, k, n = 640, 256, 200
    g = torch.Generator().manual_seed(3)
    x = torch.randn(m, k, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, generator=g) / k**0.5).to(torch.bfloat16)
    dy = torch.randn(m, n, generator=g).to(torch.bfloat16)
    ads = [AdapterConfig(16, 2.0, 0.1, 21), AdapterConfig(8, 1.0, 0.0, 22)]
    layer = FusedMultiLoRA(w.to(DEV), ads, init="gaussian", generator=torch.Generator(device=DEV).manual_seed(4),
                           dropout_rng="counter").to(DEV)
    with torch.no_grad():
        for p_ in layer.parameters():
            if p_.requires_grad:
                p_.copy_(p_.to(torch.bfloat16).float())
    segs = [Segment(0, 0, 200, 0), Segment(1, 200, 392, 0), Segment(0, 392, 640, 1)]
    xd = x.to(DEV).requires_grad_(True)
    y = layer(xd, segs)  # offset 0
    y.backward(dy.to(DEV))
    A = [layer.lora_A[i].weight.detach().cpu().to(torch.bfloat16) for i in range(2)]
    B = [layer.lora_B[i].weight.detach().cpu().to(torch.bfloat16) for i in range(2)]
    a_cat = torch.cat([A[0], torch.nn.functional.pad(A[1].float(), (0, 0, 0, 8)).to(torch.bfloat16)], 0)
    b_cat = torch.cat([B[0], torch.nn.functional.pad(B[1].float(), (0, 8)).to(torch.bfloat16)], 1)
    cols = [(0, 16), (16, 16), (0, 16)]
    oseg = [olora.OracleSegment(s.row_start, s.row_end, c0, r, ads[s.adapter].scaling, ads[s.adapter].dropout_p,
                                ads[s.adapter].seed) for s, (c0, r) in zip(segs, cols)]

    class _A:
        def __init__(self, p, seed):
            self.dropout_p, self.seed = p, seed

    keep = ophilox.keep_mask(m, k, [(i, s.row_start, s.row_end) for i, s in enumerate(oseg)],
                             [_A(s.dropout_p, s.seed) for s in oseg], 0)
    xf, wf, dyf = x.float().numpy(), w.float().numpy(), dy.float().numpy()
    af, bf = a_cat.float().numpy(), b_cat.float().numpy()
    y_ref, s_hat = olora.forward(xf, wf, af, bf, oseg, keep)
    dx_ref, da_ref, db_ref, _ = olora.backward(dyf, xf, wf, af, bf, s_hat, oseg, keep)
    H.assert_chain_close(y.detach().float().cpu().numpy(), y_ref, "shared:y")
    H.assert_chain_close(xd.grad.float().cpu().numpy(), dx_ref, "shared:dx")
    H.assert_chain_close(layer.lora_A[0].weight.grad.cpu().numpy(), da_ref[0:16], "shared:dA0")
    H.assert_chain_close(layer.lora_B[0].weight.grad.cpu().numpy(), db_ref[:, 0:16], "shared:dB0")
    H.assert_chain_close(layer.lora_A[1].weight.grad.cpu().numpy(), da_ref[16:24], "shared:dA1")
    H.assert_chain_close(layer.lora_B[1].weight.grad.cpu().numpy(), db_ref[:, 16:24], "shared:dB1")


def test_frozen_linear_no_adapter_matches_fp32_torch():
    """num_segments = 0: the tcgen05 GEMMs alone (Y = X·Wᵀ, dX = dY·W) vs a torch fp32 reference."""
    from paper_2510_00206_b200 import AdapterConfig, fused_multi_lora

    torch.manual_seed(1)
    for m, k, n in [(8192, 4096, 1024), (300, 264, 136)]:
        x = torch.randn(m, k, device=DEV).to(torch.bfloat16).requires_grad_(True)
        w = (torch.randn(n, k, device=DEV) / k**0.5).to(torch.bfloat16)
        a = torch.zeros(16, k, device=DEV, requires_grad=True)
        b = torch.zeros(n, 16, device=DEV, requires_grad=True)
        y = fused_multi_lora(x, w, [a], [b], [AdapterConfig(16)], [])
        dy = torch.randn(m, n, device=DEV).to(torch.bfloat16)
        y.backward(dy)
        yr = x.detach().float() @ w.float().T
        dxr = dy.float() @ w.float()
        H.assert_close_bf16(y.detach().float().cpu().numpy(), yr.cpu().numpy(), "frozen:y")
        H.assert_close_bf16(x.grad.float().cpu().numpy(), dxr.cpu().numpy(), "frozen:dx")


def _full_size_vs_fp32(m, k, n, seed=3, p=0.1):
    """Eq. 1 fwd+bwd at a full BASELINE size through the default launcher choices (tile width,
    CLC schedule and masked-dgrad variant are picked by problem size, as in the bench) against
    a torch fp32 restatement on the same device, on the kernels' own keep mask (pinned
    bit-exact to the oracle by test_dropout_mask_bit_exact and the row-sample check below).
    rel-Fro <= 4e-3 (SPEC.md §5: bf16 storage of Y / dX / Ŝ / dŜ, fp32 accumulation)."""
    from paper_2510_00206_b200 import AdapterConfig, Segment, dropout_keep_mask, fused_lora

    torch.backends.cuda.matmul.allow_tf32 = False
    g = torch.Generator(device=DEV).manual_seed(seed)
    x = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16).requires_grad_(True)
    w = (torch.randn(n, k, device=DEV, generator=g) / k**0.5).to(torch.bfloat16)
    a = ((torch.rand(16, k, device=DEV, generator=g) * 2 - 1) / k**0.5).requires_grad_(True)
    b = (torch.randn(n, 16, device=DEV, generator=g) / 4).requires_grad_(True)
    dy = torch.randn(m, n, device=DEV, generator=g).to(torch.bfloat16)
    y = fused_lora(x, w, a, b, 2.0, p, seed=99, offset=3)
    y.backward(dy)
    keep = dropout_keep_mask(m, k, [AdapterConfig(16, 2.0, p, 99)], [Segment(0, 0, m)], offset=3, device=DEV)
    rel = lambda g_, r_: float((g_ - r_).norm() / r_.norm())  # noqa: E731
    sc = 2.0 / (1.0 - p)
    ab, bb = a.detach().bfloat16().float(), b.detach().bfloat16().float()
    xm = x.detach().float() * keep.float()
    s = ((xm @ ab.T) * sc).bfloat16().float()
    err_y = rel(y.detach().float(), x.detach().float() @ w.float().T + s @ bb.T)
    del y
    ds = ((dy.float() @ bb) * sc).bfloat16().float()
    err_da = rel(a.grad, ds.T @ xm)
    del xm
    err_db = rel(b.grad, dy.float().T @ s)
    err_dx = rel(x.grad.float(), dy.float() @ w.float() + keep.float() * (ds @ ab))
    errs = {"y": err_y, "dx": err_dx, "dA": err_da, "dB": err_db}
    assert all(v < 4e-3 for v in errs.values()), errs
    assert abs(keep.float().mean().item() - (1.0 - p)) < 2e-3
    # the mask rows the kernels regenerate past row 8192 (C4 only) equal the oracle's bit for bit
    rows = np.unique(np.array([0, 4097, 8191, 8192, 12345, m - 1]) % m)
    want = ophilox.keep_mask_rows(rows, k, p, 99, 3)
    assert np.array_equal(keep[torch.as_tensor(rows, device=DEV)].cpu().numpy().astype(bool), want.astype(bool))


@pytest.mark.parametrize("shape", [(8192, 4096, 14336), (8192, 14336, 4096), (8192, 4096, 1024), (8192, 4096, 4096)],
                         ids=["gate_up", "down", "kv", "qo"])
def test_full_size_llama8b_shapes_vs_fp32_torch(shape):
    """BASELINE C2 (LLaMa-3.1-8B projections, 8192 tokens): too big for the CPU oracle."""
    _full_size_vs_fp32(*shape)


@pytest.mark.parametrize("shape", [(16384, 8192, 28672), (16384, 28672, 8192), (16384, 8192, 8192),
                                   (16384, 8192, 1024)], ids=["gate_up", "down", "qo", "kv"])
def test_full_size_llama70b_shapes_vs_fp32_torch(shape):
    """BASELINE C4 (LLaMa-3.1-70B projections, 16384 tokens): the launcher picks the 256 x 512
    wide tiles, the cluster-launch-control tile stream (> 100 waves) and the wide masked
    dgrad here — paths the small cases only reach when forced."""
    _full_size_vs_fp32(*shape, seed=4)


def test_full_size_c3_multi_lora_vs_fp32_torch():
    """BASELINE C3: 4 adapters (r 8/16/32/64 -> R = 128, p 0/0.05/0.1/0.1) on uneven segments
    of an 8192-token microbatch at k = n = 4096, against a torch fp32 restatement of Eq. 1 per
    segment on the kernels' own (oracle-pinned) keep mask."""
    from paper_2510_00206_b200 import AdapterConfig, dropout_keep_mask, fused_multi_lora, segments_from_lengths

    m, k, n = 8192, 4096, 4096
    ads = [AdapterConfig(r, 2.0, p_, i + 1) for i, (r, p_) in enumerate(zip((8, 16, 32, 64), (0.0, 0.05, 0.1, 0.1)))]
    segs = segments_from_lengths([0, 1, 2, 3], [3584, 2432, 1408, 768])
    g = torch.Generator(device=DEV).manual_seed(5)
    x = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16).requires_grad_(True)
    w = (torch.randn(n, k, device=DEV, generator=g) / k**0.5).to(torch.bfloat16)
    a = [((torch.rand(c.rank, k, device=DEV, generator=g) * 2 - 1) / k**0.5).requires_grad_(True) for c in ads]
    b = [(torch.randn(n, c.rank, device=DEV, generator=g) / 4).requires_grad_(True) for c in ads]
    dy = torch.randn(m, n, device=DEV, generator=g).to(torch.bfloat16)
    y = fused_multi_lora(x, w, a, b, ads, segs, offset=2)
    y.backward(dy)
    keep = dropout_keep_mask(m, k, ads, segs, offset=2, device=DEV).float()
    xf, dyf, wf = x.detach().float(), dy.float(), w.float()
    yr = xf @ wf.T
    dxr = dyf @ wf
    rel = lambda g_, r_: float((g_ - r_).norm() / r_.norm())
    for sg in segs:
        c = ads[sg.adapter]
        rows = slice(sg.row_start, sg.row_end)
        sc = c.scaling / (1.0 - c.dropout_p)
        ab, bb = a[sg.adapter].detach().bfloat16().float(), b[sg.adapter].detach().bfloat16().float()
        xm = xf[rows] * keep[rows]
        s_ = ((xm @ ab.T) * sc).bfloat16().float()
        yr[rows] += s_ @ bb.T
        ds = ((dyf[rows] @ bb) * sc).bfloat16().float()
        dxr[rows] += keep[rows] * (ds @ ab)
        assert rel(a[sg.adapter].grad, ds.T @ xm) < 4e-3, f"dA{sg.adapter}"
        assert rel(b[sg.adapter].grad, dyf[rows].T @ s_) < 4e-3, f"dB{sg.adapter}"
    assert rel(y.detach().float(), yr) < 4e-3
    assert rel(x.grad.float(), dxr) < 4e-3


def test_errors_are_loud_and_typed():
    from paper_2510_00206_b200 import ValidationError, fused_lora

    x = torch.randn(64, 64, device=DEV).to(torch.bfloat16)
    w = torch.randn(64, 64, device=DEV).to(torch.bfloat16)
    a = torch.randn(16, 64, device=DEV)
    b = torch.randn(64, 16, device=DEV)
    with pytest.raises(ValidationError, match="bfloat16"):
        fused_lora(x.float(), w, a, b, 2.0)
    with pytest.raises(ValidationError, match="frozen"):
        fused_lora(x, w.clone().requires_grad_(True), a, b, 2.0)
    with pytest.raises(ValidationError, match="shape"):
        fused_lora(x, w, a[:, :32], b, 2.0)
    with pytest.raises(ValidationError, match="multiples of 8"):
        xx = torch.randn(64, 60, device=DEV).to(torch.bfloat16)
        fused_lora(xx, torch.randn(64, 60, device=DEV).to(torch.bfloat16), a[:, :60].contiguous(), b, 2.0)


@pytest.mark.parametrize("sched,wide", [("1", "0"), ("2", "0"), ("1", "1"), ("2", "1")],
                         ids=["static", "clc", "static-wide", "clc-wide"])
def test_every_case_under_each_gemm_schedule(sched, wide):
    """The GEMM launcher picks its tile schedule by operand size (static persistent vs
    cluster-launch-control dynamic) and the forward tile width (256 x 256 or 256 x 512) by
    problem size, so the small parity cases above mostly run static and narrow: re-run the
    whole per-kernel oracle matrix with each combination forced (LF_SCHED / LF_WIDE are read
    once per process, hence the subprocess)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LF_SCHED=sched, LF_WIDE=wide)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_parity.py"), "-k",
                        "test_kernels_match_oracle or test_explicit_keep_mask or test_module_api or test_shared_adapter "
                        "or test_max_segments or test_microbatch_beyond",
                        "-m", "gpu"], cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_max_segments_many_per_tile_vs_oracle():
    """32 segments (the ABI maximum) of 4 adapters interleaved a0 a1 a2 a3 a0 ..., 24..40 rows
    each: up to 6 segments share a 128-row tile, every adapter's block is shared by 8
    segments (R = 16+16+32+64 = 128, the maximum), dropout on three of the adapters."""
    from paper_2510_00206_b200 import AdapterConfig, FusedMultiLoRA, Segment

    rng = np.random.default_rng(5)
    lens = rng.integers(24, 41, size=32)
    m, k, n = int(lens.sum()), 192, 160
    segs, row = [], 0
    for i, L in enumerate(lens):
        segs.append(Segment(i % 4, row, row + int(L), i // 4))
        row += int(L)
    ads = [AdapterConfig(8, 2.0, 0.1, 31), AdapterConfig(16, 1.0, 0.0, 32), AdapterConfig(32, 0.5, 0.2, 33),
           AdapterConfig(64, 2.0, 0.05, 34)]
    g = torch.Generator().manual_seed(6)
    x = torch.randn(m, k, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, generator=g) / k**0.5).to(torch.bfloat16)
    dy = torch.randn(m, n, generator=g).to(torch.bfloat16)
    layer = FusedMultiLoRA(w.to(DEV), ads, init="gaussian", generator=torch.Generator(device=DEV).manual_seed(7),
                           dropout_rng="counter").to(DEV)
    with torch.no_grad():
        for p_ in layer.parameters():
            if p_.requires_grad:
                p_.copy_(p_.to(torch.bfloat16).float())
    layer._offset = 3
    xd = x.to(DEV).requires_grad_(True)
    y = layer(xd, segs)
    y.backward(dy.to(DEV))
    cols = {0: 0, 1: 16, 2: 32, 3: 64}
    pr = {0: 16, 1: 16, 2: 32, 3: 64}
    a_cat = torch.zeros(128, k)
    b_cat = torch.zeros(n, 128)
    for a in range(4):
        A = layer.lora_A[a].weight.detach().cpu()
        B = layer.lora_B[a].weight.detach().cpu()
        a_cat[cols[a]:cols[a] + A.shape[0]] = A
        b_cat[:, cols[a]:cols[a] + B.shape[1]] = B
    oseg = [olora.OracleSegment(s.row_start, s.row_end, cols[s.adapter], pr[s.adapter], ads[s.adapter].scaling,
                                ads[s.adapter].dropout_p, ads[s.adapter].seed) for s in segs]

    class _A:
        def __init__(self, p, seed):
            self.dropout_p, self.seed = p, seed

    keep = ophilox.keep_mask(m, k, [(i, s.row_start, s.row_end) for i, s in enumerate(oseg)],
                             [_A(s.dropout_p, s.seed) for s in oseg], 3)
    xf, wf, dyf = x.float().numpy(), w.float().numpy(), dy.float().numpy()
    af, bf = a_cat.to(torch.bfloat16).float().numpy(), b_cat.to(torch.bfloat16).float().numpy()
    y_ref, s_hat = olora.forward(xf, wf, af, bf, oseg, keep)
    dx_ref, da_ref, db_ref, _ = olora.backward(dyf, xf, wf, af, bf, s_hat, oseg, keep)
    H.assert_chain_close(y.detach().float().cpu().numpy(), y_ref, "seg32:y")
    H.assert_chain_close(xd.grad.float().cpu().numpy(), dx_ref, "seg32:dx")
    for a in range(4):
        r = ads[a].rank
        H.assert_chain_close(layer.lora_A[a].weight.grad.cpu().numpy(), da_ref[cols[a]:cols[a] + r], f"seg32:dA{a}")
        H.assert_chain_close(layer.lora_B[a].weight.grad.cpu().numpy(), db_ref[:, cols[a]:cols[a] + r], f"seg32:dB{a}")


def test_microbatch_beyond_launch_limits_is_split_with_unchanged_masks():
    """5 adapters of rank 64 (R = 320 > 128): fused_multi_lora runs three row ranges; the
    Philox counters keep absolute microbatch rows (row_base), so outputs and gradients equal
    the oracle's on the unsplit microbatch."""
    from paper_2510_00206_b200 import AdapterConfig, FusedMultiLoRA, segments_from_lengths

    lens = [200, 136, 152, 96, 168]
    m, k, n = sum(lens), 256, 192
    ads = [AdapterConfig(64, 1.0 + 0.25 * i, 0.1 if i % 2 == 0 else 0.0, 40 + i) for i in range(5)]
    segs = segments_from_lengths(range(5), lens)
    g = torch.Generator().manual_seed(8)
    x = torch.randn(m, k, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, generator=g) / k**0.5).to(torch.bfloat16)
    dy = torch.randn(m, n, generator=g).to(torch.bfloat16)
    layer = FusedMultiLoRA(w.to(DEV), ads, init="gaussian", generator=torch.Generator(device=DEV).manual_seed(9),
                           dropout_rng="counter").to(DEV)
    with torch.no_grad():
        for p_ in layer.parameters():
            if p_.requires_grad:
                p_.copy_(p_.to(torch.bfloat16).float())
    xd = x.to(DEV).requires_grad_(True)
    y = layer(xd, segs)  # offset 0
    y.backward(dy.to(DEV))
    a_cat = torch.cat([layer.lora_A[i].weight.detach().cpu() for i in range(5)], 0)
    b_cat = torch.cat([layer.lora_B[i].weight.detach().cpu() for i in range(5)], 1)
    oseg, row = [], 0
    for i, L in enumerate(lens):
        oseg.append(olora.OracleSegment(row, row + L, 64 * i, 64, ads[i].scaling, ads[i].dropout_p, ads[i].seed))
        row += L

    class _A:
        def __init__(self, p, seed):
            self.dropout_p, self.seed = p, seed

    keep = ophilox.keep_mask(m, k, [(i, s.row_start, s.row_end) for i, s in enumerate(oseg)],
                             [_A(s.dropout_p, s.seed) for s in oseg], 0)
    xf, wf, dyf = x.float().numpy(), w.float().numpy(), dy.float().numpy()
    af, bf = a_cat.to(torch.bfloat16).float().numpy(), b_cat.to(torch.bfloat16).float().numpy()
    y_ref, s_hat = olora.forward(xf, wf, af, bf, oseg, keep)
    dx_ref, da_ref, db_ref, _ = olora.backward(dyf, xf, wf, af, bf, s_hat, oseg, keep)
    H.assert_chain_close(y.detach().float().cpu().numpy(), y_ref, "split:y")
    H.assert_chain_close(xd.grad.float().cpu().numpy(), dx_ref, "split:dx")
    for i in range(5):
        H.assert_chain_close(layer.lora_A[i].weight.grad.cpu().numpy(), da_ref[64 * i:64 * i + 64], f"split:dA{i}")
        H.assert_chain_close(layer.lora_B[i].weight.grad.cpu().numpy(), db_ref[:, 64 * i:64 * i + 64], f"split:dB{i}")


@pytest.mark.parametrize("m,k,n,p", [(8192, 4096, 1024, 0.1), (1000, 520, 264, 0.1), (8192, 5120, 4096, 0.0),
                                     (8192, 5120, 8192, 0.1)],
                         ids=["kv_short_k", "ragged", "wide", "wide_masked"])
def test_grad_input_accum_adds_in_l2(m, k, n, p):
    """lf_grad_input_accum: dx += ⑤ is the bf16 sum of the old dx and what lf_grad_input writes
    for the same problem (one rounding per element: torch's add of the two bf16 tensors),
    including the 256 x 512 tiles (wide / wide_masked) that previously needed a separate add."""
    lib = _lib().load()
    case = H.Case(m, k, n, (16,), (m,), (2.0,), (p,), (21,))
    prob, routes, ws, R = H.make_problem(case, torch.device(DEV), use_bits=True)
    g = torch.Generator(device=DEV).manual_seed(5)
    x = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16)
    dy = torch.randn(m, n, device=DEV, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, device=DEV, generator=g) / k**0.5).to(torch.bfloat16)
    a = (torch.randn(R, k, device=DEV, generator=g) / k**0.5).to(torch.bfloat16)
    ds = torch.randn(m, R, device=DEV, generator=g).to(torch.bfloat16)
    s_hat = torch.empty(m, R, device=DEV, dtype=torch.bfloat16)
    dx0 = torch.randn(m, k, device=DEV, generator=g).to(torch.bfloat16)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    pp = ctypes.byref(prob)
    _lib().check(lib.lf_build_routes(pp, P(routes), st), "routes")
    _lib().check(lib.lf_dropout_down_fwd(pp, P(x), P(a), P(s_hat), st), "down")  # writes the keep bits
    plain = torch.empty(m, k, device=DEV, dtype=torch.bfloat16)
    _lib().check(lib.lf_grad_input(pp, P(dy), P(w), P(ds), P(a), P(plain), st), "grad_input")
    acc = dx0.clone()
    _lib().check(lib.lf_grad_input_accum(pp, P(dy), P(w), P(ds), P(a), P(acc), st), "grad_input_accum")
    torch.cuda.synchronize()
    want = (dx0.float() + plain.float()).to(torch.bfloat16)
    assert torch.equal(acc, want), int((acc != want).sum())
