"""The CPU oracle, pinned before it is trusted (no GPU needed)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import lora as olora
from oracle import philox as ophilox

# Random123 kat_vectors for philox4x32-10 (published known answers; SPEC.md §3)
KAT = [
    ((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
     (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF), (0xFFFFFFFF, 0xFFFFFFFF),
     (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_known_answers(ctr, key, out):
    got = ophilox.philox4x32_10(np.array(ctr, dtype=np.uint32), key)
    assert tuple(int(v) for v in got) == out


def test_philox_vectorised_matches_scalar():
    rng = np.random.default_rng(0)
    ctrs = rng.integers(0, 2**32, size=(64, 4), dtype=np.uint64).astype(np.uint32)
    key = (0x12345678, 0x9ABCDEF0)
    batch = ophilox.philox4x32_10(ctrs, key)
    for i in range(64):
        assert np.array_equal(batch[i], ophilox.philox4x32_10(ctrs[i], key))


def test_keep_mask_layout_and_rate():
    m, k, p, seed, off = 64, 200, 0.1, 1234, 7
    keep = ophilox.keep_mask_rows(np.arange(m), k, p, seed, off)
    assert keep.shape == (m, k) and keep.dtype == np.uint8
    # element (row, col) comes from lane col&7 of philox((col>>3, row, off, 0), seed)
    for row, col in [(0, 0), (3, 9), (63, 199), (17, 128)]:
        out = ophilox.philox4x32_10(np.array([col >> 3, row, off, 0], np.uint32), (seed, 0))
        lane = col & 7
        u16 = (int(out[lane >> 1]) >> (16 * (lane & 1))) & 0xFFFF
        assert keep[row, col] == (u16 >= ophilox.dropout_threshold(p))
    big = ophilox.keep_mask_rows(np.arange(512), 4096, p, seed, off)
    assert abs(big.mean() - (1 - p)) < 3e-3


def test_keep_mask_threshold_edges():
    assert ophilox.dropout_threshold(0.0) == 0
    assert ophilox.dropout_threshold(0.5) == 32768
    assert np.all(ophilox.keep_mask_rows(np.arange(4), 64, 0.0, 1, 2) == 1)
    with pytest.raises(ValueError):
        ophilox.dropout_threshold(1.0)
    # different offsets / seeds / rows give different masks
    a = ophilox.keep_mask_rows(np.arange(8), 256, 0.3, 5, 0)
    b = ophilox.keep_mask_rows(np.arange(8), 256, 0.3, 5, 1)
    c = ophilox.keep_mask_rows(np.arange(8), 256, 0.3, 6, 0)
    assert not np.array_equal(a, b) and not np.array_equal(a, c)


def test_bf16_round_matches_torch():
    x = np.random.default_rng(1).standard_normal(10000).astype(np.float32) * 37.0
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(olora.bf16_round(x), ref)
    bits = olora.bf16_bits(ref)
    assert np.array_equal(olora.from_bf16_bits(bits), ref)


def _torch_autograd_reference(x, w, a, b, scaling, p, keep):
    """Independent restatement: Eq. 1 in torch float64 autograd (no rounding points)."""
    X = torch.tensor(x, dtype=torch.float64)
    W = torch.tensor(w, dtype=torch.float64)
    A = torch.tensor(a, dtype=torch.float64, requires_grad=True)
    B = torch.tensor(b, dtype=torch.float64, requires_grad=True)
    X.requires_grad_(True)
    Xh = X * torch.tensor(keep, dtype=torch.float64) / (1 - p)
    Y = X @ W.T + scaling * (Xh @ A.T) @ B.T
    return X, A, B, Y


@pytest.mark.parametrize("p", [0.0, 0.1])
def test_oracle_matches_independent_autograd(p):
    rng = np.random.default_rng(2)
    m, k, n, r = 96, 64, 80, 16
    bf = olora.bf16_round
    x = bf(rng.standard_normal((m, k), dtype=np.float32))
    w = bf(rng.standard_normal((n, k), dtype=np.float32) / 8)
    a = bf(rng.standard_normal((r, k), dtype=np.float32) / 8)
    b = bf(rng.standard_normal((n, r), dtype=np.float32) / 4)
    dy = bf(rng.standard_normal((m, n), dtype=np.float32))
    keep = ophilox.keep_mask_rows(np.arange(m), k, p, 99, 3)
    seg = [olora.OracleSegment(0, m, 0, r, 2.0, p, 99)]
    y, s_hat = olora.forward(x, w, a, b, seg, keep)
    dx, da, db, ds = olora.backward(dy, x, w, a, b, s_hat, seg, keep)
    X, A, B, Y = _torch_autograd_reference(x, w, a, b, 2.0, p, keep)
    Y.backward(torch.tensor(dy, dtype=torch.float64))
    # the oracle rounds Ŝ / dŜ to bf16 (SPEC.md §2); agreement is at bf16 level
    assert olora.rel_fro(y, Y.detach().numpy()) < 4e-3
    assert olora.rel_fro(dx, X.grad.numpy()) < 4e-3
    assert olora.rel_fro(da, A.grad.numpy()) < 4e-3
    assert olora.rel_fro(db, B.grad.numpy()) < 4e-3


def test_oracle_multi_segment_equals_separate_layers():
    """Rank-concat routing (SPEC.md §1) == running each segment through its own adapter."""
    rng = np.random.default_rng(3)
    bf = olora.bf16_round
    k, n = 64, 48
    lens, ranks = [40, 24, 64], [8, 16, 32]
    m = sum(lens)
    x = bf(rng.standard_normal((m, k), dtype=np.float32))
    w = bf(rng.standard_normal((n, k), dtype=np.float32) / 8)
    dy = bf(rng.standard_normal((m, n), dtype=np.float32))
    segs, a_blocks, b_blocks, row, col = [], [], [], 0, 0
    for i, (L, r) in enumerate(zip(lens, ranks)):
        rp = -(-r // 16) * 16
        a = np.zeros((rp, k), np.float32)
        a[:r] = bf(rng.standard_normal((r, k), dtype=np.float32) / 8)
        b = np.zeros((n, rp), np.float32)
        b[:, :r] = bf(rng.standard_normal((n, r), dtype=np.float32) / 4)
        a_blocks.append(a)
        b_blocks.append(b)
        segs.append(olora.OracleSegment(row, row + L, col, rp, 1.0 + i, 0.1 * i, 10 + i))
        row += L
        col += rp
    keep = np.ones((m, k), np.uint8)
    for s in segs:
        keep[s.row_start:s.row_end] = ophilox.keep_mask_rows(np.arange(s.row_start, s.row_end), k, s.dropout_p,
                                                              s.seed, 0)
    A, B = np.concatenate(a_blocks, 0), np.concatenate(b_blocks, 1)
    y, s_hat = olora.forward(x, w, A, B, segs, keep)
    dx, da, db, ds = olora.backward(dy, x, w, A, B, s_hat, segs, keep)
    for i, s in enumerate(segs):
        rows = slice(s.row_start, s.row_end)
        one = olora.OracleSegment(0, s.row_end - s.row_start, 0, s.rank, s.scaling, s.dropout_p, s.seed)
        y1, s1 = olora.forward(x[rows], w, a_blocks[i], b_blocks[i], [one], keep[rows])
        dx1, da1, db1, ds1 = olora.backward(dy[rows], x[rows], w, a_blocks[i], b_blocks[i], s1, [one], keep[rows])
        cols = slice(s.col_start, s.col_start + s.rank)
        assert np.array_equal(y[rows], y1)
        assert np.array_equal(s_hat[rows, cols], s1)
        assert np.array_equal(dx[rows], dx1)
        np.testing.assert_allclose(da[cols], da1, rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(db[:, cols], db1, rtol=1e-6, atol=1e-6)
        off = np.ones(s_hat.shape[1], bool)
        off[cols] = False
        assert not s_hat[rows][:, off].any() and not ds[rows][:, off].any()


def test_numeric_golden_reproduces():
    """The committed oracle vectors (tests/golden/numeric_*.npz) still come out bit-identical."""
    import glob
    import os

    from tests.golden import make_numeric_golden as gen

    files = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "numeric_*.npz")))
    assert files, "run tests/golden/make_numeric_golden.py"
    for path in files:
        data = np.load(path)
        name = os.path.basename(path)[len("numeric_"):-len(".npz")]
        fresh = gen.compute(gen.CASES[name])
        for key in ("y", "s_hat", "dx", "ds", "keep"):
            assert np.array_equal(olora.from_bf16_bits(data[key]) if key != "keep" else data[key],
                                  olora.from_bf16_bits(fresh[key]) if key != "keep" else fresh[key]), (name, key)
        np.testing.assert_allclose(data["da"], fresh["da"], rtol=0, atol=0)
        np.testing.assert_allclose(data["db"], fresh["db"], rtol=0, atol=0)
