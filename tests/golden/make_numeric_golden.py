"""Oracle-generated numerical golden vectors (small shapes, edge cases).

    python tests/golden/make_numeric_golden.py

Writes numeric_<case>.npz: bf16 inputs (uint16 bit patterns), the SPEC.md §3 keep mask
and every oracle output (bf16 bit patterns for Y, Ŝ, dŜ, dX; fp32 dA, dB). The reference
has no numerical implementation of this path ("parity unpinned", oracle/__init__.py), so
these vectors pin the oracle against regression and give the GPU parity tests fixed,
bit-exact inputs and integer masks.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import lora as olora  # noqa: E402
from oracle import philox as ophilox  # noqa: E402

# name: (m, k, n, [(rank, rows, scaling, p, seed)], offset, gap_rows)
CASES = {
    "single_p01": (128, 64, 96, [(16, 128, 2.0, 0.1, 1234)], 5, 0),
    "odd_edges": (130, 72, 200, [(8, 130, 2.0, 0.1, 77)], 0, 0),
    "multi3_straddle": (320, 96, 64, [(8, 64, 2.0, 0.0, 1), (16, 96, 0.5, 0.05, 2), (32, 100, 1.0, 0.1, 3)], 9, 60),
    "tiny": (1, 8, 8, [(16, 1, 2.0, 0.5, 3)], 0, 0),
}


def compute(case):
    m, k, n, segspec, offset, gap = case
    rng = np.random.default_rng(m * 1000003 + k * 1009 + n)
    bf = olora.bf16_round
    x = bf(rng.standard_normal((m, k), dtype=np.float32))
    w = bf(rng.standard_normal((n, k), dtype=np.float32) / np.sqrt(k))
    dy = bf(rng.standard_normal((m, n), dtype=np.float32))
    segs, a_blocks, b_blocks, row, col = [], [], [], 0, 0
    for r, rows, sc, p, seed in segspec:
        rp = -(-r // 16) * 16
        a = np.zeros((rp, k), np.float32)
        a[:r] = bf((rng.random((r, k), dtype=np.float32) * 2 - 1) / np.sqrt(k))
        b = np.zeros((n, rp), np.float32)
        b[:, :r] = bf(rng.standard_normal((n, r), dtype=np.float32) / np.sqrt(r))
        a_blocks.append(a)
        b_blocks.append(b)
        segs.append(olora.OracleSegment(row, row + rows, col, rp, sc, p, seed))
        row += rows
        col += rp
    assert row + gap == m or gap == 0 and row == m, case
    A, B = np.concatenate(a_blocks, 0), np.concatenate(b_blocks, 1)
    keep = np.ones((m, k), np.uint8)
    for s in segs:
        keep[s.row_start:s.row_end] = ophilox.keep_mask_rows(np.arange(s.row_start, s.row_end), k, s.dropout_p,
                                                              s.seed, offset)
    y, s_hat = olora.forward(x, w, A, B, segs, keep)
    dx, da, db, ds = olora.backward(dy, x, w, A, B, s_hat, segs, keep)
    seg_table = np.array([[s.row_start, s.row_end, s.col_start, s.rank] for s in segs], np.int32)
    seg_params = np.array([[s.scaling, s.dropout_p] for s in segs], np.float32)
    seg_seeds = np.array([s.seed for s in segs], np.uint64)
    B16 = olora.bf16_bits
    return dict(x=B16(x), w=B16(w), dy=B16(dy), a_cat=B16(A), b_cat=B16(B), keep=keep, y=B16(y), s_hat=B16(s_hat),
                dx=B16(dx), ds=B16(ds), da=da, db=db, seg_table=seg_table, seg_params=seg_params, seg_seeds=seg_seeds,
                offset=np.array([offset], np.uint64))


def main():
    for name, case in CASES.items():
        np.savez_compressed(os.path.join(HERE, f"numeric_{name}.npz"), **compute(case))
        print("wrote", name)


if __name__ == "__main__":
    main()
