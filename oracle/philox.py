"""Philox4x32-10 and the SPEC.md §3 dropout keep mask, vectorised in numpy.

TEST INFRASTRUCTURE (see oracle/__init__.py). Philox4x32-10 restated from its published
definition (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3",
SC'11; Random123 philox.h): multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key increments
0x9E3779B9 / 0xBB67AE85, 10 rounds, key bumped between rounds.

The reference leaves the dropout RNG unspecified ("Dropout mask stored at 1 byte per
element ... paper silent on storage format", reference SPEC.md:177; MASK_BYTES=1,
ls/costmodel.py:21); SPEC.md §3 of this repo defines it, and this module is its oracle.
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = 0x9E3779B9
_W1 = 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr: np.ndarray, key) -> np.ndarray:
    """ctr: (..., 4) uint32 counters; key: (k0, k1) (broadcastable). Returns (..., 4) uint32."""
    ctr = np.asarray(ctr, dtype=np.uint32)
    c0 = ctr[..., 0].astype(np.uint64)
    c1 = ctr[..., 1].astype(np.uint64)
    c2 = ctr[..., 2].astype(np.uint64)
    c3 = ctr[..., 3].astype(np.uint64)
    k0 = np.uint64(int(key[0]) & 0xFFFFFFFF)
    k1 = np.uint64(int(key[1]) & 0xFFFFFFFF)
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
        k0 = np.uint64((int(k0) + _W0) & 0xFFFFFFFF)
        k1 = np.uint64((int(k1) + _W1) & 0xFFFFFFFF)
    return np.stack([c0, c1, c2, c3], axis=-1).astype(np.uint32)


def dropout_threshold(p: float) -> int:
    """Integer threshold of SPEC.md §3: keep iff the 16-bit lane >= 2 * floor(p * 32768).

    The threshold is even (p quantised to 2^-15) so ``u16 >= thr`` equals
    ``(u16 >> 1) >= thr / 2``, the borrow-free two-lanes-per-word test the kernels use."""
    if not 0.0 <= p < 1.0:
        raise ValueError(f"dropout_p must be in [0, 1), got {p}")
    return 2 * int(np.floor(np.float64(np.float32(p)) * 32768.0))


def keep_mask_rows(rows: np.ndarray, k: int, p: float, seed: int, offset: int) -> np.ndarray:
    """Keep mask (len(rows) x k, uint8) for the given absolute token rows of one segment."""
    thr = dropout_threshold(p)
    rows = np.asarray(rows, dtype=np.int64)
    if thr == 0:
        return np.ones((rows.size, k), dtype=np.uint8)
    groups = (k + 7) // 8
    g = np.arange(groups, dtype=np.uint32)
    ctr = np.empty((rows.size, groups, 4), dtype=np.uint32)
    ctr[..., 0] = g[None, :]
    ctr[..., 1] = rows.astype(np.uint32)[:, None]
    ctr[..., 2] = np.uint32(offset & 0xFFFFFFFF)
    ctr[..., 3] = np.uint32((offset >> 32) & 0xFFFFFFFF)
    out = philox4x32_10(ctr, (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF))  # (rows, groups, 4)
    lanes = np.empty((rows.size, groups, 8), dtype=np.uint32)
    lanes[..., 0::2] = out & np.uint32(0xFFFF)
    lanes[..., 1::2] = out >> np.uint32(16)
    keep = (lanes >= np.uint32(thr)).astype(np.uint8).reshape(rows.size, groups * 8)
    return keep[:, :k]


def keep_mask(m: int, k: int, segments, adapters, offset: int) -> np.ndarray:
    """Full (m x k) keep mask of a microbatch. ``segments``: (adapter, row_start, row_end)
    triples; ``adapters``: objects with dropout_p and seed. Rows outside segments keep all."""
    keep = np.ones((m, k), dtype=np.uint8)
    for a_idx, r0, r1 in segments:
        a = adapters[a_idx]
        if r1 > r0:
            keep[r0:r1] = keep_mask_rows(np.arange(r0, r1), k, a.dropout_p, a.seed, offset)
    return keep
