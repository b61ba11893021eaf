"""Eq. 1 LoRA linear forward/backward at SPEC.md §2's rounding points (numpy, fp64).

TEST INFRASTRUCTURE (see oracle/__init__.py). Restates:
  * Eq. 1 Y = X W + alpha (X̂ A) B, X̂ = dropout(X)
  * the graph split at S (S is stored, re-read by the base GEMM) PAPER.md:438-450
  * the fused kernel list ① .. ⑤ and which tensors exist           ls/costmodel.py:252-282,
                                                                    PAPER.md:455-463
  * tile-level multi-adapter routing (rows -> adapter A/B, scale, dropout)
  * segment layout of a microbatch                                  ls/packing.py:41-98
in torch/PEFT layouts: X (m,k), W (n,k), A_cat (R,k), B_cat (n,R).

Accumulation is float64 from the bf16-exact inputs; the stored intermediates Ŝ and dŜ
and the bf16 outputs Y and dX are rounded exactly where the kernels round (fp32 first,
then bf16 round-to-nearest-even); dA and dB are returned in fp32. ``acc=np.float32``
runs the same algorithm at fp32 accumulation — used only to time the CPU baseline
(bench.py), never as the parity reference.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np


def bf16_round(a) -> np.ndarray:
    """Round to the nearest bfloat16 (ties to even), returned as float32 values."""
    f = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return u.astype(np.uint32).view(np.float32).reshape(f.shape)


def bf16_bits(a) -> np.ndarray:
    """bf16 bit patterns (uint16) of already-bf16-exact float32 values."""
    return (np.ascontiguousarray(bf16_round(a)).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def from_bf16_bits(u16) -> np.ndarray:
    return (np.asarray(u16, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


@dataclass(frozen=True)
class OracleSegment:
    """One (adapter, global batch) row segment with its column block in the rank-concat dim."""

    row_start: int
    row_end: int
    col_start: int
    rank: int  # padded (multiple of 16) block width
    scaling: float
    dropout_p: float
    seed: int = 0


def segment_scale(seg: OracleSegment) -> np.float32:
    """s = scaling / (1 - p): fp32 inputs, fp64 division, one rounding to fp32 (SPEC.md §2)."""
    return np.float32(np.float64(np.float32(seg.scaling)) / (1.0 - np.float64(np.float32(seg.dropout_p))))


def _f32(x) -> np.ndarray:
    return np.asarray(x, dtype=np.float64).astype(np.float32)


def forward(x, w, a_cat, b_cat, segments: Sequence[OracleSegment], keep,
            acc=np.float64) -> tuple[np.ndarray, np.ndarray]:
    """Returns (y, s_hat) as bf16-valued float32 arrays. ``keep``: (m,k) uint8 (1 keep)."""
    x = np.asarray(x, acc)
    m = x.shape[0]
    R = a_cat.shape[0]
    s_hat = np.zeros((m, R), np.float32)
    for s in segments:
        if s.row_end <= s.row_start:
            continue
        rows = slice(s.row_start, s.row_end)
        cols = slice(s.col_start, s.col_start + s.rank)
        xm = x[rows] * np.asarray(keep[rows], acc)
        part = _f32(xm @ np.asarray(a_cat[cols], acc).T)
        s_hat[rows, cols] = bf16_round(part * segment_scale(s))
    y = x @ np.asarray(w, acc).T
    if R:
        y = y + np.asarray(s_hat, acc) @ np.asarray(b_cat, acc).T
    return bf16_round(_f32(y)), s_hat


def backward(dy, x, w, a_cat, b_cat, s_hat, segments: Sequence[OracleSegment], keep, acc=np.float64):
    """Returns (dx bf16-valued, da fp32 (R,k), db fp32 (n,R), ds bf16-valued (m,R))."""
    dy = np.asarray(dy, acc)
    x = np.asarray(x, acc)
    m = dy.shape[0]
    R = a_cat.shape[0]
    ds = np.zeros((m, R), np.float32)
    for s in segments:
        if s.row_end <= s.row_start:
            continue
        rows = slice(s.row_start, s.row_end)
        cols = slice(s.col_start, s.col_start + s.rank)
        part = _f32(dy[rows] @ np.asarray(b_cat[:, cols], acc))
        ds[rows, cols] = bf16_round(part * segment_scale(s))
    keep64 = np.asarray(keep, acc)
    xm = x * keep64
    ds64 = np.asarray(ds, acc)
    db = _f32(dy.T @ np.asarray(s_hat, acc)) if R else np.zeros((w.shape[0], 0), np.float32)
    da = _f32(ds64.T @ xm) if R else np.zeros((0, x.shape[1]), np.float32)
    dx = dy @ np.asarray(w, acc)
    if R:
        dx = dx + keep64 * (ds64 @ np.asarray(a_cat, acc))
    return bf16_round(_f32(dx)), da, db, ds


def base_forward(x, w, s_hat, b_cat) -> np.ndarray:
    """② alone: Y = bf16(X·Wᵀ + Ŝ·B_catᵀ) for a given (device-produced) Ŝ."""
    y = np.asarray(x, np.float64) @ np.asarray(w, np.float64).T
    if s_hat.shape[1]:
        y = y + np.asarray(s_hat, np.float64) @ np.asarray(b_cat, np.float64).T
    return bf16_round(_f32(y))


def grads_given(dy, x, w, a_cat, s_hat, ds, keep):
    """③'s dB, ④ and ⑤ alone, for given (device-produced) Ŝ and dŜ: returns (dx, da, db)."""
    dy = np.asarray(dy, np.float64)
    keep64 = np.asarray(keep, np.float64)
    xm = np.asarray(x, np.float64) * keep64
    ds64 = np.asarray(ds, np.float64)
    db = _f32(dy.T @ np.asarray(s_hat, np.float64))
    da = _f32(ds64.T @ xm)
    dx = dy @ np.asarray(w, np.float64) + keep64 * (ds64 @ np.asarray(a_cat, np.float64))
    return bf16_round(_f32(dx)), da, db


def bf16_ulp(a) -> np.ndarray:
    """Spacing of bf16 values at |a| (8 significant bits)."""
    a = np.abs(np.asarray(a, np.float64))
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    return np.where(a > 0, 2.0 ** (e - 7), 2.0**-133)


def rel_fro(got, ref) -> float:
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / den) if den > 0 else float(np.linalg.norm(got - ref))
