"""Segment table -> per-128-row-tile routing table (integer, bit-exact).

TEST INFRASTRUCTURE (see oracle/__init__.py). Restates the multi-adapter routing the
reference charges as ``adapter_routing_table`` — one ROUTING_ENTRY_BYTES = 16 descriptor
per ROUTING_TILE_ROWS = 128 rows (ls/costmodel.py:23-26, 279-281) — with the entry
layout of SPEC.md §4: {seg_lo, seg_hi, col_lo, col_hi} as int32. Segments follow
lorasched's microbatch layout: consecutive padded segments (ls/packing.py:30-32, 41-98).
"""
from __future__ import annotations

import numpy as np

TILE_ROWS = 128
ENTRY_BYTES = 16


def padded_len(raw_tokens: int, padding_multiple: int) -> int:
    """Least multiple of padding_multiple >= raw_tokens (ls/packing.py:30-32)."""
    return -(-int(raw_tokens) // int(padding_multiple)) * int(padding_multiple)


def pad_rank(r: int) -> int:
    return -(-int(r) // 16) * 16


def column_blocks(ranks, adapters=None) -> list[int]:
    """col_start of each segment's block in the rank-concat dimension. With ``adapters``
    (one slot per segment), segments of the same adapter share one block, assigned in
    order of first appearance (SPEC.md §1)."""
    out, c, seen = [], 0, {}
    for i, r in enumerate(ranks):
        if adapters is not None and adapters[i] in seen:
            out.append(seen[adapters[i]])
            continue
        out.append(c)
        if adapters is not None:
            seen[adapters[i]] = c
        c += pad_rank(r)
    return out


def routes(seg_rows, seg_cols, m: int) -> np.ndarray:
    """seg_rows: [(row_start, row_end)], seg_cols: [(col_start, width)] -> (ceil(m/128), 4) int32."""
    tiles = -(-m // TILE_ROWS)
    out = np.zeros((tiles, 4), dtype=np.int32)
    for t in range(tiles):
        r0, r1 = t * TILE_ROWS, min(m, (t + 1) * TILE_ROWS)
        hit = [i for i, (a, b) in enumerate(seg_rows) if a < b and a < r1 and b > r0]
        if not hit:
            out[t] = (0, -1, 0, 0)
        else:
            lo, hi = hit[0], hit[-1]
            # hull of the hit segments' column blocks (SPEC.md §4; blocks may be shared)
            c0 = min(seg_cols[i][0] for i in hit)
            c1 = max(seg_cols[i][0] + seg_cols[i][1] for i in hit)
            out[t] = (lo, hi, c0, c1)
    return out


def table_bytes(m: int) -> int:
    """Bytes of the routing table for m rows (what the reference's model charges)."""
    return -(-m // TILE_ROWS) * ENTRY_BYTES
