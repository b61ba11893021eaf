"""Per-wave L2 floor of the GEMM DRAM traffic, next to the ncu-measured bytes of one C2 step.

    python tools/gemm_l2_floor.py [profiles/gemm_traffic.json [c2|c4|c1]]

SURVEY.md §8(d)'s algorithmic bytes assume every operand byte crosses HBM once. With 126 MB
of L2 and operands of 120-350 MB that is unreachable for the long-K GEMMs: the 74 resident
CTA pairs of one wave sweep K together, so a wave must stream the full K-extent of every A
row-block and B column-block its tiles touch, and the next wave streams its own again. This
script walks the launcher's raster (grouped, 8 m-tiles per n-sweep; 256x256 pair tiles or
256x512 wide tiles by the launcher's rule, lf_gemm.cu gemm_launch) in waves of 74 tiles and
sums those per-wave operand bytes + the output: the traffic of a perfectly K-synchronous
wave with no reuse between waves. Measured / floor > 1 is drift inside a wave; algorithmic /
floor < 1 is the re-reading that the tile size and the L2 make unavoidable.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PAIRS = 74  # 148 SMs / cta_group::2
GROUP = 8


def wave_floor(M: int, N: int, K: int, wide: bool, e: int = 2) -> float:
    bm, bn = 256, 512 if wide else 256
    tm, tn = -(-M // bm), -(-N // bn)
    order = []
    for t in range(tm * tn):
        per_group = GROUP * tn
        g, r = divmod(t, per_group)
        gm = min(GROUP, tm - g * GROUP)
        order.append((g * GROUP + r % gm, r // gm))
    total = 0.0
    for w in range(0, len(order), PAIRS):
        wave = order[w:w + PAIRS]
        ms = {mb for mb, _ in wave}
        ns = {nb for _, nb in wave}
        total += (len(ms) * min(bm, M) + len(ns) * min(bn, N)) * K * e
    return total + M * N * e


def wide_rule(M: int, N: int, K: int, masked_dgrad: bool) -> bool:
    min_k = 8192 if masked_dgrad else 4096
    return (-(-M // 256)) * (-(-N // 512)) >= 4 * PAIRS and K >= min_k


def main() -> None:
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "gemm_traffic.json")
    config = sys.argv[2] if len(sys.argv) > 2 else "c2"
    with open(path) as f:
        tr = json.load(f)
    from bench import projections, tokens_per_gpu

    shapes = {name: (k, n) for name, k, n, _ in projections(config)}
    m = tokens_per_gpu(config)
    rows = []
    for launch in tr["per_launch"]:
        name, kind = launch["launcher"].split()
        k, n = shapes[name]
        if kind == "base_fwd":
            M, N, K, masked = m, n, k, False
        else:  # grad_input: dX[m, k] = dY[m, n] · W[n, k], dropout on (masked)
            M, N, K, masked = m, k, n, True
        wide = wide_rule(M, N, K, masked)
        floor = wave_floor(M, N, K, wide)
        meas = launch["dram_read"] + launch["dram_write"]
        rows.append({"launcher": launch["launcher"], "tile": "256x512" if wide else "256x256",
                     "algorithmic_MB": round(launch["algorithmic"] / 1e6, 1),
                     "wave_floor_MB": round(floor / 1e6, 1), "measured_MB": round(meas / 1e6, 1),
                     "measured_over_floor": round(meas / floor, 2),
                     "measured_over_algorithmic": round(meas / launch["algorithmic"], 2)})
    tot = {k: round(sum(r[k] for r in rows), 1) for k in ("algorithmic_MB", "wave_floor_MB", "measured_MB")}
    print(json.dumps({"source": os.path.relpath(path, ROOT), "launches": rows, "total": tot}, indent=1))


if __name__ == "__main__":
    main()
