"""Independent byte-count restatement of the reference's per-kernel DRAM traffic model.

TEST INFRASTRUCTURE (see oracle/__init__.py). Restates ls/costmodel.py:219-306
(``_frozen_kernels``, ``_unfused_kernels``, ``_fused_kernels``, ``traffic``,
``roundtrip_bytes``) and adds the ``b200_minimal`` variant of SURVEY.md §8(d) — the
bytes the sm_100a kernels of this repo are designed to move (mask regenerated, no
mk-sized intermediate, fp32 gradients). Counting rule (ls/costmodel.py:6-11): every
operand charged once per kernel that touches it, masks 1 byte per element.

Returns plain (kernel, bytes_read, bytes_written) tuples so it shares no code with the
product's paper_2510_00206_b200.traffic.
"""
from __future__ import annotations

import math


def kernels(m, k, n, r, e=2, variant="unfused", pass_name="forward", mask_bytes=1):
    mk, mn, kn, mr, kr, rn = m * k, m * n, k * n, m * r, k * r, r * n
    fwd = pass_name == "forward"
    if r == 0:
        if fwd:
            return [("base_gemm", e * (mk + kn), e * mn)]
        return [("grad_input_gemm", e * (mn + kn), e * mk), ("grad_weight_gemm", e * (mk + mn), e * kn)]
    if variant == "unfused":
        if fwd:
            return [
                ("dropout", e * mk, e * mk + mask_bytes * mk),
                ("down_proj_gemm", e * (mk + kr), e * mr),
                ("up_proj_gemm", e * (mr + rn), e * mn),
                ("base_gemm", e * (mk + kn), e * mn),
                ("add_scale", 2 * e * mn, e * mn),
            ]
        return [
            ("grad_up_input_gemm", e * (mn + rn), e * mr),
            ("grad_up_weight_gemm", e * (mr + mn), e * rn),
            ("grad_down_input_gemm", e * (mr + kr), e * mk),
            ("grad_down_weight_gemm", e * (mk + mr), e * kr),
            ("grad_base_input_gemm", e * (mn + kn), e * mk),
            ("dropout_grad_accum", 2 * e * mk + mask_bytes * mk, e * mk),
        ]
    if variant in ("fused_lora", "fused_multi_lora"):
        if fwd:
            out = [
                ("dropout_down_proj_fused", e * (mk + kr), e * mk + mask_bytes * mk + e * mr),
                ("base_gemm_epilogue_fused", e * (mk + kn + mr + rn), e * mn),
            ]
        else:
            out = [
                ("grad_up_fused", e * (mn + mr + rn), e * (mr + rn)),
                ("grad_down_fused", e * (mk + mr + kr), e * (kr + mk)),
                ("grad_base_accum_fused", e * (mn + kn + mk) + mask_bytes * mk, e * mk),
            ]
        if variant == "fused_multi_lora":
            out.append(("adapter_routing_table", math.ceil(m / 128) * 16, 0))
        return out
    if variant == "b200_built":
        bits = m * -(-k // 8)  # bit-packed keep mask
        rows = kernels(m, k, n, r, e, "b200_minimal", pass_name)
        add = {"dropout_down_proj_fused": (0, bits), "grad_down_fused": (bits, 0), "grad_base_accum_fused": (bits, 0)}
        return [(nm, rd + add.get(nm, (0, 0))[0], wr + add.get(nm, (0, 0))[1]) for nm, rd, wr in rows]
    if variant == "b200_minimal":
        f = 4  # fp32 gradient accumulators
        if fwd:
            return [
                ("dropout_down_proj_fused", e * (mk + kr), e * mr),
                ("base_gemm_epilogue_fused", e * (mk + kn + mr + rn), e * mn),
            ]
        return [
            ("grad_up_fused", e * (mn + rn + mr), e * mr + f * rn),
            ("grad_down_fused", e * (mk + mr), f * kr),
            ("grad_base_accum_fused", e * (mn + kn + mr + kr), e * mk),
        ]
    raise ValueError(variant)


def total(m, k, n, r, e=2, variant="unfused"):
    return sum(a + b for p in ("forward", "backward") for _, a, b in kernels(m, k, n, r, e, variant, p))
