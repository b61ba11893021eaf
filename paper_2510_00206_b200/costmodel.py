"""DRAM-traffic model of the LoRA linear layer — drop-in mirror of ``lorasched.costmodel``'s
traffic API (ls/costmodel.py:21-124, 158-216, 219-306), extended with ``b200_minimal``.

The reference's variants ``unfused`` / ``fused_lora`` / ``fused_multi_lora`` keep their
kernel names and byte counts exactly (pinned by tests/golden/traffic_reference.json,
generated from lorasched itself); ``b200_minimal`` is SURVEY.md §8(d)'s floor for this
design: the dropout mask is regenerated from Philox instead of being stored, ④ writes no
mk-sized LoRA input-gradient (the term is accumulated inside ⑤'s GEMM), and dA/dB are
fp32 accumulators; ``b200_built`` is what the sm_100a kernels actually move with dropout
on — ``b200_minimal`` plus the bit-packed keep mask ① writes and ④/⑤ read (m·k/8 bytes
each way, 1/16 of X), which replaces two of the three Philox passes.

Every kernel is a table row of (name, read terms, write terms): a term is a
(coefficient, monomial) pair over the operand sizes mk, mn, kn, mr, kr, rn, with
``e`` = element bytes, ``mask`` = 1 byte per element, ``f32`` = 4 bytes.
"""
from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

from .errors import ValidationError

MASK_BYTES = 1
ROUTING_TILE_ROWS = 128
ROUTING_ENTRY_BYTES = 16
VARIANTS = ("unfused", "fused_lora", "fused_multi_lora", "b200_minimal", "b200_built")
PASSES = ("forward", "backward")


@dataclass(frozen=True)
class HardwareProfile:
    """Peak dense half-precision FLOP/s and HBM bandwidth; balance = their ratio."""

    peak_flops_half: float
    mem_bandwidth: float
    machine_balance: float | None = None

    def __post_init__(self):
        if not (self.peak_flops_half > 0 and self.mem_bandwidth > 0):
            raise ValidationError("hardware rates must be strictly positive")
        derived = self.peak_flops_half / self.mem_bandwidth
        if self.machine_balance is None:
            object.__setattr__(self, "machine_balance", derived)
        elif abs(self.machine_balance - derived) > 1e-6 * derived:
            raise ValidationError(
                f"machine_balance {self.machine_balance} inconsistent with peak/bandwidth ratio {derived}"
            )


H100_SXM = HardwareProfile(peak_flops_half=989e12, mem_bandwidth=3.35e12)
# measured on this pool's B200s (MEASURED_PEAKS.json): cuBLAS bf16 8192^3 burst, copy bandwidth
B200 = HardwareProfile(peak_flops_half=1611.4e12, mem_bandwidth=6532.9e9)


@dataclass(frozen=True)
class GemmShape:
    m: int
    k: int
    n: int
    r: int
    element_bytes: int = 2

    def __post_init__(self):
        if min(self.m, self.k, self.n) < 1:
            raise ValidationError(f"m, k, n must all be >= 1, got {(self.m, self.k, self.n)}")
        if self.r < 0:
            raise ValidationError(f"rank must be >= 0, got {self.r}")
        if self.element_bytes < 1:
            raise ValidationError("element_bytes must be >= 1")
        if self.r > min(self.n, self.k):
            warnings.warn(
                f"rank {self.r} exceeds min(n, k) = {min(self.n, self.k)}; low-rank factorization buys nothing",
                stacklevel=2,
            )


@dataclass(frozen=True)
class KernelTraffic:
    kernel: str
    bytes_read: int
    bytes_written: int

    @property
    def total_bytes(self) -> int:
        return self.bytes_read + self.bytes_written


@dataclass(frozen=True)
class TrafficReport:
    variant: str
    pass_name: str
    kernels: tuple

    @property
    def bytes_read(self) -> int:
        return sum(k.bytes_read for k in self.kernels)

    @property
    def bytes_written(self) -> int:
        return sum(k.bytes_written for k in self.kernels)

    @property
    def total_bytes(self) -> int:
        return self.bytes_read + self.bytes_written

    def to_dict(self) -> dict:
        return {
            "variant": self.variant,
            "pass": self.pass_name,
            "kernels": [
                {"kernel": k.kernel, "bytes_read": k.bytes_read, "bytes_written": k.bytes_written}
                for k in self.kernels
            ],
            "bytes_read": self.bytes_read,
            "bytes_written": self.bytes_written,
            "total_bytes": self.total_bytes,
        }


# (name, reads, writes); unit "e" = element bytes, "mask" = 1 B, "f32" = 4 B, "byte" = 1 B
# (with the "mk8" size: the bit-packed keep mask, m x ceil(k/8) bytes)
_E, _M, _F, _B = "e", "mask", "f32", "byte"
_TABLE = {
    ("frozen", "forward"): [
        ("base_gemm", [(_E, "mk"), (_E, "kn")], [(_E, "mn")]),
    ],
    ("frozen", "backward"): [
        ("grad_input_gemm", [(_E, "mn"), (_E, "kn")], [(_E, "mk")]),
        ("grad_weight_gemm", [(_E, "mk"), (_E, "mn")], [(_E, "kn")]),
    ],
    ("unfused", "forward"): [
        ("dropout", [(_E, "mk")], [(_E, "mk"), (_M, "mk")]),
        ("down_proj_gemm", [(_E, "mk"), (_E, "kr")], [(_E, "mr")]),
        ("up_proj_gemm", [(_E, "mr"), (_E, "rn")], [(_E, "mn")]),
        ("base_gemm", [(_E, "mk"), (_E, "kn")], [(_E, "mn")]),
        ("add_scale", [(_E, "mn"), (_E, "mn")], [(_E, "mn")]),
    ],
    ("unfused", "backward"): [
        ("grad_up_input_gemm", [(_E, "mn"), (_E, "rn")], [(_E, "mr")]),
        ("grad_up_weight_gemm", [(_E, "mr"), (_E, "mn")], [(_E, "rn")]),
        ("grad_down_input_gemm", [(_E, "mr"), (_E, "kr")], [(_E, "mk")]),
        ("grad_down_weight_gemm", [(_E, "mk"), (_E, "mr")], [(_E, "kr")]),
        ("grad_base_input_gemm", [(_E, "mn"), (_E, "kn")], [(_E, "mk")]),
        ("dropout_grad_accum", [(_E, "mk"), (_E, "mk"), (_M, "mk")], [(_E, "mk")]),
    ],
    ("fused", "forward"): [
        ("dropout_down_proj_fused", [(_E, "mk"), (_E, "kr")], [(_E, "mk"), (_M, "mk"), (_E, "mr")]),
        ("base_gemm_epilogue_fused", [(_E, "mk"), (_E, "kn"), (_E, "mr"), (_E, "rn")], [(_E, "mn")]),
    ],
    ("fused", "backward"): [
        ("grad_up_fused", [(_E, "mn"), (_E, "mr"), (_E, "rn")], [(_E, "mr"), (_E, "rn")]),
        ("grad_down_fused", [(_E, "mk"), (_E, "mr"), (_E, "kr")], [(_E, "kr"), (_E, "mk")]),
        ("grad_base_accum_fused", [(_E, "mn"), (_E, "kn"), (_E, "mk"), (_M, "mk")], [(_E, "mk")]),
    ],
    ("b200_minimal", "forward"): [
        ("dropout_down_proj_fused", [(_E, "mk"), (_E, "kr")], [(_E, "mr")]),
        ("base_gemm_epilogue_fused", [(_E, "mk"), (_E, "kn"), (_E, "mr"), (_E, "rn")], [(_E, "mn")]),
    ],
    ("b200_minimal", "backward"): [
        ("grad_up_fused", [(_E, "mn"), (_E, "rn"), (_E, "mr")], [(_E, "mr"), (_F, "rn")]),
        ("grad_down_fused", [(_E, "mk"), (_E, "mr")], [(_F, "kr")]),
        ("grad_base_accum_fused", [(_E, "mn"), (_E, "kn"), (_E, "mr"), (_E, "kr")], [(_E, "mk")]),
    ],
    # what the built kernels move with dropout on: ① writes the Philox keep mask
    # bit-packed (m x k/8 bytes) so ④ and ⑤ read it instead of re-running Philox
    ("b200_built", "forward"): [
        ("dropout_down_proj_fused", [(_E, "mk"), (_E, "kr")], [(_E, "mr"), (_B, "mk8")]),
        ("base_gemm_epilogue_fused", [(_E, "mk"), (_E, "kn"), (_E, "mr"), (_E, "rn")], [(_E, "mn")]),
    ],
    ("b200_built", "backward"): [
        ("grad_up_fused", [(_E, "mn"), (_E, "rn"), (_E, "mr")], [(_E, "mr"), (_F, "rn")]),
        ("grad_down_fused", [(_E, "mk"), (_E, "mr"), (_B, "mk8")], [(_F, "kr")]),
        ("grad_base_accum_fused", [(_E, "mn"), (_E, "kn"), (_E, "mr"), (_E, "kr"), (_B, "mk8")], [(_E, "mk")]),
    ],
}


def _bytes(terms, sizes: dict, unit: dict) -> int:
    return sum(unit[u] * sizes[mono] for u, mono in terms)


def traffic(shape: GemmShape, pass_name: str, variant: str) -> TrafficReport:
    """Per-kernel DRAM bytes of one pass of one execution variant (rank 0 = frozen,
    trainable base linear, as in the reference)."""
    if pass_name not in PASSES:
        raise ValidationError(f"pass must be one of {PASSES}, got {pass_name!r}")
    if variant not in VARIANTS:
        raise ValidationError(f"variant must be one of {VARIANTS}, got {variant!r}")
    m, k, n, r = shape.m, shape.k, shape.n, shape.r
    sizes = {"mk": m * k, "mn": m * n, "kn": k * n, "mr": m * r, "kr": k * r, "rn": r * n, "mk8": m * -(-k // 8)}
    unit = {_E: shape.element_bytes, _M: MASK_BYTES, _F: 4, _B: 1}
    if r == 0:
        key = "frozen"
    elif variant in ("fused_lora", "fused_multi_lora"):
        key = "fused"
    else:
        key = variant
    rows = [KernelTraffic(name, _bytes(rd, sizes, unit), _bytes(wr, sizes, unit))
            for name, rd, wr in _TABLE[(key, pass_name)]]
    if r and variant == "fused_multi_lora":
        rows.append(KernelTraffic("adapter_routing_table", math.ceil(m / ROUTING_TILE_ROWS) * ROUTING_ENTRY_BYTES, 0))
    return TrafficReport(variant=variant, pass_name=pass_name, kernels=tuple(rows))


def roundtrip_bytes(shape: GemmShape, variant: str) -> int:
    return sum(traffic(shape, p, variant).total_bytes for p in PASSES)


def arithmetic_intensity(r: int, n: int, m: int) -> float:
    """Eq. 2: 1 / (1/r + 1/n + 1/m) FLOP per byte."""
    if min(r, n, m) < 1:
        raise ValidationError(f"r, n, m must all be >= 1, got {(r, n, m)}")
    return 1.0 / (1.0 / r + 1.0 / n + 1.0 / m)


def down_projection_intensity(r: int, k: int, m: int) -> float:
    """2mkr FLOPs over the half-precision bytes of X, A and S: 1 / (1/r + 1/k + 1/m)."""
    if min(r, k, m) < 1:
        raise ValidationError(f"r, k, m must all be >= 1, got {(r, k, m)}")
    return 1.0 / (1.0 / r + 1.0 / k + 1.0 / m)


@dataclass(frozen=True)
class MemoryFootprint:
    full_ft_bytes: int
    lora_bytes: int
    reduction_factor: float
    trainable_fraction: float

    def to_dict(self) -> dict:
        return dict(full_ft_bytes=self.full_ft_bytes, lora_bytes=self.lora_bytes,
                    reduction_factor=self.reduction_factor, trainable_fraction=self.trainable_fraction)


def lora_memory_bytes(n: int, k: int, r: int) -> MemoryFootprint:
    """Model-state bytes per linear: 16nk (full FT) vs 2nk + 32r(n+k)."""
    if min(n, k, r) < 1:
        raise ValidationError(f"n, k, r must all be >= 1, got {(n, k, r)}")
    full, lora = 16 * n * k, 2 * n * k + 32 * r * (n + k)
    return MemoryFootprint(full, lora, full / lora, r * (n + k) / (n * k))


def lora_flops(m: int, k: int, n: int, r: int) -> dict:
    """Algorithmic FLOPs of one fwd+bwd with frozen W."""
    fwd = 2 * m * k * n + 2 * m * r * (k + n)
    bwd = 2 * m * n * k + 4 * m * r * (k + n)
    return {"forward": fwd, "backward": bwd, "total": fwd + bwd}
