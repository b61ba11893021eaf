"""LoRAFusion-B200: B200-native FusedLoRA / FusedMultiLoRA (arXiv 2510.00206).

Public API
  FusedLoRA, FusedMultiLoRA          nn.Modules (PEFT parameter names lora_A / lora_B)
  FusedLoRAGroup, FusedMultiLoRAGroup  projections sharing one input (q/k/v, gate/up): ②/④/⑤ as
                                     one launch each for the group
  fused_lora, fused_multi_lora       functional forms (autograd; torch.ops.lorafusion_b200.lora_fwd/_bwd)
  fused_lora_group, fused_multi_lora_group   the group forms (torch.ops.lorafusion_b200.lora_group_*)
  invalidate_operand_caches          forget cached bf16 adapter operands after out-of-optimizer updates
  AdapterConfig, Segment, LayerPlan  adapter hyper-parameters and microbatch segment tables
  dropout_keep_mask                  SPEC.md §3 mask the kernels regenerate
  traffic, GemmShape, ...            DRAM-traffic model mirroring lorasched.costmodel
  unfused_lora                       the PEFT-style torch baseline (cuBLAS + elementwise)
  unfused_multi_lora                 its per-segment multi-adapter form

The compute path is the sm_100a shared library liblorafusion_b200.so (C ABI in
include/lorafusion_b200.h). There is no CPU fallback.
"""
from .errors import ExtensionMissingError, KernelError, LoRAFusionError, ValidationError
from .functional import (dropout_keep_mask, fused_lora, fused_lora_group, fused_multi_lora, fused_multi_lora_group,
                         invalidate_operand_caches)
from .modules import FusedLoRA, FusedLoRAGroup, FusedMultiLoRA, FusedMultiLoRAGroup
from .plan import AdapterConfig, LayerPlan, Segment, padded_rank, segments_from_lengths
from .costmodel import (
    B200,
    H100_SXM,
    VARIANTS,
    GemmShape,
    HardwareProfile,
    KernelTraffic,
    TrafficReport,
    arithmetic_intensity,
    down_projection_intensity,
    lora_memory_bytes,
    roundtrip_bytes,
    traffic,
)
from .baseline import unfused_lora, unfused_multi_lora

__all__ = [
    "AdapterConfig",
    "B200",
    "ExtensionMissingError",
    "FusedLoRA",
    "FusedLoRAGroup",
    "FusedMultiLoRA",
    "FusedMultiLoRAGroup",
    "GemmShape",
    "H100_SXM",
    "HardwareProfile",
    "KernelError",
    "KernelTraffic",
    "LayerPlan",
    "LoRAFusionError",
    "Segment",
    "TrafficReport",
    "VARIANTS",
    "ValidationError",
    "arithmetic_intensity",
    "down_projection_intensity",
    "dropout_keep_mask",
    "fused_lora",
    "fused_lora_group",
    "fused_multi_lora",
    "fused_multi_lora_group",
    "invalidate_operand_caches",
    "lora_memory_bytes",
    "padded_rank",
    "roundtrip_bytes",
    "segments_from_lengths",
    "traffic",
    "unfused_lora",
    "unfused_multi_lora",
]
