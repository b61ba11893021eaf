"""Exception types of the B200 FusedLoRA layer.

Follows the reference's convention (ls/errors.py:8-42): invalid arguments raise a
``ValueError`` subclass, so callers that catch the reference's ``ValidationError``
semantics (``except ValueError``) behave the same; device failures raise
``RuntimeError``.
"""
from __future__ import annotations


class LoRAFusionError(Exception):
    """Base class for all errors raised by this package."""


class ValidationError(LoRAFusionError, ValueError):
    """Invalid argument: shape, dtype, layout, alignment, segment table or hyper-parameter."""


class KernelError(LoRAFusionError, RuntimeError):
    """A CUDA launch or driver call failed, or the device is not a B200 (sm_100)."""


class ExtensionMissingError(LoRAFusionError, ImportError):
    """The sm_100a shared library is not built; there is no CPU fallback."""
