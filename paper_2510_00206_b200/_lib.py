"""ctypes binding of ``liblorafusion_b200.so`` (include/lorafusion_b200.h).

The structures below mirror the C header field for field; ``check_abi()`` verifies the
sizes against the library at load time. There is no CPU fallback: if the shared library
is missing the import of any op raises :class:`ExtensionMissingError`.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import ExtensionMissingError, KernelError, ValidationError

LF_ABI_VERSION = 6
LF_MAX_SEGMENTS = 32
LF_MAX_COPY_BLOCKS = 64  # lf_copy_column_blocks blocks per call
LF_MAX_GROUP = 3  # projections of one shared-input group launch (lf_*_group)
LF_MAX_RANK_TOTAL = 128
ROUTE_TILE_ROWS = 128  # ls/costmodel.py:25
ROUTE_ENTRY_BYTES = 16  # ls/costmodel.py:26

LF_OK = 0
LF_E_INVALID = -1
LF_E_CUDA = -2
LF_E_UNSUPPORTED = -3

LIB_PATH = Path(__file__).resolve().parent / "liblorafusion_b200.so"
# LF_LIB: load another build of the same library instead (interleaved A/B runs of two builds
# on one box: tools/ab.sh "LF_LIB=_variants/a.so" "LF_LIB=_variants/b.so")
if os.environ.get("LF_LIB"):
    LIB_PATH = Path(os.environ["LF_LIB"]).resolve()

# every symbol include/lorafusion_b200.h declares
EXPORTED_SYMBOLS = (
    "lf_workspace_bytes",
    "lf_grad_up_grid",
    "lf_build_routes",
    "lf_dropout_down_fwd",
    "lf_base_fwd",
    "lf_grad_up",
    "lf_grad_down",
    "lf_grad_down_group",
    "lf_grad_up_group",
    "lf_grad_input",
    "lf_grad_input_accum",
    "lf_base_fwd_group",
    "lf_grad_input_group",
    "lf_dropout_mask",
    "lf_keep_bits",
    "lf_copy_column_blocks",
    "lf_last_error",
    "lf_abi_version",
)


class LfSegment(ctypes.Structure):
    _fields_ = [
        ("row_start", ctypes.c_int32),
        ("row_end", ctypes.c_int32),
        ("col_start", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("scaling", ctypes.c_float),
        ("dropout_p", ctypes.c_float),
        ("seed", ctypes.c_uint64),
        ("offset", ctypes.c_uint64),
    ]


class LfProblem(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("rank_total", ctypes.c_int32),
        ("num_segments", ctypes.c_int32),
        ("row_base", ctypes.c_int32),
        ("segments", LfSegment * LF_MAX_SEGMENTS),
        ("routes", ctypes.c_void_p),
        ("keep_mask", ctypes.c_void_p),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_size_t),
        ("keep_bits", ctypes.c_void_p),
        ("offset_dev", ctypes.c_void_p),
    ]


_P = ctypes.POINTER(LfProblem)
_V = ctypes.c_void_p
_SIGNATURES = {
    "lf_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int32]),
    "lf_grad_up_grid": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]),
    "lf_build_routes": (ctypes.c_int, [_P, _V, _V]),
    "lf_dropout_down_fwd": (ctypes.c_int, [_P, _V, _V, _V, _V]),
    "lf_base_fwd": (ctypes.c_int, [_P, _V, _V, _V, _V, _V, _V]),
    "lf_grad_up": (ctypes.c_int, [_P, _V, _V, _V, _V, _V, _V]),
    "lf_grad_down": (ctypes.c_int, [_P, _V, _V, _V, _V]),
    "lf_grad_down_group": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int32, _V, ctypes.POINTER(_V),
                                          ctypes.POINTER(_V), _V]),
    "lf_grad_up_group": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int32, ctypes.POINTER(_V), ctypes.POINTER(_V),
                                        ctypes.POINTER(_V), ctypes.POINTER(_V), ctypes.POINTER(_V), _V]),
    "lf_grad_input": (ctypes.c_int, [_P, _V, _V, _V, _V, _V, _V]),
    "lf_grad_input_accum": (ctypes.c_int, [_P, _V, _V, _V, _V, _V, _V]),
    "lf_base_fwd_group": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int32, _V, ctypes.POINTER(_V),
                                         ctypes.POINTER(_V), ctypes.POINTER(_V), ctypes.POINTER(_V), _V]),
    "lf_grad_input_group": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int32, ctypes.POINTER(_V),
                                           ctypes.POINTER(_V), ctypes.POINTER(_V), ctypes.POINTER(_V), _V, _V]),
    "lf_dropout_mask": (ctypes.c_int, [_P, _V, _V]),
    "lf_keep_bits": (ctypes.c_int, [_P, _V, _V]),
    "lf_copy_column_blocks": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(_V), ctypes.POINTER(ctypes.c_int32),
                                             ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                                             ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_V), _V]),
    "lf_last_error": (ctypes.c_char_p, []),
    "lf_abi_version": (ctypes.c_int, []),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library. Raises ExtensionMissingError if absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise ExtensionMissingError(
                f"{p.name} is not built (expected at {p}); run `python -m paper_2510_00206_b200.build` "
                "or __graft_entry__.build(). There is no CPU fallback for the fused LoRA kernels."
            )
        lib = ctypes.CDLL(str(p))
        for name, (restype, argtypes) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = restype
            fn.argtypes = argtypes
        ver = lib.lf_abi_version()
        if ver != LF_ABI_VERSION:
            raise ExtensionMissingError(f"{p.name} ABI version {ver} != expected {LF_ABI_VERSION}; rebuild it")
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    return load().lf_last_error().decode(errors="replace")


def check(rc: int, what: str) -> None:
    """Map a C-ABI return code onto the package's exception types."""
    if rc == LF_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == LF_E_INVALID:
        raise ValidationError(msg)
    raise KernelError(msg)


def workspace_bytes(m: int, rank_total: int) -> int:
    return int(load().lf_workspace_bytes(m, rank_total))
