"""The C-ABI shared library: loads, exports every symbol include/*.h declares, matches the
ctypes struct layout, and rejects bad arguments with LF_E_INVALID before touching a GPU."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from paper_2510_00206_b200 import _lib
from paper_2510_00206_b200.errors import ValidationError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lorafusion_b200.h")


def _declared_symbols() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"LF_API\s+[\w\s\*]+?\b(lf_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    declared = _declared_symbols()
    assert declared, "no LF_API declarations found"
    assert sorted(_lib.EXPORTED_SYMBOLS) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (lf_\w+)", out))
    assert set(declared) <= exported, set(declared) - exported


def test_abi_version(lib):
    assert lib.lf_abi_version() == _lib.LF_ABI_VERSION


def test_library_is_sm100a_only():
    """The shared object carries sm_100a SASS (tcgen05 / TMA instructions) and nothing else."""
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCMMA" in sass, "no tcgen05.mma (UTC*MMA) in SASS"
    assert "UTMALDG" in sass, "no TMA loads (UTMALDG) in SASS"


def test_struct_layout_matches_c(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "lorafusion_b200.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(LfSegment), sizeof(LfProblem),"
        " offsetof(LfProblem, segments), offsetof(LfProblem, routes), offsetof(LfProblem, keep_mask),"
        " offsetof(LfProblem, workspace), offsetof(LfProblem, workspace_bytes), offsetof(LfProblem, keep_bits),"
        " offsetof(LfProblem, offset_dev));"
        "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    P = _lib.LfProblem
    want = [ctypes.sizeof(_lib.LfSegment), ctypes.sizeof(P), P.segments.offset, P.routes.offset, P.keep_mask.offset,
            P.workspace.offset, P.workspace_bytes.offset, P.keep_bits.offset, P.offset_dev.offset]
    assert got == want


def test_workspace_bytes(lib):
    assert _lib.workspace_bytes(8192, 16) >= 8192 * 16 * 4 + 64 * 4
    assert _lib.workspace_bytes(0, 0) == 0
    assert _lib.workspace_bytes(1, 16) % 256 == 0


def _grad_up_grid(lib, m, n, R, sms=148):
    ns, ms = ctypes.c_int32(), ctypes.c_int32()
    rc = lib.lf_grad_up_grid(m, n, R, sms, ctypes.byref(ns), ctypes.byref(ms))
    return rc, ns.value, ms.value


@pytest.mark.parametrize("m,n,R", [(16384, 28672, 16), (2048, 28672, 16), (4096, 28672, 16), (8192, 14336, 16),
                                   (8192, 4096, 16), (8192, 1024, 16), (16384, 8192, 16), (128, 1024, 16),
                                   (8192, 4096, 128), (8192, 14336, 128), (300, 200, 64)])
def test_grad_up_grid_one_wave_and_bounded_tail(lib, m, n, R):
    """③'s CTA grid (host logic, no GPU): one resident wave (a grid wider than the SMs ran
    C4 gate/up in two waves, 275 vs 152 µs), at most 8 n-subtiles per CTA (their dB partials
    are flushed at the CTA's end), and the dB/dŜ accumulators within TMEM's 512 columns."""
    rc, ns, ms = _grad_up_grid(lib, m, n, R)
    assert rc == 0, _lib.last_error()
    tiles_m, tiles_n = -(-m // 128), -(-n // 128)
    assert 1 <= ns <= tiles_n and 1 <= ms <= tiles_m
    assert ns * ms <= 148
    nsub = -(-tiles_n // ns)
    assert nsub <= 8 and (2 + nsub) * R <= 512


def test_grad_up_grid_c4_gate_and_rejects(lib):
    assert _grad_up_grid(lib, 16384, 28672, 16)[1:] == (28, 5)
    assert _grad_up_grid(lib, 0, 4096, 16)[0] == _lib.LF_E_INVALID
    assert _grad_up_grid(lib, 8192, 4096, 24)[0] == _lib.LF_E_INVALID  # not a multiple of 16
    assert _grad_up_grid(lib, 8192, 4096, 256)[0] == _lib.LF_E_INVALID  # beyond LF_MAX_RANK_TOTAL


def _problem(m=256, k=64, n=64, R=16, segs=((0, 256, 0, 16, 2.0, 0.1),)):
    p = _lib.LfProblem()
    p.m, p.k, p.n, p.rank_total = m, k, n, R
    p.num_segments = len(segs)
    for i, (r0, r1, c0, r, sc, dp) in enumerate(segs):
        d = p.segments[i]
        d.row_start, d.row_end, d.col_start, d.rank, d.scaling, d.dropout_p = r0, r1, c0, r, sc, dp
    return p


BAD = {
    "k_not_multiple_of_8": dict(k=60),
    "n_not_multiple_of_8": dict(n=36),
    "m_zero": dict(m=0),
    "rank_total_not_16": dict(R=24, segs=((0, 256, 0, 16, 2.0, 0.0),)),
    "rank_total_too_big": dict(R=144, segs=((0, 256, 0, 16, 2.0, 0.0),)),
    "segment_rank_not_16": dict(segs=((0, 256, 0, 8, 2.0, 0.0),)),
    "segment_rows_outside": dict(segs=((0, 300, 0, 16, 2.0, 0.0),)),
    "segments_unsorted": dict(R=32, segs=((128, 256, 0, 16, 2.0, 0.0), (0, 128, 16, 16, 2.0, 0.0))),
    "segments_overlap_cols": dict(R=32, segs=((0, 128, 0, 16, 2.0, 0.0), (128, 256, 8, 16, 2.0, 0.0))),
    "segments_partial_overlap_cols": dict(R=32, segs=((0, 128, 0, 32, 2.0, 0.0), (128, 256, 16, 16, 2.0, 0.0))),
    "dropout_one": dict(segs=((0, 256, 0, 16, 2.0, 1.0),)),
    "dropout_negative": dict(segs=((0, 256, 0, 16, 2.0, -0.1),)),
    "scaling_nan": dict(segs=((0, 256, 0, 16, float("nan"), 0.0),)),
}


@pytest.mark.parametrize("name", sorted(BAD))
def test_invalid_problem_rejected_before_launch(lib, name):
    p = _problem(**BAD[name])
    rc = lib.lf_build_routes(ctypes.byref(p), ctypes.c_void_p(16), None)
    assert rc == _lib.LF_E_INVALID, (name, rc, _lib.last_error())
    with pytest.raises(ValidationError):
        _lib.check(rc, "lf_build_routes")


def test_null_and_misaligned_pointers_rejected(lib):
    p = _problem()
    assert lib.lf_build_routes(ctypes.byref(p), None, None) == _lib.LF_E_INVALID
    assert "routes_out" in _lib.last_error()
    assert lib.lf_build_routes(ctypes.byref(p), ctypes.c_void_p(18), None) == _lib.LF_E_INVALID
    assert "aligned" in _lib.last_error()
    # launchers need routes and a workspace
    assert lib.lf_dropout_down_fwd(ctypes.byref(p), ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16),
                                   None) == _lib.LF_E_INVALID
    assert "routes" in _lib.last_error()
    p.routes = 4096
    assert lib.lf_dropout_down_fwd(ctypes.byref(p), ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16),
                                   None) == _lib.LF_E_INVALID
    assert "workspace" in _lib.last_error()
    assert lib.lf_grad_up(None, None, None, None, None, None, None) == _lib.LF_E_INVALID


def test_group_entry_points_reject_bad_arguments(lib):
    """ABI 5 group launchers (lf_base_fwd_group / lf_grad_input_group) and the ABI 4 one
    (lf_grad_down_group): projection counts outside 1..3, missing arrays and projections that
    do not share the input are LF_E_INVALID before anything touches a GPU."""
    P = ctypes.POINTER(_lib.LfProblem)
    V = ctypes.c_void_p
    a, b = _problem(), _problem(k=128)
    a.routes = b.routes = 4096
    probs = (P * 2)(ctypes.pointer(a), ctypes.pointer(b))
    arr = (V * 3)(16, 16, 16)
    x = V(16)
    assert lib.lf_base_fwd_group(probs, 0, x, arr, arr, arr, arr, None) == _lib.LF_E_INVALID
    assert lib.lf_base_fwd_group(probs, 4, x, arr, arr, arr, arr, None) == _lib.LF_E_INVALID
    assert lib.lf_base_fwd_group(probs, 2, x, None, arr, arr, arr, None) == _lib.LF_E_INVALID
    assert lib.lf_base_fwd_group(probs, 2, x, arr, arr, arr, arr, None) == _lib.LF_E_INVALID
    assert "share the input" in _lib.last_error()
    assert lib.lf_grad_input_group(probs, 0, arr, arr, arr, arr, x, None) == _lib.LF_E_INVALID
    assert lib.lf_grad_input_group(probs, 2, arr, arr, arr, None, x, None) == _lib.LF_E_INVALID
    assert lib.lf_grad_input_group(probs, 2, arr, arr, arr, arr, None, None) == _lib.LF_E_INVALID
    assert lib.lf_grad_input_group(probs, 2, arr, arr, arr, arr, x, None) == _lib.LF_E_INVALID
    assert "share the input" in _lib.last_error()
    assert lib.lf_grad_down_group(probs, 4, x, arr, arr, None) == _lib.LF_E_INVALID


def test_copy_column_blocks_rejects_bad_arguments(lib):
    """ABI 6 lf_copy_column_blocks: block counts outside 0..LF_MAX_COPY_BLOCKS, NULL arrays
    or pointers and column ranges past the row are LF_E_INVALID; zero blocks is a no-op."""
    V, I = ctypes.c_void_p, ctypes.c_int32
    src, dst = (V * 2)(16, 16), (V * 2)(32, 32)
    rows, ld, col, wid = (I * 2)(4, 4), (I * 2)(128, 128), (I * 2)(0, 64), (I * 2)(64, 64)
    assert lib.lf_copy_column_blocks(0, None, None, None, None, None, None, None) == _lib.LF_OK
    assert lib.lf_copy_column_blocks(-1, src, rows, ld, col, wid, dst, None) == _lib.LF_E_INVALID
    assert lib.lf_copy_column_blocks(_lib.LF_MAX_COPY_BLOCKS + 1, src, rows, ld, col, wid, dst, None) == _lib.LF_E_INVALID
    assert lib.lf_copy_column_blocks(2, src, rows, ld, col, None, dst, None) == _lib.LF_E_INVALID
    bad = (I * 2)(0, 65)
    assert lib.lf_copy_column_blocks(2, src, rows, ld, bad, wid, dst, None) == _lib.LF_E_INVALID
    assert "block 1" in _lib.last_error()
    nul = (V * 2)(16, None)
    assert lib.lf_copy_column_blocks(2, nul, rows, ld, col, wid, dst, None) == _lib.LF_E_INVALID


def test_no_gpu_reports_cuda_error_not_crash(lib):
    """A valid problem on a machine without a B200 fails with LF_E_CUDA/UNSUPPORTED, never a crash."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = _problem()
    rc = lib.lf_build_routes(ctypes.byref(p), ctypes.c_void_p(4096), None)
    assert rc in (_lib.LF_E_CUDA, _lib.LF_E_UNSUPPORTED)
    with pytest.raises(RuntimeError):
        _lib.check(rc, "lf_build_routes")


def test_product_has_no_cpu_fallback():
    """The product package never imports the oracle and refuses CPU tensors."""
    import torch

    import paper_2510_00206_b200 as pkg

    pkg_dir = os.path.dirname(pkg.__file__)
    for fn in os.listdir(pkg_dir):
        if fn.endswith(".py"):
            text = open(os.path.join(pkg_dir, fn)).read()
            assert "import oracle" not in text and "from oracle" not in text, fn
    x = torch.zeros(4, 8, dtype=torch.bfloat16)
    w = torch.zeros(8, 8, dtype=torch.bfloat16)
    a = torch.zeros(16, 8, dtype=torch.bfloat16)
    b = torch.zeros(8, 16, dtype=torch.bfloat16)
    with pytest.raises(ValidationError, match="CUDA"):
        pkg.fused_lora(x, w, a, b, 2.0)


def test_missing_library_fails_loudly(tmp_path):
    from paper_2510_00206_b200.errors import ExtensionMissingError

    with pytest.raises(ExtensionMissingError):
        _lib.load(tmp_path / "liblorafusion_b200.so")
