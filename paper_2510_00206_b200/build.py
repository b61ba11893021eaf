"""Build the sm_100a shared library ``liblorafusion_b200.so`` in-tree with nvcc.

The library is a plain C-ABI shared object (include/lorafusion_b200.h): nvcc compiles
each ``csrc/*.cu`` for ``-gencode arch=compute_100a,code=sm_100a`` (the `a` target is
required for tcgen05/TMA PTX) and links them with the static CUDA runtime, so the
product has no dependency on torch's bundled runtime version. The object lands next to
this file so it travels with a repo snapshot to the GPU box.

Usage: ``python -m paper_2510_00206_b200.build [--force] [--debug]``
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
INCLUDE = REPO / "include"
LIB_NAME = "liblorafusion_b200.so"
LIB_PATH = PKG_DIR / LIB_NAME
BUILD_DIR = PKG_DIR / "_build"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found: the CUDA 12.9 toolkit is required to build lorafusion_b200")
    return cand


def _extra_flags() -> list[str]:
    """LF_EXTRA_NVCC: extra nvcc flags for A/B experiments (e.g. -DLF_SUSPEND_NS=0)."""
    return os.environ.get("LF_EXTRA_NVCC", "").split()


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _fingerprint(debug: bool) -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*")) + list(INCLUDE.glob("*.h"))):
        if p.is_file():
            h.update(p.name.encode())
            h.update(p.read_bytes())
    h.update(repr((ARCH_FLAGS, debug, _extra_flags())).encode())
    return h.hexdigest()[:16]


def build(force: bool = False, debug: bool = False, verbose: bool = False) -> Path:
    """Compile every kernel source and link the shared library; returns its path."""
    stamp = PKG_DIR / ".lib_fingerprint"
    fp = _fingerprint(debug)
    if not force and LIB_PATH.exists() and stamp.exists() and stamp.read_text().strip() == fp:
        return LIB_PATH
    nvcc = _nvcc()
    BUILD_DIR.mkdir(exist_ok=True)
    opt = ["-O0", "-G"] if debug else ["-O3"]
    common = [
        *ARCH_FLAGS,
        *opt,
        *_extra_flags(),
        "-lineinfo",
        "-std=c++17",
        "-Xcompiler",
        "-fPIC,-O3,-fvisibility=hidden",
        "-I",
        str(INCLUDE),
        "-I",
        str(CSRC),
    ]

    def compile_one(src: Path) -> Path:
        obj = BUILD_DIR / (src.stem + ".o")
        cmd = [nvcc, *common, "-Xptxas", "-v", "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
        if verbose:
            sys.stderr.write(res.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH_FLAGS, "-shared", "--cudart", "static", "-o", str(tmp), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    os.replace(tmp, LIB_PATH)
    stamp.write_text(fp)
    return LIB_PATH


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--debug", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    args = ap.parse_args()
    print(build(force=args.force, debug=args.debug, verbose=args.verbose))


if __name__ == "__main__":
    main()
