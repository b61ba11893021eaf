import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionstart(session):
    """A fresh checkout has no library (it is git-ignored): build it in-tree once if nvcc is
    here, so the C-ABI tests run from any order of build / test. Does nothing when it is
    current (the build is fingerprinted)."""
    import shutil

    if shutil.which("nvcc") or os.path.exists("/usr/local/cuda/bin/nvcc"):
        from paper_2510_00206_b200 import build

        build.build()


def _has_b200() -> bool:
    try:
        import torch

        return torch.cuda.is_available() and torch.cuda.get_device_capability(0) == (10, 0)
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_b200():
        return
    skip = pytest.mark.skip(reason="no B200 (sm_100) visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
