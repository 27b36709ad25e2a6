import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # Build the product library (and the oracle here, where the reference
    # sources exist) once per session if absent.
    from paper_2511_14124_b200 import _build
    if not os.path.exists(_build.LIB):
        _build.build()
    ref_so = os.path.join(ROOT, "oracle", "_ref", "libtencache_ref.so")
    if not os.path.exists(ref_so) and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "-j8"], check=True, capture_output=True)


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device here; runs on the GPU box")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture
def tmpd(tmp_path):
    return str(tmp_path)
