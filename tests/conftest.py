import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(params=["absorbed", "unabsorbed"])
def kernel_path(request, monkeypatch):
    """Run a fused-decode test through both kernels: the V-absorbed default
    (csrc/xq_absorb.cu) and the unabsorbed remat kernel (csrc/xq_decode.cu)."""
    from paper_2508_10395_b200 import cache

    monkeypatch.setattr(cache, "FUSED_KERNEL", request.param)
    return request.param
