import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    """On a host without CUDA, `gpu` tests are skipped instead of erroring
    (the driver selects them with -m gpu on a B200 box)."""
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="needs a CUDA GPU (B200)")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def lib():
    """The built libmsinfer (GPU tests): fail loudly if it is missing."""
    from paper_2504_02263_b200 import _lib
    return _lib.load()
