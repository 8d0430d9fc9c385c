import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity of the sm_100a engine")
    config.addinivalue_line("markers", "slow: long-running CPU check")


def _cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def emu():
    """TEST-ONLY host emulation of the device engine (build/libmfsim_emu.so)."""
    from paper_2603_17456_b200.native import Native
    path = os.path.join(ROOT, "build", "libmfsim_emu.so")
    if not os.path.exists(path):
        pytest.skip("emulation library not built")
    return Native(path)


@pytest.fixture(scope="session")
def product():
    from paper_2603_17456_b200.native import product as p
    return p()
