import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libncsg.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port

    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, Ref

    if not os.path.exists(REF_SO):
        pytest.skip("reference build oracle/_ref/libncsref.so not present")
    return Ref()


@pytest.fixture(scope="session")
def ncsg():
    from paper_1810_13100_b200 import ncsg as mod

    mod.lib()
    return mod
