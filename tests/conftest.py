import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA engine)")


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle
    if not Oracle.available("reference"):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def eng():
    if not have_gpu():
        pytest.skip("no GPU")
    from paper_2603_08883_b200 import iqcc, native
    native.init(0)
    return iqcc
