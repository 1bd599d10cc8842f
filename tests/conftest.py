import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the driver's GPU tier)")


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import load

    return load("orc")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import available, load

    if not available("ref"):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return load("ref")


@pytest.fixture(scope="session")
def sg():
    from paper_2312_12491_b200 import stagger

    return stagger
