import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def native_lib():
    from paper_2108_05818_b200 import _build, _native
    _build.build_library()
    return _native.load()


@pytest.fixture(scope="session")
def oracle_lib():
    from paper_2108_05818_b200 import _build
    _build.build_oracle()
    from oracle import numerics
    return numerics
