import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libdco_gpu.so")
    config.addinivalue_line("markers", "slow: long-running CPU sweep")


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as r

    if not r.available():
        import oracle

        oracle.build()
    return r


@pytest.fixture(scope="session")
def gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2203_02300_b200 import dco

    dco.context()
    return dco
