import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libvibro_b200.so)")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture(scope="session")
def cuda():
    import torch
    from paper_2310_04734_b200 import _lib
    _lib.require_cuda()
    _lib.load()
    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def golden_dir():
    return ROOT / "tests" / "golden"
