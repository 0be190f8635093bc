import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels through the C-ABI)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _has_gpu() -> bool:
    try:
        from paper_2605_23727_b200 import _abi
        return _abi.lib().ms_device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not _has_gpu():
        pytest.fail("gpu test selected but no CUDA device is visible (the B200 path has no CPU fallback)")
    return True
