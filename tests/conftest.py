import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

GOLDEN_PATH = ROOT / "tests" / "golden" / "golden.json"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def golden():
    return json.loads(GOLDEN_PATH.read_text())


@pytest.fixture(scope="session")
def native_built():
    from paper_2601_17707_b200 import _build

    _build.build_all()
    return True


def has_gpu() -> bool:
    try:
        from paper_2601_17707_b200 import _lib

        return _lib.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu(native_built):
    if not has_gpu():
        pytest.fail("GPU test selected but no CUDA device is visible (the counter has no CPU fallback)")
    return 0


@pytest.fixture(scope="session")
def threads():
    return len(os.sched_getaffinity(0))
