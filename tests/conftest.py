import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libbfgpu.so)")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu() -> bool:
    try:
        from paper_2206_07896_b200 import _lib
        return _lib.device_count() > 0
    except Exception:
        return False


REFERENCE_SRC = Path("/root/reference/pkg/src")


@pytest.fixture(scope="session")
def reference():
    """The reference package, when this container has it (never on the GPU box)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not available")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.append(str(REFERENCE_SRC))
    import blockfuse
    return blockfuse
