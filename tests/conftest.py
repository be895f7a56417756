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


# The unmodified reference package: the read-only source tree in this
# container, or its pip install under baseline/_ref (git-ignored; it travels
# to the GPU box with the snapshot, /root/reference does not).
REFERENCE_PATHS = [Path("/root/reference/pkg/src"), ROOT / "baseline" / "_ref"]


def reference_path():
    for p in REFERENCE_PATHS:
        if (p / "blockfuse" / "__init__.py").exists():
            return p
    return None


@pytest.fixture(scope="session")
def reference():
    """The reference package `blockfuse`, or skip when it is unavailable."""
    p = reference_path()
    if p is None:
        pytest.skip("reference package not available")
    if str(p) not in sys.path:
        sys.path.append(str(p))
    import blockfuse
    import blockfuse.bench  # noqa: F401
    import blockfuse.runtime  # noqa: F401
    return blockfuse
