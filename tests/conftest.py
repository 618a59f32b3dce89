import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))  # shared helpers (torch_ref, test_gpu_layer)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def product_lib():
    """The product C ABI library; built in-tree if missing (no fallback)."""
    from paper_2602_11686_b200 import build, _lib
    if not build.lib_path().exists():
        build.build()
    return _lib.load()


@pytest.fixture(scope="session")
def ref():
    """The reference library itself (oracle/_ref); skip where it cannot exist."""
    from oracle import ref as R
    if not R.available():
        pytest.skip("reference oracle (oracle/_ref) not built and /root/reference absent")
    return R
