import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")


@pytest.fixture(scope="session", autouse=True)
def _built_lib():
    from paper_2603_16104_b200 import build
    build.build()
    yield


def has_reference_lib() -> bool:
    from oracle import refpy
    return refpy.LIB.exists() or Path("/root/reference/proj/src").exists()


needs_ref = pytest.mark.skipif(not has_reference_lib(), reason="reference library not built")
