import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built native library")
    config.addinivalue_line("markers", "reference: needs the read-only reference checkout (container only)")
    config.addinivalue_line("markers", "slow: long-running")


def have_reference() -> bool:
    return (REFERENCE_SRC / "wap" / "__init__.py").exists()


@pytest.fixture(scope="session")
def ref_wap():
    """The reference package imported from /root/reference (only in the build container)."""
    if not have_reference():
        pytest.skip("reference checkout not present")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    import importlib

    return importlib.import_module("wap")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but CUDA is not available")
    from paper_1811_01532_b200 import _native

    _native.lib()
    return torch.device("cuda:0")
