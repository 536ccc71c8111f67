import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the oracle (and the CUDA extension when missing) once per session."""
    import oracle
    if not oracle.available("restatement"):
        oracle.build(reference=True)
    from paper_1810_05762_b200 import abi
    if not os.path.exists(abi.LIB_PATH):
        from paper_1810_05762_b200 import build
        build.build()
    yield


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
