import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

REFERENCE_SRC = Path("/root/reference/pkg/src")
REF_INSTALL = ROOT / "baseline" / "_ref"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running parity sweeps")


def reference_headbalance():
    """The reference package itself (live oracle), or None when absent
    (e.g. on the GPU box, where /root/reference does not exist)."""
    for p in (REF_INSTALL, REFERENCE_SRC):
        if (p / "headbalance" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.append(str(p))
            try:
                import headbalance  # noqa: F401
                return headbalance
            except Exception:
                return None
    return None


@pytest.fixture(scope="session")
def cuda_device():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
