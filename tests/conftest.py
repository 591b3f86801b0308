import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libbfgpu.so")
    config.addinivalue_line("markers", "slow: long-running")


def reference_available():
    return os.path.isdir(os.path.join(REF_SRC, "blockflow"))


@pytest.fixture(scope="session")
def ref():
    """The reference package itself (development container only)."""
    if not reference_available():
        pytest.skip("reference package not present on this machine")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import blockflow.decomp
    import blockflow.exchange
    import blockflow.halo
    import blockflow.mesh
    import blockflow.physics
    import blockflow.solver
    import blockflow.topology
    import blockflow.cli
    return blockflow


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
