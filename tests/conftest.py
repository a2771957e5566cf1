import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    _ensure_library()


def _ensure_library():
    """The in-tree .so is git-ignored: on a fresh checkout build it once (nvcc
    cross-compiles sm_100a without a GPU) so the ABI tests test the real library."""
    import shutil

    from paper_2406_03482_b200 import _lib

    if os.path.exists(_lib.LIB_PATH) or "QJL_LIB" in os.environ or shutil.which("nvcc") is None:
        return
    import __graft_entry__

    __graft_entry__.build()


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
