import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_v1.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a) and the built librectri_cu.so")
    config.addinivalue_line("markers", "slow: long-running property test")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test requires CUDA (run with -m 'not gpu' on CPU hosts)")
    from paper_2504_13821_b200 import _lib

    _lib.load()  # must be the in-tree sm_100a library: no fallback
    return torch.device("cuda:0")
