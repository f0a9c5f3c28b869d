import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


def csr_from(z, prefix):
    import scipy.sparse as sp
    data, idx, ptr = z[prefix + "_data"], z[prefix + "_indices"], z[prefix + "_indptr"]
    n = ptr.size - 1
    return sp.csr_matrix((data, idx, ptr), shape=(n, n))


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
