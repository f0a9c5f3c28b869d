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
    if os.environ.get("SWB_TEST_NANFILL") == "1":
        # debugging aid: every torch.empty comes back full of NaN, so a kernel
        # that lets a padding element reach a result (NaN * 0) fails loudly
        # instead of depending on what the allocator handed out
        torch.use_deterministic_algorithms(True, warn_only=True)
        torch.utils.deterministic.fill_uninitialized_memory = True
    return True
