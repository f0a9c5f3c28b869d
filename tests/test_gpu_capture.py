"""CapturedStep: CUDA-graph replays of chained update_and_solve steps (c1
shape) give the same eigenvalues, basis and labels as the eager chain."""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = Path(__file__).resolve().parent.parent


def _setup():
    sys.path.insert(0, str(ROOT))
    import bench
    state = bench.setup_gpu("c1", None, 50, 0)
    state["method"] = "first_order"
    return bench, state


def test_captured_chain_matches_eager(cuda_ok):
    from paper_1607_04174_b200.capture import CapturedStep
    bench, st_e = _setup()
    _, st_g = _setup()
    p = st_e["params"]

    def two(state):
        x = state["pack"]
        x.ensure_vtg()
        f0 = bench.gpu_step(state, 0)
        f1 = bench.gpu_step(state, 1)
        z = state["pack"]
        x.values_dev.copy_(z.values_dev)
        x.vtg.copy_(z.vtg)
        state["pack"] = x
        return f0, f1

    cs = CapturedStep(lambda: two(st_g), warmup=2)     # 4 eager steps (the capture executes nothing)
    # the eager reference: the same number of chained steps
    for i in range(4):
        bench.gpu_step(st_e, i)
    for r in range(3):
        f0, f1 = cs.replay()
        cs.check()
        for i in range(2):
            fe = bench.gpu_step(st_e, i)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(f1.labels_dev.cpu().numpy(), fe.labels_dev.cpu().numpy())
        np.testing.assert_allclose(st_g["pack"].values_dev.cpu().numpy(), st_e["pack"].values_dev.cpu().numpy(),
                                   rtol=0, atol=1e-15)
        m = st_e["pack"].m
        np.testing.assert_allclose(st_g["pack"].V[:, :m].cpu().numpy(), st_e["pack"].V[:, :m].cpu().numpy(),
                                   rtol=0, atol=1e-14)
    assert p["labels"] == 2
