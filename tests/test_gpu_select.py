"""GPU parity of the dynamic basis size (select_m / seed_fit / prior_residual)
against the reference golden vectors and the oracle."""

import numpy as np
import pytest

import paper_1607_04174_b200 as swb
from conftest import load_golden
from oracle import rw_oracle as O

pytestmark = pytest.mark.gpu


def _pack(V, lam, d_sqrt, dims):
    return swb.SpectralPack(dims=dims, spacing=(), beta=1.0, eigen=swb.EigenBasis(np.asfortranarray(V), lam),
                            d_sqrt=d_sqrt, provenance=swb.PackProvenance(b""))


@pytest.mark.parametrize("tag", ["default", "loose", "tight", "eps3e4"])
def test_select_m_seeds_matches_reference(cuda_ok, tag):
    z = load_golden("phantom16")
    pack = _pack(z["V"], z["lam"], z["d_sqrt"], (16, 16))
    n = z["d_sqrt"].size
    prob = swb.LabelProblem(num_labels=2, seeds=swb.SeedPartition(n, z[f"sel_{tag}_idx"], z[f"sel_{tag}_lab"]))
    m, info = swb.select_m(pack, prob, swb.AdaptivePolicy(epsilon=float(z[f"sel_{tag}_eps"])))
    assert m == int(z[f"sel_{tag}_m"])
    assert info["saturated"] == bool(z[f"sel_{tag}_sat"])
    np.testing.assert_array_equal([s["m"] for s in info["steps"]], z[f"sel_{tag}_steps_m"])
    np.testing.assert_allclose(np.array([s["f"] for s in info["steps"]]), z[f"sel_{tag}_steps_f"],
                               rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("tag,key,k", [("p_loose", "pri4", 4), ("p_tight", "pri4", 4), ("p_mid", "pri4", 4),
                                       ("ps_a", "psmooth", 2), ("ps_b", "psmooth", 2), ("ps_c", "psmooth", 2)])
def test_select_m_priors_matches_reference(cuda_ok, tag, key, k):
    z = load_golden("phantom16")
    pack = _pack(z["V"], z["lam"], z["d_sqrt"], (16, 16))
    n = z["d_sqrt"].size
    prob = swb.LabelProblem(num_labels=k, seeds=swb.SeedPartition(n, [], []), priors=z[key], gamma=1.0)
    m, info = swb.select_m(pack, prob, swb.AdaptivePolicy(epsilon=float(z[f"sel_{tag}_eps"])))
    assert m == int(z[f"sel_{tag}_m"])
    assert info["saturated"] == bool(z[f"sel_{tag}_sat"])
    np.testing.assert_allclose(np.array([s["g"] for s in info["steps"]]), z[f"sel_{tag}_steps_g"],
                               rtol=1e-9, atol=1e-10)


@pytest.mark.parametrize("n,m,s,k,bound_scale", [(3000, 40, 60, 2, 1.0), (3000, 40, 20, 3, 1.0),
                                                 (5000, 96, 150, 2, 1e-3), (2000, 30, 30, 2, 1.0)])
def test_seed_fit_schedule_matches_oracle(cuda_ok, n, m, s, k, bound_scale):
    rng = np.random.default_rng(n + m + s)
    V = np.linalg.qr(rng.standard_normal((n, m)))[0]
    d_sqrt = 1.0 + rng.random(n)
    seeds = np.sort(rng.choice(n, s, replace=False))
    labs = rng.integers(0, k, s)
    pack = _pack(V, np.linspace(0, 0.1, m), d_sqrt * bound_scale, (n, 1))
    prob = swb.LabelProblem(num_labels=k, seeds=swb.SeedPartition(n, seeds, labs))
    pol = swb.AdaptivePolicy(epsilon=1e-12)       # never passes: every step evaluated
    m_use, info = swb.select_m(pack, prob, pol)
    # the oracle, forced through every scheduled step (f values only: with
    # S < m the fit is exact and f is rounding noise around 0)
    sched = pol.schedule(m, k)
    bound = float(np.sqrt(np.sum((d_sqrt * bound_scale) ** 2)))
    u = np.zeros((s, k))
    u[np.arange(s), labs] = 1.0
    u *= (d_sqrt * bound_scale)[seeds, None]
    want = np.array([[O.seed_fit(V[seeds, :mm], u[:, c], bound) for c in range(k)] for mm in sched])
    assert len(info["steps"]) == len(sched) or not info["saturated"]
    got = np.array([st["f"] for st in info["steps"]])
    want = want[: len(got)]
    np.testing.assert_allclose(got, want, rtol=1e-8, atol=1e-10 * max(1.0, np.abs(want).max()))


def test_select_m_then_solve_refreshed(cuda_ok):
    """select_m on a refreshed pack reads columns through the permutation."""
    z = load_golden("phantom16")
    img = swb.Image((16, 16), z["intensities"])
    pack = swb.SpectralPack(dims=(16, 16), spacing=(), beta=15.0,
                            eigen=swb.EigenBasis(np.asfortranarray(z["V"]), z["lam"]), d_sqrt=z["d_sqrt"],
                            provenance=swb.PackProvenance(img.content_hash()))
    r = swb.refresh(pack, img, 45.0)
    n = 256
    prob = swb.LabelProblem(num_labels=2, seeds=swb.SeedPartition(n, z["sel_eps3e4_idx"], z["sel_eps3e4_lab"]))
    m, info = swb.select_m(r, prob, swb.AdaptivePolicy(epsilon=3e-4))
    lap = O.build_laplacian(z["intensities"], (16, 16), 45.0)
    lam, order = O.refresh(z["V"], lap)
    m_o, info_o = O.select_m(z["V"][:, order], lap.d_sqrt, z["sel_eps3e4_idx"], z["sel_eps3e4_lab"], 2,
                             epsilon=3e-4)
    assert m == m_o
    np.testing.assert_allclose(np.array([s["f"] for s in info["steps"]]),
                               np.array([s["f"] for s in info_o["steps"]]), rtol=1e-9, atol=1e-12)


def _seed_fit_gpu(V, seeds, labs, d_sqrt, k, steps, bound):
    """swb_seed_fit_schedule straight through the C ABI (row-major V)."""
    import torch

    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200.device import WORKSPACE, ptr, round_up, stream_handle
    n, m = V.shape
    ldv = round_up(m, 2)
    Vd = torch.zeros((n, ldv), dtype=torch.float64, device="cuda")
    Vd[:, :m] = torch.from_numpy(np.asarray(V, dtype=np.float64))
    s = len(seeds)
    sidx = torch.tensor(seeds, dtype=torch.int64, device="cuda")
    slab = torch.tensor(labs, dtype=torch.int32, device="cuda")
    d = torch.tensor(d_sqrt, dtype=torch.float64, device="cuda")
    st = torch.tensor(steps, dtype=torch.int32, device="cuda")
    f = torch.empty((len(steps), k), dtype=torch.float64, device="cuda")
    ws = WORKSPACE.get("seed_fit_t", _lib.size("swb_seed_fit_workspace_bytes", s, m, k, len(steps)))
    _lib.call("swb_seed_fit_schedule", ptr(Vd), ldv, None, ptr(sidx), ptr(slab), s, ptr(d), m, k, ptr(st), len(steps),
              int(max(steps)), float(bound), ptr(f), ptr(ws), ws.numel(), stream_handle())
    return f.cpu().numpy()


def test_seed_fit_known_answers(cuda_ok):
    """The reference's seed_fit closed forms (tests/test_adaptive.py): exact
    span, 0.6/0.8 projection (0.64), zero bound, active bound (ridge path)."""
    # exact span: q_s = I_3, u = e_0
    f = _seed_fit_gpu(np.eye(3), [0, 1, 2], [0, 1, 1], [1.0, 1.0, 1.0], 2, [3], 100.0)
    assert f[0, 0] < 1e-12
    # closed form: q_s = [0.6, 0.8]^T, u = [1, 0] -> 0.64
    f = _seed_fit_gpu(np.array([[0.6], [0.8]]), [0, 1], [0, 1], [1.0, 1.0], 2, [1], 100.0)
    assert abs(f[0, 0] - 0.64) < 1e-10
    # zero bound: alpha = 0, f = |u|^2 = 3
    f = _seed_fit_gpu(np.ones((4, 2)), [0, 1, 2, 3], [0, 1, 0, 0], [1.0] * 4, 2, [2], 0.0)
    assert abs(f[0, 0] - 3.0) < 1e-12
    # active bound: the minimum-norm coefficient (1e3) exceeds the bound
    q = np.array([[1e-3], [0.0]])
    f_free = _seed_fit_gpu(q, [0, 1], [0, 1], [1.0, 1.0], 2, [1], 1e9)
    assert f_free[0, 0] < 1e-12
    f_tight = _seed_fit_gpu(q, [0, 1], [0, 1], [1.0, 1.0], 2, [1], 1.0)
    assert abs(f_tight[0, 0] - (1 - 1e-3) ** 2) < 1e-3 * (1 - 1e-3) ** 2


@pytest.mark.parametrize("n,m,s,k,bound_scale,dup", [(5000, 150, 400, 2, 1e-2, False), (4000, 60, 200, 3, 1.0, True),
                                                     (4000, 60, 200, 2, 1e-2, True), (3000, 64, 64, 2, 1e-2, False)])
def test_seed_fit_both_paths_match_oracle(cuda_ok, n, m, s, k, bound_scale, dup):
    """select.cu has two paths per scheduled m: the bidiagonal ridge (square,
    well-conditioned R_m: sigma_min > 1e-6 sigma_0) and the Jacobi SVD
    (ill-conditioned or S < m).  A basis column that nearly duplicates its
    neighbour (difference 1e-9) makes every R_m past it ill-conditioned
    (sigma_min ~ 1e-9 sigma_0: kept by the reference's 1e-13 cutoff, but
    below the fast path's gate), so those steps take the Jacobi path while
    the earlier ones take the bidiagonal one; a small bound makes the ridge
    (adaptive.py:96-110) bind.  (An exactly duplicated column is not a
    well-posed comparison: the reference's left singular vector of the zero
    singular value, and so its perp, is whatever LAPACK's gesdd picks.)"""
    rng = np.random.default_rng(n + m + s + int(dup))
    V = np.linalg.qr(rng.standard_normal((n, m)))[0]
    if dup:
        V[:, m // 2] = V[:, m // 2 - 1] + 1e-9 * V[:, m // 2]
    d_sqrt = 1.0 + rng.random(n)
    seeds = np.sort(rng.choice(n, s, replace=False))
    labs = rng.integers(0, k, s)
    pack = _pack(V, np.linspace(0, 0.1, m), d_sqrt * bound_scale, (n, 1))
    prob = swb.LabelProblem(num_labels=k, seeds=swb.SeedPartition(n, seeds, labs))
    pol = swb.AdaptivePolicy(epsilon=1e-12)
    m_use, info = swb.select_m(pack, prob, pol)
    sched = pol.schedule(m, k)
    bound = float(np.sqrt(np.sum((d_sqrt * bound_scale) ** 2)))
    u = np.zeros((s, k))
    u[np.arange(s), labs] = 1.0
    u *= (d_sqrt * bound_scale)[seeds, None]
    want = np.array([[O.seed_fit(V[seeds, :mm], u[:, c], bound) for c in range(k)] for mm in sched])
    got = np.array([st["f"] for st in info["steps"]])
    assert got.shape == want.shape
    np.testing.assert_allclose(got, want, rtol=1e-8, atol=1e-10 * max(1.0, np.abs(want).max()))
