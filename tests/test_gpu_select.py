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
