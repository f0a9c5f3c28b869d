"""GPU parity on the BASELINE-shaped workflows: many labels (registration-like
gamma > 0 priors, L up to 125), interactive rounds with dynamic basis size
(c3-like), and the full-size c1 / c2 2-D configs, against the oracle."""

import numpy as np
import pytest

import paper_1607_04174_b200 as swb
from oracle import rw_oracle as O

pytestmark = pytest.mark.gpu


def _eig_pack(img, dims, beta, mode, conn, m):
    lap = O.build_laplacian(img, dims, beta, mode, conn)
    vals, vecs = np.linalg.eigh(lap.matrix.toarray())
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=beta,
                            eigen=swb.EigenBasis(np.asfortranarray(vecs[:, :m]), vals[:m]), d_sqrt=lap.d_sqrt,
                            provenance=swb.PackProvenance(image.content_hash()))
    return pack, image, lap, vecs[:, :m], vals[:m]


def _qr_pack(img, dims, beta, mode, conn, m, seed):
    lap = O.build_laplacian(img, dims, beta, mode, conn)
    rng = np.random.default_rng(seed)
    V = np.linalg.qr(rng.standard_normal((img.size, m)))[0]
    lam = np.sort(rng.uniform(1e-4, 1e-1, m))
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=beta, eigen=swb.EigenBasis(np.asfortranarray(V), lam),
                            d_sqrt=lap.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    return pack, image, lap, V, lam


@pytest.mark.parametrize("k,n_seeds", [(27, 0), (27, 30), (125, 0), (12, 15)])
def test_many_label_priors_solve(cuda_ok, k, n_seeds):
    dims = (10, 10, 10)
    rng = np.random.default_rng(k + n_seeds)
    n = 1000
    img = np.clip(rng.random(n), 0, 1)
    m_use = max(80, k + 25)
    pack, image, lap, V, lam = _eig_pack(img, dims, 50.0, "abs", 6, m_use + 16)
    pri = rng.random((n, k)) ** 4
    pri /= pri.sum(axis=1, keepdims=True)
    seeds = np.sort(rng.choice(n, n_seeds, replace=False)) if n_seeds else np.zeros(0, np.int64)
    labs = rng.integers(0, k, n_seeds)
    prob = swb.LabelProblem(num_labels=k, seeds=swb.SeedPartition(n, seeds, labs), priors=pri, gamma=1.0)
    f = swb.solve_fast(pack, lap, prob, m_use=m_use, want_field=True)
    u = O.solve_fast(V, lam, lap.d_sqrt, lap.matrix, seeds, labs, k, gamma=1.0, priors=pri, m_use=m_use)
    np.testing.assert_allclose(f.values, u, atol=1e-10)
    gap = O.top2_gap(u)
    lab = swb.hard_labels(f).labels
    assert not ((lab != O.hard_labels(u)) & (gap > 1e-9)).any()


def test_registration_like_select_m_with_label_subset(cuda_ok):
    dims = (12, 12, 8)
    n = int(np.prod(dims))
    rng = np.random.default_rng(5)
    img = np.clip(rng.random(n), 0, 1)
    pack, image, lap, V, lam = _eig_pack(img, dims, 50.0, "abs", 6, 64)
    k = 125
    pri = np.exp(-rng.random((n, k)) * 8)
    pri /= pri.sum(axis=1, keepdims=True)
    prob = swb.LabelProblem(num_labels=k, seeds=swb.SeedPartition(n, [], []), priors=pri, gamma=1.0)
    pol = swb.AdaptivePolicy(epsilon=0.05, stride=4, grid_extents=(5, 5, 5))
    m, info = swb.select_m(pack, prob, pol)
    m_o, info_o = O.select_m(V, lap.d_sqrt, [], [], k, priors=pri, epsilon=0.05, stride=4, grid_extents=(5, 5, 5))
    assert m == m_o and info["saturated"] == info_o["saturated"]
    np.testing.assert_allclose(np.array([s["g"] for s in info["steps"]]), np.array([s["g"] for s in info_o["steps"]]),
                               rtol=1e-9, atol=1e-10)
    assert len(info["steps"][0]["g"]) == 8  # {0,4}^3 of the 5x5x5 grid


def test_c3_like_interactive_rounds(cuda_ok):
    """Rounds of growing seeds + one beta update + select_m + solve (c3 workflow, small)."""
    dims = (16, 16, 16)
    n = 4096
    rng = np.random.default_rng(3)
    x, y, z = np.meshgrid(*[np.arange(16.0)] * 3, indexing="ij")
    inside = (((x - 7.5) / 5) ** 2 + ((y - 7.5) / 4) ** 2 + ((z - 7.5) / 3) ** 2 <= 1).reshape(-1, order="F")
    img = np.clip(np.where(inside, 0.65, 0.35) + rng.normal(0, 0.08, n), 0, 1)
    pack, image, lap0, V, lam = _qr_pack(img, dims, 100.0, "sq", 6, 48, 11)
    dp = swb.to_device(pack, image=image, connectivity=6, weight_mode="sq")
    up = swb.update_basis(dp, image, 140.0)
    lap1 = O.build_laplacian(img, dims, 140.0, "sq", 6)
    V1, lam1, _, _, _ = O.first_order_update(V, lam, lap0, lap1)
    truth = inside.astype(int)
    seeds, labs = np.zeros(0, np.int64), np.zeros(0, np.int64)
    for rnd in range(3):
        r = np.random.default_rng([3, 1, rnd])
        for lab in (0, 1):
            cand = np.setdiff1d(np.flatnonzero(truth == lab), seeds)
            pick = r.choice(cand, 15, replace=False)
            seeds = np.concatenate([seeds, pick])
            labs = np.concatenate([labs, np.full(15, lab)])
        o = np.argsort(seeds)
        seeds, labs = seeds[o], labs[o]
        prob = swb.LabelProblem(num_labels=2, seeds=swb.SeedPartition(n, seeds, labs))
        m, info = swb.select_m(up, prob, swb.AdaptivePolicy(epsilon=1e-3))
        m_o, info_o = O.select_m(V1, lap1.d_sqrt, seeds, labs, 2, epsilon=1e-3)
        assert m == m_o
        f = swb.solve_fast(up, up.laplacian, prob, m_use=m, want_field=True)
        u = O.solve_fast(V1, lam1, lap1.d_sqrt, lap1.matrix, seeds, labs, 2, m_use=m)
        np.testing.assert_allclose(f.values, u, atol=1e-9)


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_full_size_2d_configs(cuda_ok, cfg):
    """Full c1 (128^2, K=50) / c2 (512^2 8-conn + 32x32 cut, K=200 -> K=64 here)
    with seeded orthonormal bases: update + solve vs the oracle."""
    from paper_1607_04174_b200 import workloads as W
    w = W.make_image(cfg)
    p = w.params
    m = p["m"] if cfg == "c1" else 64
    pack, image, lap0, V, lam = _qr_pack(w.intensities, w.dims, p["beta0"], p["weight_mode"], p["connectivity"], m, 1)
    dp = swb.to_device(pack, image=image, connectivity=p["connectivity"], weight_mode=p["weight_mode"])
    cut = None
    if cfg == "c2":
        rng = np.random.default_rng([2, 3])
        x0, y0 = (int(v) for v in rng.integers(0, 512 - 32, 2))
        cut = O.block_cut_mask(w.dims, x0, y0, size=32, connectivity=8)
    up = swb.update_basis(dp, image, p["beta1"], cut_edges=cut)
    lap1 = O.build_laplacian(w.intensities, w.dims, p["beta1"], p["weight_mode"], p["connectivity"], cut_edges=cut)
    V1, lam1, _, _, _ = O.first_order_update(V, lam, lap0, lap1)
    np.testing.assert_allclose(up.lambda_hat, lam1, rtol=1e-9, atol=1e-13)
    seeds, labs = W.seeds_for(w)
    prob = swb.LabelProblem(num_labels=p["labels"], seeds=swb.SeedPartition(w.truth.size, seeds, labs))
    f = swb.solve_fast(up, up.laplacian, prob, want_field=True)
    u = O.solve_fast(V1, lam1, lap1.d_sqrt, lap1.matrix, seeds, labs, p["labels"])
    np.testing.assert_allclose(f.values, u, atol=1e-9)
    gap = O.top2_gap(u)
    assert not ((swb.hard_labels(f).labels != O.hard_labels(u)) & (gap > 1e-9)).any()
