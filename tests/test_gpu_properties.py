"""GPU restatements of the reference's property / known-answer tests for the
hot path: refresh identity, null direction of a uniform image,
refresh value range / ordering / idempotence, the min-eigenvalue bound,
log-beta pack choice, full-basis exactness, constant priors, truncated row
sums, streaming parity and bitwise determinism (solve, first-order update,
precompute).  Packs come from the reference golden vectors or from the GPU
precompute."""

import numpy as np
import pytest

import paper_1607_04174_b200 as swb
from conftest import csr_from, load_golden
from oracle import rw_oracle as O

pytestmark = pytest.mark.gpu


def _golden_pack():
    z = load_golden("phantom16")
    dims = tuple(int(d) for d in z["dims"])
    img = swb.Image(dims, z["intensities"])
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=float(z["beta"]),
                            eigen=swb.EigenBasis(np.asfortranarray(z["V"]), z["lam"]), d_sqrt=z["d_sqrt"],
                            provenance=swb.PackProvenance(image_hash=img.content_hash()))
    return z, img, pack, csr_from(z, "lap")


def _seeds(n, k=2, per=3, seed=0):
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, per * k, replace=False))
    return swb.SeedPartition(n, idx, np.arange(idx.size) % k)


def test_refresh_identity(cuda_ok):
    z, img, pack, lap = _golden_pack()
    r = swb.refresh(pack, img, pack.beta)
    assert np.abs(r.lambda_hat - z["lam"]).max() < 1e-5
    prob = swb.LabelProblem(num_labels=2, seeds=_seeds(img.n_voxels), gamma=0.0)
    u0 = swb.solve_fast(pack, lap, prob, want_field=True).values
    u1 = swb.solve_fast(r, r.laplacian, prob, want_field=True).values
    assert np.abs(u0 - u1).max() <= 1e-6


def test_refresh_uniform_image_keeps_null(cuda_ok):
    img = swb.Image((6, 5), np.full(30, 0.5))
    pack = swb.precompute(img, 10.0, 8, eig_tol=1e-9)
    r = swb.refresh(pack, img, 80.0)
    assert r.lambda_hat[0] <= 1e-2


def test_refresh_range_order_idempotent(cuda_ok):
    z, img, pack, lap = _golden_pack()
    r1 = swb.refresh(pack, img, 45.0)
    r2 = swb.refresh(pack, img, 45.0)
    assert np.array_equal(r1.lambda_hat, r2.lambda_hat)
    assert r1.lambda_hat.min() >= -1e-8 and r1.lambda_hat.max() <= 2 + 1e-8
    assert np.all(np.diff(r1.lambda_hat) >= 0)


def test_refresh_min_bound(cuda_ok):
    z, img, pack, lap = _golden_pack()
    r = swb.refresh(pack, img, 33.0)
    vals = np.linalg.eigvalsh(r.laplacian.matrix.toarray())
    assert r.lambda_hat.min() >= vals[0] - 1e-8


def test_nearest_pack_log_scale_and_refresh_from_set(cuda_ok):
    z, img, _, _ = _golden_pack()
    packs = swb.PackSet(tuple(swb.precompute(img, b, 4, eig_tol=1e-9) for b in (25.0, 50.0, 100.0)))
    assert swb.nearest_pack(packs, 60.0).beta == 50.0
    assert swb.nearest_pack(packs, 90.0).beta == 100.0
    assert swb.nearest_pack(packs, 50.0).beta == 50.0
    two = swb.PackSet(tuple(swb.precompute(img, b, 16, eig_tol=1e-9) for b in (10.0, 15.0)))
    r = swb.refresh_from_set(two, img, 15.0)
    assert r.base.beta == 15.0
    assert np.abs(r.lambda_hat - two.packs[1].values).max() < 1e-5


@pytest.mark.parametrize("trial", range(4))
def test_full_basis_matches_dense(cuda_ok, trial):
    rng = np.random.default_rng(6 + trial)
    dims = tuple(int(x) for x in rng.integers(4, 9, size=2))
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * (rng.random(n) > 0.5) + rng.normal(0, 0.05, n), 0, 1)
    lap = O.build_laplacian(img, dims, 15.0)
    vals, vecs = np.linalg.eigh(lap.matrix.toarray())
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=15.0, eigen=swb.EigenBasis(np.asfortranarray(vecs), vals),
                            d_sqrt=lap.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    seeds = _seeds(n, 2, 2, seed=trial)
    if trial % 2:
        pri = rng.random((n, 2))
        pri /= pri.sum(axis=1, keepdims=True)
        prob = swb.LabelProblem(num_labels=2, seeds=seeds, priors=pri, gamma=0.5)
        u_ref = O.solve_fast(vecs, vals, lap.d_sqrt, lap.matrix, seeds.seed_indices, seeds.seed_labels, 2,
                             gamma=0.5, priors=pri, m_use=n)
    else:
        prob = swb.LabelProblem(num_labels=2, seeds=seeds, gamma=0.0)
        u_ref = O.solve_fast(vecs, vals, lap.d_sqrt, lap.matrix, seeds.seed_indices, seeds.seed_labels, 2, m_use=n)
    u = swb.solve_fast(pack, lap.matrix, prob, m_use=n, want_field=True).values
    assert np.abs(u - u_ref).max() < 1e-9


def test_no_seeds_constant_priors_identity(cuda_ok):
    z, img, pack, lap = _golden_pack()
    n = img.n_voxels
    pri = np.tile([0.3, 0.7], (n, 1))
    prob = swb.LabelProblem(num_labels=2, seeds=swb.SeedPartition(n, [], []), priors=pri, gamma=2.0)
    u = swb.solve_fast(pack, lap, prob, m_use=8, want_field=True).values
    assert np.abs(u - pri).max() < 1e-9


def test_row_sums_truncated_and_streaming_parity(cuda_ok):
    z, img, pack, lap = _golden_pack()
    prob = swb.LabelProblem(num_labels=2, seeds=_seeds(img.n_voxels, 2, 4, seed=7), gamma=0.0)
    u = swb.solve_fast(pack, lap, prob, m_use=24, want_field=True).values
    assert np.abs(u.sum(axis=1) - 1.0).max() < 1e-6
    u2 = swb.solve_fast(pack, lap, prob, m_use=24, streaming_block=7, want_field=True).values
    assert np.array_equal(u, u2)


def test_bitwise_determinism(cuda_ok):
    z, img, pack, lap = _golden_pack()
    prob = swb.LabelProblem(num_labels=2, seeds=_seeds(img.n_voxels, 2, 4, seed=9), gamma=0.0)
    u1 = swb.solve_fast(pack, lap, prob, m_use=32, want_field=True).values
    u2 = swb.solve_fast(pack, lap, prob, m_use=32, want_field=True).values
    assert np.array_equal(u1, u2)
    dp = swb.to_device(pack, image=img)
    a = swb.update_basis(dp, img, 21.0, method="first_order")
    b = swb.update_basis(dp, img, 21.0, method="first_order")
    assert np.array_equal(a.V.cpu().numpy(), b.V.cpu().numpy())
    assert np.array_equal(a.lambda_hat, b.lambda_hat)
    p1 = swb.precompute(img, 15.0, 12, eig_tol=1e-9, seed=3)
    p2 = swb.precompute(img, 15.0, 12, eig_tol=1e-9, seed=3)
    assert np.array_equal(p1.V.cpu().numpy(), p2.V.cpu().numpy())


def test_c4_geometry_update_determinism(cuda_ok):
    """A 64^3 c4-shaped volume, K = 96 (synthetic QR basis, as the bench):
    the first-order update is bitwise reproducible and keeps unit columns
    (the rotation's columns are normalised; the synthetic basis is not an
    eigenbasis, so off-diagonal orthogonality is not a property here)."""
    import torch

    from paper_1607_04174_b200 import workloads as W
    from paper_1607_04174_b200.device import DevicePack, LatticeSpec
    w = W.make_image("c4", dims=(64, 64, 64))
    p = w.params
    n, m = 64 ** 3, 96
    image = swb.Image(w.dims, w.intensities)
    lat = LatticeSpec.make(w.dims, p["connectivity"], p["weight_mode"])
    V = W.orthonormal_basis_device(n, m, seed=5)
    img_dev = torch.from_numpy(np.array(w.intensities)).cuda()
    g0 = swb.DeviceGraph.build(img_dev, lat, p["beta0"])
    lam = torch.from_numpy(W.synthetic_lambda("c4", m)).cuda()
    dp = DevicePack(V, m, lam, g0.d_sqrt_dev, g0.dnorm, w.dims, (), p["beta0"],
                    swb.PackProvenance(image_hash=image.content_hash()), lat, image_dev=img_dev, graph=g0)
    a = swb.update_basis(dp, image, p["beta1"], method="first_order")
    b = swb.update_basis(dp, image, p["beta1"], method="first_order")
    Va, Vb = a.V[:, :m], b.V[:, :m]
    assert torch.equal(Va, Vb)
    G = (Va.T @ Va).cpu().numpy()
    assert np.abs(np.diag(G) - 1.0).max() < 1e-12
    assert np.isfinite(G).all()
