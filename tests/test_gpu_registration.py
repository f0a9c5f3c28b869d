"""GPU parity for the registration data term: similarity
priors (registration.py:95-129), the 27-label priors solve and the expected
displacement readout (registration.py:132-136) vs the reference golden
vectors.  Tolerance: 1e-12 relative on priors (the same FP64 operations in a
different summation order), 1e-9 on solve outputs (north star)."""

import numpy as np
import pytest

import paper_1607_04174_b200 as swb
from conftest import csr_from, load_golden
from oracle import rw_oracle as O
from paper_1607_04174_b200 import registration as R

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag", ["2", "3"])
def test_similarity_priors(cuda_ok, tag):
    z = load_golden("registration")
    dims = tuple(int(d) for d in z["dims" + tag])
    grid = R.DisplacementGrid((3,) * len(dims))
    np.testing.assert_array_equal(grid.vectors(), z["vec" + tag])
    pri = R.similarity_priors(swb.Image(dims, z["f" + tag]), swb.Image(dims, z["m" + tag]), grid, patch_radius=1)
    np.testing.assert_allclose(pri.values, z["pri" + tag], rtol=1e-12, atol=1e-15)
    _, sigma = O.similarity_priors(z["f" + tag], z["m" + tag], dims, z["vec" + tag], patch_radius=1)
    assert abs(pri.sigma - sigma) <= 1e-13 * sigma


@pytest.mark.parametrize("radius,ext", [(0, (3, 3)), (2, (5, 3)), (3, (3, 5, 3)), (2, (5, 5, 5)), (7, (3, 3, 3)),
                                        (20, (3, 3))])
def test_similarity_priors_radius_and_grid(cuda_ok, radius, ext):
    rng = np.random.default_rng(7 + radius)
    dims = (45, 37) if len(ext) == 2 else ((7, 6, 5) if radius == 7 else (35, 19, 9))
    f = rng.random(int(np.prod(dims)))
    m = rng.random(int(np.prod(dims)))
    grid = R.DisplacementGrid(ext, step=2 if radius == 2 else 1)
    pri = R.similarity_priors(swb.Image(dims, f), swb.Image(dims, m), grid, patch_radius=radius)
    want, sigma = O.similarity_priors(f, m, dims, grid.vectors(), patch_radius=radius)
    np.testing.assert_allclose(pri.values, want, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(pri.values.sum(axis=1), 1.0, atol=1e-14)


def test_identical_images_are_sharp(cuda_ok):
    rng = np.random.default_rng(3)
    dims = (10, 9)
    f = rng.random(90)
    grid = R.DisplacementGrid((3, 3))
    pri = R.similarity_priors(swb.Image(dims, f), swb.Image(dims, f), grid, patch_radius=1)
    assert (pri.values.argmax(axis=1) == grid.zero_label()).all()


def test_registration_solve_and_displacement(cuda_ok):
    z = load_golden("registration")
    dims = tuple(int(d) for d in z["dims3"])
    img = swb.Image(dims, z["f3"])
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=50.0,
                            eigen=swb.EigenBasis(np.asfortranarray(z["V3"]), z["lam3"]), d_sqrt=z["d3"],
                            provenance=swb.PackProvenance(image_hash=img.content_hash()))
    grid = R.DisplacementGrid((3, 3, 3))
    pri = R.similarity_priors(img, swb.Image(dims, z["m3"]), grid, patch_radius=1)
    n = img.n_voxels
    prob = swb.LabelProblem(num_labels=27, seeds=swb.SeedPartition(n, [], []), priors=pri.values, gamma=1.0)
    lap = csr_from(z, "lap3")
    u = swb.solve_fast(pack, lap, prob, m_use=50, want_field=True)
    np.testing.assert_allclose(u.values, z["U3"], rtol=1e-9, atol=1e-12)
    disp = R.expected_displacement(u, grid)
    np.testing.assert_allclose(disp, z["disp3"], rtol=1e-9, atol=1e-12)


def test_c5_workflow_matches_oracle(cuda_ok):
    """BASELINE config 5 at reduced size (the bench's c5 step): beta 50 -> 70
    first-order update of a QR basis, similarity priors on the c5 pair,
    125-label gamma = 1 solve, argmax + expected displacement."""
    from paper_1607_04174_b200 import workloads as W
    w = W.make_image("c5", dims=(14, 12, 10))
    p = w.params
    dims, n, m = w.dims, int(np.prod(w.dims)), 160
    lap0 = O.build_laplacian(w.intensities, dims, p["beta0"], p["weight_mode"], p["connectivity"])
    lap1 = O.build_laplacian(w.intensities, dims, p["beta1"], p["weight_mode"], p["connectivity"])
    rng = np.random.default_rng(55)
    V = np.linalg.qr(rng.standard_normal((n, m)))[0]
    lam = np.sort(rng.uniform(1e-4, 1e-1, m))
    image = swb.Image(dims, w.intensities)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=p["beta0"], eigen=swb.EigenBasis(np.asfortranarray(V), lam),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    dp = swb.to_device(pack, image=image, connectivity=p["connectivity"], weight_mode=p["weight_mode"])
    up = swb.update_basis(dp, image, p["beta1"], method="first_order")
    grid = R.DisplacementGrid(p["grid"])
    field, disp, rep = R.register(image, swb.Image(dims, p["moving"]), up, grid=grid, gamma=p["gamma"],
                                  patch_radius=p["patch_radius"])
    Vo, lamo, _, _, _ = O.first_order_update(V, lam, lap0, lap1)
    pri, _ = O.similarity_priors(w.intensities, p["moving"], dims, grid.vectors(), p["patch_radius"])
    u = O.solve_fast(Vo, lamo, lap1.d_sqrt, lap1.matrix, [], [], 125, gamma=p["gamma"], priors=pri)
    np.testing.assert_allclose(field.values, u, rtol=1e-9, atol=1e-12)
    gap = O.top2_gap(u)
    lab = swb.hard_labels(field).labels
    assert not ((lab != O.hard_labels(u)) & (gap >= 1e-9)).any()
    np.testing.assert_allclose(disp, u @ grid.vectors(), rtol=1e-9, atol=1e-12)
