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


@pytest.mark.parametrize("radius,ext", [(0, (3, 3)), (2, (5, 3)), (3, (3, 5, 3))])
def test_similarity_priors_radius_and_grid(cuda_ok, radius, ext):
    rng = np.random.default_rng(7 + radius)
    dims = (9, 8) if len(ext) == 2 else (7, 6, 5)
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
