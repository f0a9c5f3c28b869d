"""Pin the CPU oracle (oracle/rw_oracle.py) to golden vectors produced by the
unmodified reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import csr_from, load_golden
from oracle import rw_oracle as O


def _lap(z, prefix="lap"):
    mat = csr_from(z, prefix)
    return mat


def test_path3_known_answer():
    z = load_golden("path3")
    np.testing.assert_allclose(z["lam"], [0.0, 1.0, 2.0], atol=1e-9)
    lap = O.build_laplacian(z["intensities"], tuple(z["dims"]), 1.0)
    np.testing.assert_allclose(lap.matrix.toarray(), _lap(z).toarray(), rtol=0, atol=1e-15)
    u = O.solve_fast(z["V"], z["lam"], z["d_sqrt"], lap.matrix, z["seed_idx"], z["seed_lab"], 2, m_use=3)
    np.testing.assert_allclose(u, [[1, 0], [0.5, 0.5], [0, 1]], atol=1e-9)
    np.testing.assert_allclose(u, z["U"], atol=1e-12)


@pytest.mark.parametrize("name", ["phantom16", "blobs3d"])
def test_laplacian_matches_reference(name):
    z = load_golden(name)
    lap = O.build_laplacian(z["intensities"], tuple(z["dims"]), float(z["beta"]))
    ref = _lap(z)
    assert (lap.matrix != ref).nnz == 0 or np.abs((lap.matrix - ref)).max() == 0.0


@pytest.mark.parametrize("beta", [15, 33, 45])
def test_refresh_matches_reference(beta):
    z = load_golden("phantom16")
    lap = O.build_laplacian(z["intensities"], tuple(z["dims"]), float(beta))
    np.testing.assert_array_equal(lap.matrix.toarray(), csr_from(z, f"refresh_{beta}_lap").toarray())
    np.testing.assert_array_equal(lap.d_sqrt, z[f"refresh_{beta}_d_sqrt"])
    lam, order = O.refresh(z["V"], lap)
    np.testing.assert_array_equal(order, z[f"refresh_{beta}_order"])
    np.testing.assert_allclose(lam, z[f"refresh_{beta}_lam"], rtol=1e-12, atol=1e-15)


def test_refresh_3d_matches_reference():
    z = load_golden("blobs3d")
    lap = O.build_laplacian(z["intensities"], tuple(z["dims"]), 25.0)
    lam, order = O.refresh(z["V"], lap)
    np.testing.assert_array_equal(order, z["refresh_25_order"])
    np.testing.assert_allclose(lam, z["refresh_25_lam"], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("m_use", [24, 32, 64])
def test_solve_gamma0_matches_reference(m_use):
    z = load_golden("phantom16")
    lap = _lap(z)
    u = O.solve_fast(z["V"], z["lam"], z["d_sqrt"], lap, z["seeds0_idx"], z["seeds0_lab"], 2, m_use=m_use)
    np.testing.assert_allclose(u, z[f"solve0_m{m_use}_U"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(O.hard_labels(u), z[f"solve0_m{m_use}_labels"])


def test_solve_priors_matches_reference():
    z = load_golden("phantom16")
    lap = _lap(z)
    u = O.solve_fast(z["V"], z["lam"], z["d_sqrt"], lap, z["seeds1_idx"], z["seeds1_lab"], 2,
                     gamma=0.5, priors=z["priors"], m_use=40)
    np.testing.assert_allclose(u, z["solveg_m40_U"], rtol=0, atol=1e-12)
    n = z["d_sqrt"].size
    cpri = np.tile([0.3, 0.7], (n, 1))
    u = O.solve_fast(z["V"], z["lam"], z["d_sqrt"], lap, [], [], 2, gamma=2.0, priors=cpri, m_use=8)
    np.testing.assert_allclose(u, z["solve_noseed_U"], atol=1e-12)
    np.testing.assert_allclose(u, cpri, atol=1e-9)
    u = O.solve_fast(z["V"], z["lam"], z["d_sqrt"], lap, [], [], 2, gamma=1.0, priors=z["priors"], m_use=48)
    np.testing.assert_allclose(u, z["solve_noseed_rand_U"], atol=1e-12)


def test_solve_refreshed_pack_matches_reference():
    z = load_golden("phantom16")
    lap = O.build_laplacian(z["intensities"], tuple(z["dims"]), 45.0)
    lam, order = O.refresh(z["V"], lap)
    u = O.solve_fast(z["V"][:, order], lam, lap.d_sqrt, lap.matrix, z["seeds0_idx"], z["seeds0_lab"], 2, m_use=40)
    np.testing.assert_allclose(u, z["solve_refresh45_m40_U"], atol=1e-12)


def test_solve_3d_matches_reference():
    z = load_golden("blobs3d")
    lap = _lap(z)
    u = O.solve_fast(z["V"], z["lam"], z["d_sqrt"], lap, z["seeds_idx"], z["seeds_lab"], 2, m_use=20)
    np.testing.assert_allclose(u, z["solve0_m20_U"], atol=1e-12)
    u = O.solve_fast(z["V"], z["lam"], z["d_sqrt"], lap, [3, 50, 97], [0, 1, 2], 3, gamma=0.25,
                     priors=z["priors3"], m_use=30)
    np.testing.assert_allclose(u, z["solveg3_m30_U"], atol=1e-12)
    lap2 = O.build_laplacian(z["intensities"], tuple(z["dims"]), 25.0)
    lam, order = O.refresh(z["V"], lap2)
    u = O.solve_fast(z["V"][:, order], lam, lap2.d_sqrt, lap2.matrix, z["seeds_idx"], z["seeds_lab"], 2, m_use=30)
    np.testing.assert_allclose(u, z["solve_refresh_m30_U"], atol=1e-12)


@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("mode", ["abs", "sq"])
@pytest.mark.parametrize("beta", [60, 90])
def test_modes_laplacian_matches_reference_primitives(conn, mode, beta):
    z = load_golden("modes")
    lap = O.build_laplacian(z["intensities"], tuple(z["dims"]), float(beta), mode, conn)
    tag = f"c{conn}_{mode}_{beta}"
    np.testing.assert_array_equal(lap.matrix.toarray(), csr_from(z, tag).toarray())
    np.testing.assert_array_equal(lap.d_sqrt, z[tag + "_d_sqrt"])


def test_cut_laplacian_and_solve_match_reference():
    z = load_golden("modes")
    dims = tuple(z["dims"])
    cut = O.block_cut_mask(dims, 5, 3, size=4, connectivity=8)
    np.testing.assert_array_equal(cut, z["cut_mask"])
    lap = O.build_laplacian(z["intensities"], dims, 60.0, "sq", 8, cut_edges=cut)
    np.testing.assert_array_equal(lap.matrix.toarray(), csr_from(z, "cut_c8_sq_60").toarray())
    u = O.solve_fast(z["cut_V"], z["cut_lam"], lap.d_sqrt, lap.matrix, z["cut_seeds_idx"],
                     z["cut_seeds_lab"], 2, m_use=40)
    np.testing.assert_allclose(u, z["cut_U"], atol=1e-12)


@pytest.mark.parametrize("tag", ["default", "loose", "tight", "eps3e4"])
def test_select_m_seeds_matches_reference(tag):
    z = load_golden("phantom16")
    m, info = O.select_m(z["V"], z["d_sqrt"], z[f"sel_{tag}_idx"], z[f"sel_{tag}_lab"], 2,
                         epsilon=float(z[f"sel_{tag}_eps"]))
    assert m == int(z[f"sel_{tag}_m"])
    assert info["saturated"] == bool(z[f"sel_{tag}_sat"])
    np.testing.assert_array_equal([s["m"] for s in info["steps"]], z[f"sel_{tag}_steps_m"])
    np.testing.assert_allclose(np.array([s["f"] for s in info["steps"]]), z[f"sel_{tag}_steps_f"],
                               rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("tag,key,k", [("p_loose", "pri4", 4), ("p_tight", "pri4", 4), ("p_mid", "pri4", 4),
                                       ("ps_a", "psmooth", 2), ("ps_b", "psmooth", 2), ("ps_c", "psmooth", 2)])
def test_select_m_priors_matches_reference(tag, key, k):
    z = load_golden("phantom16")
    m, info = O.select_m(z["V"], z["d_sqrt"], [], [], k, priors=z[key], epsilon=float(z[f"sel_{tag}_eps"]))
    assert m == int(z[f"sel_{tag}_m"])
    assert info["saturated"] == bool(z[f"sel_{tag}_sat"])
    np.testing.assert_allclose(np.array([s["g"] for s in info["steps"]]), z[f"sel_{tag}_steps_g"],
                               rtol=1e-10, atol=1e-12)


def test_seed_fit_and_prior_residual_match_reference():
    z = load_golden("adaptive")
    for i in range(5):
        f = O.seed_fit(z[f"sf{i}_q"], z[f"sf{i}_u"], float(z[f"sf{i}_b"]))
        np.testing.assert_allclose(f, float(z[f"sf{i}_f"]), rtol=1e-10, atol=1e-14)
    g1, r1 = O.prior_residual(z["pr_q"][:, :6], z["pr_p"])
    g2, r2 = O.prior_residual(z["pr_q"], z["pr_p"], cached=r1, cached_m=6)
    np.testing.assert_allclose([g1, g2], [float(z["pr_g1"]), float(z["pr_g2"])], rtol=1e-12)
    np.testing.assert_allclose(r2, z["pr_r2"], atol=1e-14)


def test_seed_fit_closed_forms():
    # reference tests/test_adaptive.py:12-35
    assert O.seed_fit(np.eye(3), np.array([1.0, 0, 0]), 100.0) < 1e-12
    assert np.isclose(O.seed_fit(np.array([[0.6], [0.8]]), np.array([1.0, 0.0]), 100.0), 0.64, atol=1e-10)
    assert O.seed_fit(np.ones((4, 2)), np.array([1.0, 0, 1, 1]), 0.0) == pytest.approx(3.0)
    assert np.isclose(O.seed_fit(np.array([[1e-3], [0.0]]), np.array([1.0, 0.0]), 1.0), (1 - 1e-3) ** 2, rtol=1e-3)


def test_error_kinds_and_all_seeded():
    z = load_golden("errors")
    lap = _lap(z)
    kinds = dict(zip(z["kinds_keys"].tolist(), z["kinds_vals"].tolist()))
    for tag, m_use in (("m1", 1), ("m0", 0), ("m99", 99)):
        with pytest.raises(O.OracleError) as exc:
            O.solve_fast(z["V"], z["lam"], z["d_sqrt"], lap, z["seeds_idx"], z["seeds_lab"], 2, m_use=m_use)
        assert exc.value.kind == kinds[tag]
    u = O.solve_fast(z["V"], z["lam"], z["d_sqrt"], lap, np.arange(64), np.arange(64) % 2, 2, m_use=4)
    np.testing.assert_array_equal(u, z["allseed_U"])
    np.testing.assert_array_equal(O.hard_labels(z["ties_in"]), z["ties_out"])


@pytest.mark.parametrize("tag", ["2", "3"])
def test_similarity_priors_matches_reference(tag):
    z = load_golden("registration")
    vec = z["vec" + tag]
    np.testing.assert_array_equal(O.grid_vectors((3,) * len(z["dims" + tag])), vec)
    pri, sigma = O.similarity_priors(z["f" + tag], z["m" + tag], tuple(z["dims" + tag]), vec, patch_radius=1)
    np.testing.assert_allclose(pri, z["pri" + tag], rtol=1e-12, atol=1e-15)
    assert sigma > 0


def test_registration_solve_matches_reference():
    z = load_golden("registration")
    lap = csr_from(z, "lap3")
    u = O.solve_fast(z["V3"], z["lam3"], z["d3"], lap, [], [], 27, gamma=1.0, priors=z["pri3"], m_use=50)
    np.testing.assert_allclose(u, z["U3"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(u @ z["vec3"].astype(float), z["disp3"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("tag", ["2", "3"])
def test_aggregation_matches_reference(tag):
    z = load_golden("aggregation")
    dims = tuple(int(d) for d in z["dims" + tag])
    cid, ns = O.build_aggregation(z["pri" + tag], dims, int(z["radius" + tag]), float(z["tol" + tag]))
    np.testing.assert_array_equal(cid, z["cid" + tag])
    assert ns == int(z["nsup" + tag])
    np.testing.assert_array_equal(O.delta_weights(cid, dims), z["delta" + tag])
    for v, var in (("d", "delta"), ("n", "naive")):
        q, lam, dsq, lap = O.coarsen_basis(z["V" + tag], cid, ns, z["img" + tag], dims, float(z["beta" + tag]), var,
                                           int(z["muse" + tag]))
        np.testing.assert_allclose(q, z[f"q{v}{tag}"], atol=1e-12)
        np.testing.assert_allclose(lam, z[f"lb{v}{tag}"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(dsq, z[f"dsqbar{v}{tag}"], rtol=1e-14)
        np.testing.assert_allclose(lap.matrix.toarray(), csr_from(z, f"lapbar{v}{tag}").toarray(), atol=1e-15)
    pbar = O.aggregate_priors(z["pri" + tag], cid, ns)
    pbar /= pbar.sum(axis=1, keepdims=True)
    np.testing.assert_allclose(pbar, z["pbar" + tag], rtol=1e-14, atol=1e-16)
    q, lam, dsq, lap = O.coarsen_basis(z["V" + tag], cid, ns, z["img" + tag], dims, float(z["beta" + tag]), "delta",
                                       int(z["muse" + tag]))
    ubar = O.solve_fast(q, lam, dsq, lap.matrix, [], [], pbar.shape[1], gamma=1.0, priors=pbar, m_use=q.shape[1])
    np.testing.assert_allclose(ubar, z["ubar" + tag], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(ubar[cid], z["u" + tag], rtol=1e-9, atol=1e-12)
