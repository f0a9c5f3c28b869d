"""GPU parity: the sm_100a path through the C ABI vs the oracle / golden vectors.

Tolerances (north star): FP64 results within 1e-9 relative (absolute floor
1e-12 for probabilities, 1e-13 for near-zero eigenvalues); label maps
bit-exact except where the top-two probabilities differ by < 1e-9.
"""

import numpy as np
import pytest

import paper_1607_04174_b200 as swb
from conftest import csr_from, load_golden
from oracle import rw_oracle as O

pytestmark = pytest.mark.gpu

RTOL = 1e-9


def host_pack(z, beta=None, dims=None, image=None):
    dims = tuple(int(d) for d in (dims if dims is not None else z["dims"]))
    if image is not None:
        img = image
    elif "intensities" in z.files:
        img = swb.Image(dims, z["intensities"])
    else:
        img = swb.Image(dims, np.zeros(int(np.prod(dims))))
    return swb.SpectralPack(dims=dims, spacing=(), beta=float(z["beta"] if beta is None else beta),
                            eigen=swb.EigenBasis(np.asfortranarray(z["V"]), z["lam"]), d_sqrt=z["d_sqrt"],
                            provenance=swb.PackProvenance(image_hash=img.content_hash())), img


def assert_labels_match(lab_gpu, u_ref, tol=1e-9):
    ref_lab = O.hard_labels(u_ref)
    gap = O.top2_gap(u_ref)
    bad = (lab_gpu != ref_lab) & (gap >= tol)
    assert not bad.any(), f"{bad.sum()} label mismatches outside near-ties"


def assert_lam(got, want):
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=1e-13)


# ---------------------------------------------------------------------------
# graph / Laplacian
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["phantom16", "blobs3d"])
def test_graph_matches_reference_laplacian(cuda_ok, name):
    z = load_golden(name)
    import torch
    lat = swb.LatticeSpec.make(tuple(z["dims"]))
    g = swb.DeviceGraph.build(torch.from_numpy(z["intensities"]).cuda(), lat, float(z["beta"]))
    ref = csr_from(z, "lap").toarray()
    np.testing.assert_allclose(g.matrix.toarray(), ref, rtol=1e-14, atol=1e-16)
    np.testing.assert_allclose(g.d_sqrt, O.build_laplacian(z["intensities"], tuple(z["dims"]), float(z["beta"])).d_sqrt,
                               rtol=1e-15)


@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("mode", ["abs", "sq"])
def test_graph_modes_match_reference_primitives(cuda_ok, conn, mode):
    import torch
    z = load_golden("modes")
    dims = tuple(z["dims"])
    lat = swb.LatticeSpec.make(dims, conn, mode)
    for beta in (60, 90):
        g = swb.DeviceGraph.build(torch.from_numpy(z["intensities"]).cuda(), lat, float(beta))
        np.testing.assert_allclose(g.matrix.toarray(), csr_from(z, f"c{conn}_{mode}_{beta}").toarray(),
                                   rtol=1e-14, atol=1e-16)


def test_graph_cut_matches_reference(cuda_ok):
    import torch
    z = load_golden("modes")
    dims = tuple(z["dims"])
    lat = swb.LatticeSpec.make(dims, 8, "sq")
    vm = lat.edge_mask_to_voxel_mask(z["cut_mask"])
    g = swb.DeviceGraph.build(torch.from_numpy(z["intensities"]).cuda(), lat, 60.0, torch.from_numpy(vm).cuda())
    np.testing.assert_allclose(g.matrix.toarray(), csr_from(z, "cut_c8_sq_60").toarray(), rtol=1e-14, atol=1e-16)


# ---------------------------------------------------------------------------
# refresh (beta update, eigenvalue half)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("beta", [15, 33, 45])
def test_refresh_matches_reference(cuda_ok, beta):
    z = load_golden("phantom16")
    pack, img = host_pack(z)
    r = swb.refresh(pack, img, float(beta))
    assert_lam(r.lambda_hat, z[f"refresh_{beta}_lam"])
    np.testing.assert_array_equal(r.order, z[f"refresh_{beta}_order"])
    np.testing.assert_allclose(r.d_sqrt, z[f"refresh_{beta}_d_sqrt"], rtol=1e-15)


def test_refresh_3d_matches_reference(cuda_ok):
    z = load_golden("blobs3d")
    pack, img = host_pack(z)
    r = swb.refresh(pack, img, 25.0)
    assert_lam(r.lambda_hat, z["refresh_25_lam"])
    np.testing.assert_array_equal(r.order, z["refresh_25_order"])


def test_refresh_image_mismatch(cuda_ok):
    z = load_golden("phantom16")
    pack, _ = host_pack(z)
    other = swb.Image((16, 16), np.linspace(0, 1, 256))
    with pytest.raises(swb.ImageMismatch):
        swb.refresh(pack, other, 20.0)


# ---------------------------------------------------------------------------
# solve_fast
# ---------------------------------------------------------------------------

def _prob(idx, lab, k=2, **kw):
    n = kw.pop("n")
    return swb.LabelProblem(num_labels=k, seeds=swb.SeedPartition(n, idx, lab), **kw)


def test_path3_known_answer(cuda_ok):
    z = load_golden("path3")
    pack, img = host_pack(z)
    lap = swb.DeviceGraph.build(__import__("torch").from_numpy(z["intensities"]).cuda(),
                                swb.LatticeSpec.make((3, 1)), 1.0)
    f = swb.solve_fast(pack, lap, _prob([0, 2], [0, 1], n=3), m_use=3, want_field=True)
    np.testing.assert_allclose(f.values, [[1, 0], [0.5, 0.5], [0, 1]], atol=1e-9)
    np.testing.assert_allclose(f.values, z["U"], atol=1e-12)
    assert swb.hard_labels(f).labels.tolist() == z["labels"].tolist()


@pytest.mark.parametrize("m_use", [24, 32, 64])
@pytest.mark.parametrize("lap_kind", ["device", "host"])
def test_solve_gamma0_matches_reference(cuda_ok, m_use, lap_kind):
    z = load_golden("phantom16")
    pack, img = host_pack(z)
    n = z["d_sqrt"].size
    dp = swb.to_device(pack)
    if lap_kind == "device":
        import torch
        lap = swb.DeviceGraph.build(torch.from_numpy(z["intensities"]).cuda(), dp.lattice, 15.0)
    else:
        lap = O.Lap(csr_from(z, "lap"), z["d_sqrt"], z["d_sqrt"] ** 2)
    f = swb.solve_fast(dp, lap, _prob(z["seeds0_idx"], z["seeds0_lab"], n=n), m_use=m_use, want_field=True)
    np.testing.assert_allclose(f.values, z[f"solve0_m{m_use}_U"], rtol=0, atol=1e-10)
    np.testing.assert_array_equal(swb.hard_labels(f).labels, z[f"solve0_m{m_use}_labels"])


def test_solve_priors_matches_reference(cuda_ok):
    z = load_golden("phantom16")
    pack, img = host_pack(z)
    n = z["d_sqrt"].size
    lap = O.Lap(csr_from(z, "lap"), z["d_sqrt"], z["d_sqrt"] ** 2)
    f = swb.solve_fast(pack, lap, _prob(z["seeds1_idx"], z["seeds1_lab"], n=n, priors=z["priors"], gamma=0.5),
                       m_use=40, want_field=True)
    np.testing.assert_allclose(f.values, z["solveg_m40_U"], atol=1e-10)
    cpri = np.tile([0.3, 0.7], (n, 1))
    f = swb.solve_fast(pack, lap, _prob([], [], n=n, priors=cpri, gamma=2.0), m_use=8, want_field=True)
    np.testing.assert_allclose(f.values, z["solve_noseed_U"], atol=1e-10)
    np.testing.assert_allclose(f.values, cpri, atol=1e-9)
    f = swb.solve_fast(pack, lap, _prob([], [], n=n, priors=z["priors"], gamma=1.0), m_use=48, want_field=True)
    np.testing.assert_allclose(f.values, z["solve_noseed_rand_U"], atol=1e-10)


def test_solve_refreshed_pack_matches_reference(cuda_ok):
    z = load_golden("phantom16")
    pack, img = host_pack(z)
    n = z["d_sqrt"].size
    r = swb.refresh(pack, img, 45.0)
    f = swb.solve_fast(r, r.laplacian, _prob(z["seeds0_idx"], z["seeds0_lab"], n=n), m_use=40, want_field=True)
    np.testing.assert_allclose(f.values, z["solve_refresh45_m40_U"], atol=1e-10)


def test_solve_3d_matches_reference(cuda_ok):
    z = load_golden("blobs3d")
    pack, img = host_pack(z)
    n = z["d_sqrt"].size
    lap = O.Lap(csr_from(z, "lap"), z["d_sqrt"], z["d_sqrt"] ** 2)
    f = swb.solve_fast(pack, lap, _prob(z["seeds_idx"], z["seeds_lab"], n=n), m_use=20, want_field=True)
    np.testing.assert_allclose(f.values, z["solve0_m20_U"], atol=1e-10)
    f = swb.solve_fast(pack, lap, _prob([3, 50, 97], [0, 1, 2], k=3, n=n, priors=z["priors3"], gamma=0.25),
                       m_use=30, want_field=True)
    np.testing.assert_allclose(f.values, z["solveg3_m30_U"], atol=1e-10)
    r = swb.refresh(pack, img, 25.0)
    f = swb.solve_fast(r, r.laplacian, _prob(z["seeds_idx"], z["seeds_lab"], n=n), m_use=30, want_field=True)
    np.testing.assert_allclose(f.values, z["solve_refresh_m30_U"], atol=1e-10)


def test_solve_cut_laplacian_matches_reference(cuda_ok):
    z = load_golden("modes")
    dims = tuple(z["dims"])
    n = int(np.prod(dims))
    lap = O.build_laplacian(z["intensities"], dims, 60.0, "sq", 8, cut_edges=z["cut_mask"])
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=60.0, eigen=swb.EigenBasis(z["cut_V"], z["cut_lam"]),
                            d_sqrt=lap.d_sqrt, provenance=swb.PackProvenance(b""))
    dp = swb.to_device(pack, connectivity=8, weight_mode="sq")
    f = swb.solve_fast(dp, lap, _prob(z["cut_seeds_idx"], z["cut_seeds_lab"], n=n), m_use=40, want_field=True)
    np.testing.assert_allclose(f.values, z["cut_U"], atol=1e-10)


def test_solve_errors_and_all_seeded(cuda_ok):
    z = load_golden("errors")
    pack, _ = host_pack(z, beta=15.0, dims=(8, 8))
    lap = O.Lap(csr_from(z, "lap"), z["d_sqrt"], z["d_sqrt"] ** 2)
    prob = _prob(z["seeds_idx"], z["seeds_lab"], n=64)
    with pytest.raises(swb.InsufficientBasis):
        swb.solve_fast(pack, lap, prob, m_use=1)
    with pytest.raises(swb.InvalidParam):
        swb.solve_fast(pack, lap, prob, m_use=0)
    with pytest.raises(swb.InvalidParam):
        swb.solve_fast(pack, lap, prob, m_use=99)
    alls = _prob(np.arange(64), np.arange(64) % 2, n=64)
    f = swb.solve_fast(pack, lap, alls, m_use=4, want_field=True)
    np.testing.assert_array_equal(f.values, z["allseed_U"])


def test_hard_labels_ties(cuda_ok):
    f = swb.ProbabilityField((2, 1), [[0.2, 0.8], [0.5, 0.5]])
    assert swb.hard_labels(f).labels.tolist() == [1, 0]
    f = swb.ProbabilityField((3, 1), [[1, 0], [0, 1], [0.4, 0.6]])
    assert swb.hard_labels(f).labels.tolist() == [0, 1, 1]


# ---------------------------------------------------------------------------
# DMMA GEMMs and the dense LU against numpy / LAPACK
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("rows,m1,m2,sym", [(1000, 50, 50, 1), (4099, 400, 400, 1), (777, 150, 150, 0),
                                            (5000, 300, 125, 0), (333, 7, 3, 0), (12345, 200, 4, 0)])
def test_gemm_tn(cuda_ok, rows, m1, m2, sym):
    import torch
    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200.device import ptr, round_up, stream_handle
    rng = np.random.default_rng(rows)
    ld1, ld2 = round_up(m1, 8), round_up(m2, 8)
    X = rng.standard_normal((rows, ld1))
    Y = X.copy() if sym else rng.standard_normal((rows, ld2))
    if sym:
        ld2 = ld1
    xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    out = torch.zeros((m1, round_up(m2, 2)), dtype=torch.float64, device="cuda")
    ws = torch.empty(_lib.size("swb_gemm_tn_workspace_bytes", rows, m1, m2), dtype=torch.uint8, device="cuda")
    _lib.call("swb_gemm_tn", ptr(xd), ld1, ptr(yd), ld2, rows, m1, m2, sym, ptr(out), out.shape[1], ptr(ws),
              ws.numel(), stream_handle())
    want = X[:, :m1].T @ Y[:, :m2]
    got = out.cpu().numpy()[:, :m2]
    np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-11 * np.abs(want).max())


@pytest.mark.parametrize("rows,k,m2", [(1000, 50, 50), (4099, 400, 400), (777, 150, 150), (5000, 300, 125),
                                       (333, 7, 3), (100, 32, 64)])
def test_gemm_nn(cuda_ok, rows, k, m2):
    import torch
    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200.device import ptr, round_up, stream_handle
    rng = np.random.default_rng(k)
    lda, ldb = round_up(k, 8), round_up(m2, 2)
    A = rng.standard_normal((rows, lda))
    B = rng.standard_normal((k, ldb))
    ad, bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    out = torch.zeros((rows, ldb), dtype=torch.float64, device="cuda")
    _lib.call("swb_gemm_nn", ptr(ad), lda, ptr(bd), ldb, rows, k, m2, ptr(out), ldb, 0, stream_handle())
    want = A[:, :k] @ B[:, :m2]
    np.testing.assert_allclose(out.cpu().numpy()[:, :m2], want, rtol=1e-11, atol=1e-12 * np.abs(want).max())


@pytest.mark.parametrize("rows,k,m2", [(500, 125, 3), (300, 7, 3), (257, 33, 64)])
def test_gemm_nn_odd_k_ignores_padding_columns(cuda_ok, rows, k, m2):
    """An odd reduction length ends in half a 16-byte chunk: the column past
    K - 1 (here NaN, as uninitialised padding of a probability field can be)
    must not reach the product (expected_displacement: 125 labels, ld 126)."""
    import torch
    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200.device import ptr, round_up, stream_handle
    rng = np.random.default_rng(k + rows)
    lda, ldb = round_up(k, 2), round_up(m2, 2)
    A = rng.standard_normal((rows, lda))
    A[:, k:] = np.nan
    B = rng.standard_normal((k, ldb))
    ad, bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    out = torch.zeros((rows, ldb), dtype=torch.float64, device="cuda")
    _lib.call("swb_gemm_nn", ptr(ad), lda, ptr(bd), ldb, rows, k, m2, ptr(out), ldb, 0, stream_handle())
    want = A[:, :k] @ B[:, :m2]
    np.testing.assert_allclose(out.cpu().numpy()[:, :m2], want, rtol=1e-11, atol=1e-12 * np.abs(want).max())


@pytest.mark.parametrize("n", [1, 5, 33, 64, 201, 801, 1001])
def test_lu_solve_and_rcond_match_lapack(cuda_ok, n):
    import scipy.linalg as sla
    import torch
    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200.device import ptr, round_up, stream_handle
    rng = np.random.default_rng(n)
    A = np.eye(n) * 3 + rng.standard_normal((n, n)) / np.sqrt(n)
    B = rng.standard_normal((n, 4))
    lda = round_up(n, 8)
    Ad = torch.zeros((n, lda), dtype=torch.float64, device="cuda")
    Ad[:, :n] = torch.from_numpy(A)
    Bd = torch.from_numpy(B.copy()).cuda()
    piv = torch.empty(n, dtype=torch.int32, device="cuda")
    anorm = torch.empty(1, dtype=torch.float64, device="cuda")
    rc = torch.empty(1, dtype=torch.float64, device="cuda")
    ws = torch.empty(_lib.size("swb_lu_workspace_bytes", n), dtype=torch.uint8, device="cuda")
    st = stream_handle()
    _lib.call("swb_lu_factor", ptr(Ad), n, lda, ptr(piv), ptr(anorm), ptr(ws), ws.numel(), st)
    rws = torch.empty(_lib.size("swb_lu_solve_workspace_bytes", n, 4), dtype=torch.uint8, device="cuda")
    _lib.call("swb_lu_solve", ptr(Ad), n, lda, ptr(piv), ptr(Bd), 4, 4, ptr(rws), rws.numel(), st)
    _lib.call("swb_lu_rcond", ptr(Ad), n, lda, ptr(piv), ptr(anorm), ptr(rc), ptr(ws), ws.numel(), st)
    x = np.linalg.solve(A, B)
    np.testing.assert_allclose(Bd.cpu().numpy(), x, rtol=1e-11, atol=1e-12)
    lu, p = sla.lu_factor(A)
    want = sla.lapack.dgecon(lu, np.linalg.norm(A, 1), norm="1")[0]
    assert abs(anorm.item() - np.linalg.norm(A, 1)) <= 1e-13 * np.linalg.norm(A, 1)
    np.testing.assert_allclose(rc.item(), want, rtol=1e-6)


@pytest.mark.parametrize("n,kind,nrhs", [(1, "gen", 2), (5, "gen", 4), (33, "singular", 2), (41, "gen", 2),
                                         (41, "pivot", 4), (64, "pivot", 27), (64, "gen", 192), (37, "zero_col", 3),
                                         (65, "pivot", 3), (151, "gen", 3), (160, "pivot", 4), (129, "pivot", 12)])
def test_small_dense_column_owner_kernel(cuda_ok, n, kind, nrhs):
    """swb_small_dense_solve without the condition estimate (the
    column-owner kernel, one barrier per column; n <= 160): factors and pivots
    bit-equal to the row-parallel kernel's (same operations per element),
    both equal to LAPACK's; solutions vs numpy."""
    import scipy.linalg as sla
    import torch
    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200.device import ptr, round_up, stream_handle
    rng = np.random.default_rng(n + len(kind) + nrhs)
    A = np.eye(n) * 3 + rng.standard_normal((n, n)) / np.sqrt(n)
    if kind == "pivot":
        A = rng.standard_normal((n, n))
    if kind == "singular":
        A[:, 3] = A[:, 5]
    if kind == "zero_col":
        A[:, 7] = 0.0
    B = rng.standard_normal((n, nrhs))
    lda = round_up(n, 8)

    def run(with_rcond):
        Ad = torch.zeros((n, lda), dtype=torch.float64, device="cuda")
        Ad[:, :n] = torch.from_numpy(A)
        Bd = torch.from_numpy(B.copy()).cuda()
        piv = torch.empty(n, dtype=torch.int32, device="cuda")
        anorm = torch.empty(1, dtype=torch.float64, device="cuda")
        rc = torch.empty(1, dtype=torch.float64, device="cuda")
        _lib.call("swb_small_dense_solve", ptr(Ad), n, lda, ptr(piv), ptr(Bd), nrhs, nrhs, ptr(anorm),
                  ptr(rc) if with_rcond else None, stream_handle())
        torch.cuda.synchronize()
        return Ad[:, :n].cpu().numpy(), piv.cpu().numpy(), Bd.cpu().numpy(), anorm.item()

    lu_c, piv_c, x_c, an_c = run(False)
    lu_r, piv_r, x_r, an_r = run(True)
    np.testing.assert_array_equal(piv_c, piv_r)
    np.testing.assert_array_equal(lu_c, lu_r)
    assert an_c == an_r
    if kind in ("singular", "zero_col"):
        return
    lu, p = sla.lu_factor(A)
    np.testing.assert_array_equal(piv_c, p)
    np.testing.assert_allclose(lu_c, lu, rtol=0, atol=1e-12 * np.abs(lu).max())
    x = np.linalg.solve(A, B)
    np.testing.assert_allclose(x_c, x, rtol=1e-11, atol=1e-11 * np.abs(x).max())
    np.testing.assert_allclose(x_c, x_r, rtol=1e-12, atol=1e-12 * np.abs(x).max())


@pytest.mark.parametrize("n,kind", [(1, "gen"), (5, "gen"), (41, "gen"), (41, "pivot"), (128, "gen"),
                                    (160, "gen"), (97, "ill"), (33, "singular")])
def test_small_dense_solve_matches_lapack(cuda_ok, n, kind):
    """swb_small_dense_solve (n <= 160 in one launch) vs LAPACK: the solve,
    the pivots (dgetrf's), ||A||_1 and dgecon's rcond; exactly singular ->
    rcond 0."""
    import scipy.linalg as sla
    import torch
    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200.device import ptr, round_up, stream_handle
    rng = np.random.default_rng(n + len(kind))
    A = np.eye(n) * 3 + rng.standard_normal((n, n)) / np.sqrt(n)
    if kind == "pivot":
        A = rng.standard_normal((n, n))               # partial pivoting does real work
    if kind == "ill":
        U, _, Vt = np.linalg.svd(rng.standard_normal((n, n)))
        A = U @ np.diag(np.logspace(0, -11, n)) @ Vt
    if kind == "singular":
        A[:, 3] = A[:, 5]
    B = rng.standard_normal((n, 4))
    lda = round_up(n, 8)
    Ad = torch.zeros((n, lda), dtype=torch.float64, device="cuda")
    Ad[:, :n] = torch.from_numpy(A)
    Bd = torch.from_numpy(B.copy()).cuda()
    piv = torch.empty(n, dtype=torch.int32, device="cuda")
    anorm = torch.empty(1, dtype=torch.float64, device="cuda")
    rc = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.call("swb_small_dense_solve", ptr(Ad), n, lda, ptr(piv), ptr(Bd), 4, 4, ptr(anorm), ptr(rc), stream_handle())
    lu, p = sla.lu_factor(A)
    assert abs(anorm.item() - np.linalg.norm(A, 1)) <= 1e-13 * np.linalg.norm(A, 1)
    if kind == "singular":
        assert rc.item() < 1e-14
        return
    np.testing.assert_array_equal(piv.cpu().numpy(), p)
    want = sla.lapack.dgecon(lu, np.linalg.norm(A, 1), norm="1")[0]
    if kind == "ill":
        # cond ~1e11: factors / solutions agree only to ~cond * eps (LAPACK's
        # recursive getrf orders the updates differently); the estimate, and
        # the SingularSmallSystem decision on it, agree
        np.testing.assert_allclose(rc.item(), want, rtol=1e-3)
        r = A @ Bd.cpu().numpy() - B
        assert np.abs(r).max() <= 1e-6 * np.abs(B).max()
        return
    np.testing.assert_allclose(Ad[:, :n].cpu().numpy(), lu, rtol=0, atol=1e-12 * np.abs(lu).max())
    x = np.linalg.solve(A, B)
    np.testing.assert_allclose(Bd.cpu().numpy(), x, rtol=1e-11, atol=1e-11 * np.abs(x).max())
    np.testing.assert_allclose(rc.item(), want, rtol=1e-6)


def test_singular_small_system_raises(cuda_ok):
    # duplicated eigenvector columns make the seed system singular
    z = load_golden("errors")
    V = np.asfortranarray(z["V"]).copy()
    V[:, 2] = V[:, 1]
    V[:, 3] = V[:, 1]
    pack = swb.SpectralPack(dims=(8, 8), spacing=(), beta=15.0, eigen=swb.EigenBasis(V, np.zeros(16) + 1e-3),
                            d_sqrt=z["d_sqrt"], provenance=swb.PackProvenance(b""))
    lap = O.Lap(csr_from(z, "lap"), z["d_sqrt"], z["d_sqrt"] ** 2)
    prob = _prob(np.arange(0, 64, 2), np.arange(32) % 2, n=64)
    try:
        O.solve_fast(V, np.zeros(16) + 1e-3, z["d_sqrt"], lap.matrix, np.arange(0, 64, 2), np.arange(32) % 2, 2,
                     m_use=4)
        expect = None
    except O.OracleError as exc:
        expect = exc.kind
    if expect == "SingularSmallSystem":
        with pytest.raises(swb.SingularSmallSystem):
            swb.solve_fast(pack, lap, prob, m_use=4)
    else:
        swb.solve_fast(pack, lap, prob, m_use=4)


# ---------------------------------------------------------------------------
# first-order update vs the restated oracle
# ---------------------------------------------------------------------------

def _match_columns(Vg, Vo, lam_old, order, label=""):
    """Columns up to sign at 1e-9 relative (normwise); groups of near-equal
    stored λ compared by the principal angle of their spans (vprime_check)."""
    from vprime_check import compare_vprime
    compare_vprime(Vg, Vo, lam_old, order, label=label)


@pytest.mark.parametrize("dims,conn,mode,m,b0,b1", [((24, 20), 4, "abs", 30, 15.0, 22.0),
                                                    ((32, 32), 4, "sq", 40, 90.0, 120.0),
                                                    ((20, 18), 8, "sq", 36, 60.0, 80.0),
                                                    ((10, 9, 8), 6, "abs", 40, 10.0, 14.0)])
def test_first_order_update_matches_oracle(cuda_ok, dims, conn, mode, m, b0, b1):
    import scipy.sparse.linalg as spla
    rng = np.random.default_rng(sum(dims))
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * np.sign(rng.standard_normal(n)) * (rng.random(n) < 0.1) +
                  rng.normal(0, 0.05, n), 0, 1)
    lap0 = O.build_laplacian(img, dims, b0, mode, conn)
    vals, vecs = np.linalg.eigh(lap0.matrix.toarray())
    V, lam = vecs[:, :m], vals[:m]
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=b0, eigen=swb.EigenBasis(np.asfortranarray(V), lam),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    dp = swb.to_device(pack, image=image, connectivity=conn, weight_mode=mode)
    up = swb.update_basis(dp, image, b1, method="first_order", keep_P=True)
    lap1 = O.build_laplacian(img, dims, b1, mode, conn)
    Vo, lamo, order, P, Cf = O.first_order_update(V, lam, lap0, lap1)
    np.testing.assert_allclose(up.P.cpu().numpy()[:, :m], P, rtol=0, atol=1e-12)
    assert_lam(up.lambda_hat, lamo)
    np.testing.assert_array_equal(up.order, order)
    Vg = up.V.cpu().numpy()[:, :m]
    _match_columns(Vg, Vo, lam, order, label=f"eigh basis {dims} conn {conn} {mode} m {m} beta {b0}->{b1}")
    # and the updated pack solves like the oracle on the updated basis
    seeds = np.sort(rng.choice(n, 12, replace=False))
    labs = np.arange(12) % 2
    f = swb.solve_fast(up, up.laplacian, _prob(seeds, labs, n=n), want_field=True)
    u_ref = O.solve_fast(Vo, lamo, lap1.d_sqrt, lap1.matrix, seeds, labs, 2)
    np.testing.assert_allclose(f.values, u_ref, atol=1e-9)
    assert_labels_match(swb.hard_labels(f).labels, u_ref)


@pytest.mark.parametrize("dims,m", [((32, 24), 512), ((30, 30), 520)])
def test_first_order_update_basis_size_limits(cuda_ok, dims, m):
    """K = 512 (the largest K of the INT8 digit-product rotation: every group
    sum still an exact int32) and K = 520 (beyond it: the rotation runs on the
    DMMA GEMM) both match the oracle.  With 512 of 768 eigenpairs of a 2-D
    grid the upper spectrum is clustered (gaps ~1e-5), so C = P / gap
    amplifies the 1e-12 agreement of P; the rotation itself is checked
    against V C with C from the GPU's own P (the oracle's coefficient rule)."""
    rng = np.random.default_rng(m)
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * (rng.random(n) < 0.2) + rng.normal(0, 0.05, n), 0, 1)
    lap0 = O.build_laplacian(img, dims, 30.0, "abs", 4)
    vals, vecs = np.linalg.eigh(lap0.matrix.toarray())
    V, lam = vecs[:, :m], vals[:m]
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=30.0, eigen=swb.EigenBasis(np.asfortranarray(V), lam),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    dp = swb.to_device(pack, image=image, connectivity=4, weight_mode="abs")
    up = swb.update_basis(dp, image, 36.0, method="first_order", keep_P=True)
    lap1 = O.build_laplacian(img, dims, 36.0, "abs", 4)
    Vo, lamo, order, P, _ = O.first_order_update(V, lam, lap0, lap1)
    np.testing.assert_allclose(up.P.cpu().numpy()[:, :m], P, rtol=0, atol=1e-12)
    assert_lam(up.lambda_hat, lamo)
    np.testing.assert_array_equal(up.order, order)
    Pg = up.P.cpu().numpy()[:, :m]
    lam_hat_unsorted = np.empty(m)
    lam_hat_unsorted[up.order] = up.lambda_hat
    Cg = O.update_coefficients(Pg, lam, lam_hat_unsorted, 0.5)[0]
    np.testing.assert_allclose(up.V.cpu().numpy()[:, :m], V @ Cg, rtol=0, atol=1e-12)


def test_cut_update_matches_oracle(cuda_ok):
    dims = (28, 24)
    rng = np.random.default_rng(5)
    n = int(np.prod(dims))
    img = np.clip(0.5 + rng.normal(0, 0.05, n), 0, 1)
    lap0 = O.build_laplacian(img, dims, 60.0, "sq", 8)
    vals, vecs = np.linalg.eigh(lap0.matrix.toarray())
    m = 32
    V, lam = vecs[:, :m], vals[:m]
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=60.0, eigen=swb.EigenBasis(np.asfortranarray(V), lam),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    cut = O.block_cut_mask(dims, 9, 7, size=8, connectivity=8)
    dp = swb.to_device(pack, image=image, connectivity=8, weight_mode="sq")
    up = swb.update_basis(dp, image, 60.0, cut_edges=cut, method="first_order", keep_P=True)
    lap1 = O.build_laplacian(img, dims, 60.0, "sq", 8, cut_edges=cut)
    Vo, lamo, order, P, Cf = O.first_order_update(V, lam, lap0, lap1)
    np.testing.assert_allclose(up.P.cpu().numpy()[:, :m], P, rtol=0, atol=1e-12)
    assert_lam(up.lambda_hat, lamo)
    np.testing.assert_array_equal(up.order, order)
    _match_columns(up.V.cpu().numpy()[:, :m], Vo, lam, order, label="eigh basis (28, 24) 8-conn block cut")
    # rayleigh + cut = refresh restated on the cut Laplacian
    r = swb.update_basis(dp, image, 60.0, cut_edges=cut, method="rayleigh")
    lam_r, order_r = O.refresh(V, lap1)
    assert_lam(r.lambda_hat, lam_r)
    np.testing.assert_array_equal(r.order, order_r)


def test_solve_large_seed_system(cuda_ok):
    """S = 2000 seeds: a 2001^2 bordered system (panels beyond the
    register-resident size and beyond the shared-memory panel rows)."""
    rng = np.random.default_rng(21)
    dims = (60, 50)
    n = 3000
    img = np.clip(0.5 + 0.3 * (np.add.outer(np.arange(60), np.arange(50)).ravel(order="F") > 55) +
                  rng.normal(0, 0.05, n), 0, 1)
    lap = O.build_laplacian(img, dims, 20.0)
    vals, vecs = np.linalg.eigh(lap.matrix.toarray())
    m = 120
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=20.0, eigen=swb.EigenBasis(np.asfortranarray(vecs[:, :m]),
                                                                                    vals[:m]),
                            d_sqrt=lap.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    seeds = np.sort(rng.choice(n, 2000, replace=False))
    labs = (np.add.outer(np.arange(60), np.arange(50)).ravel(order="F")[seeds] > 55).astype(int)
    f = swb.solve_fast(pack, lap.matrix, _prob(seeds, labs, n=n), m_use=m, want_field=True)
    u = O.solve_fast(vecs[:, :m], vals[:m], lap.d_sqrt, lap.matrix, seeds, labs, 2, m_use=m)
    np.testing.assert_allclose(f.values, u, atol=1e-9)
    assert_labels_match(swb.hard_labels(f).labels, u)


@pytest.mark.parametrize("dims", [(1, 23), (23, 1), (2, 2), (3, 1, 5), (1, 1, 9)])
def test_degenerate_shapes_update_and_solve(cuda_ok, dims):
    """Lines of length one, single-line volumes and tiny lattices through the
    stencil ring, the projection / rotation and the solve."""
    rng = np.random.default_rng(sum(dims))
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.2 * rng.standard_normal(n), 0, 1)
    lap0 = O.build_laplacian(img, dims, 5.0)
    vals, vecs = np.linalg.eigh(lap0.matrix.toarray())
    m = min(n, 4)
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=5.0, eigen=swb.EigenBasis(np.asfortranarray(vecs[:, :m]),
                                                                                   vals[:m]),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    dp = swb.to_device(pack, image=image)
    up = swb.update_basis(dp, image, 7.0, method="first_order", keep_P=True)
    lap1 = O.build_laplacian(img, dims, 7.0)
    Vo, lamo, order, P, _ = O.first_order_update(vecs[:, :m], vals[:m], lap0, lap1)
    np.testing.assert_allclose(up.P.cpu().numpy()[:, :m], P, rtol=0, atol=1e-12)
    assert_lam(up.lambda_hat, lamo)
    seeds = np.array([0, n - 1])
    f = swb.solve_fast(up, up.laplacian, _prob(seeds, [0, 1], n=n), want_field=True)
    u = O.solve_fast(Vo, lamo, lap1.d_sqrt, lap1.matrix, seeds, [0, 1], 2)
    np.testing.assert_allclose(f.values, u, atol=1e-9)


def test_single_voxel_graph_is_degenerate(cuda_ok):
    import torch
    lat = swb.LatticeSpec.make((1, 1))
    with pytest.raises(swb.DegenerateGraph):
        swb.DeviceGraph.build(torch.tensor([0.5], dtype=torch.float64, device="cuda"), lat, 1.0)


@pytest.mark.parametrize("dims,conn,m,S,gamma", [((40, 36), 4, 30, 200, 0.0), ((40, 36), 4, 30, 200, 0.7),
                                                 ((14, 12, 10), 6, 60, 300, 0.0), ((48, 40), 8, 20, 600, 0.0)])
def test_woodbury_seed_system_matches_lapack(cuda_ok, dims, conn, m, S, gamma):
    """With many more seeds than basis columns the seed system A = I - Ut Vt^T
    (rank m, or m + 2 with the gamma = 0 border) is solved through the r x r
    K = I - Vt^T Ut (Woodbury) and its rcond estimated from the same identity:
    fields match the oracle's LU solve, rcond LAPACK dgecon on the full A."""
    rng = np.random.default_rng(S + m)
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * (rng.random(n) < 0.25) + rng.normal(0, 0.05, n), 0, 1)
    lap = O.build_laplacian(img, dims, 20.0, "abs", conn)
    vals, vecs = np.linalg.eigh(lap.matrix.toarray())
    V, lam = vecs[:, :m], vals[:m]
    k = 3
    seeds = np.sort(rng.choice(n, S, replace=False))
    labs = rng.integers(0, k, S)
    pri = None
    if gamma > 0:
        pri = rng.random((n, k))
        pri /= pri.sum(axis=1, keepdims=True)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=20.0, eigen=swb.EigenBasis(np.asfortranarray(V), lam),
                            d_sqrt=lap.d_sqrt, provenance=swb.PackProvenance(b""))
    prob = swb.LabelProblem(num_labels=k, seeds=swb.SeedPartition(n, seeds, labs), priors=pri, gamma=gamma)
    f = swb.solve_fast(pack, lap, prob, want_field=True)
    u_ref, parts = O.solve_fast(V, lam, lap.d_sqrt, lap.matrix, seeds, labs, k, gamma=gamma, priors=pri,
                                return_parts=True)
    np.testing.assert_allclose(f.values, u_ref, rtol=0, atol=1e-10)
    assert_labels_match(swb.hard_labels(f).labels, u_ref)
    np.testing.assert_allclose(f.rcond_dev.item(), parts["rcond"], rtol=1e-6)


def test_woodbury_singular_seed_system(cuda_ok):
    """A rank-deficient basis (duplicated columns) makes the seed system
    singular; through the Woodbury path it raises SingularSmallSystem exactly
    when the oracle's LU / dgecon does."""
    dims = (40, 36)
    rng = np.random.default_rng(3)
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * (rng.random(n) < 0.25) + rng.normal(0, 0.05, n), 0, 1)
    lap = O.build_laplacian(img, dims, 20.0, "abs", 4)
    vals, vecs = np.linalg.eigh(lap.matrix.toarray())
    m = 12
    V = vecs[:, :m].copy()
    V[:, 3] = V[:, 2]
    V[:, 4] = V[:, 2]
    lam = np.full(m, 1e-3)
    seeds = np.sort(rng.choice(n, 150, replace=False))
    labs = np.arange(150) % 2
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=20.0, eigen=swb.EigenBasis(np.asfortranarray(V), lam),
                            d_sqrt=lap.d_sqrt, provenance=swb.PackProvenance(b""))
    prob = _prob(seeds, labs, n=n)
    try:
        O.solve_fast(V, lam, lap.d_sqrt, lap.matrix, seeds, labs, 2)
        expect = None
    except O.OracleError as exc:
        expect = exc.kind
    if expect == "SingularSmallSystem":
        with pytest.raises(swb.SingularSmallSystem):
            swb.solve_fast(pack, lap, prob)
    else:
        f = swb.solve_fast(pack, lap, prob, want_field=True)
        np.testing.assert_allclose(f.values, O.solve_fast(V, lam, lap.d_sqrt, lap.matrix, seeds, labs, 2),
                                   rtol=0, atol=1e-9)
