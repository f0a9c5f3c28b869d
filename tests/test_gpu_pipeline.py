"""The composite C entry points (swb_update_first_order, swb_rw_solve,
swb_update_and_solve) --
the whole update / whole solve for hosts that bind the C ABI directly --
against the Python API path (same kernels; tolerance 1e-12) and, through
it, the oracle."""

import ctypes as C

import numpy as np
import pytest

import paper_1607_04174_b200 as swb
from oracle import rw_oracle as O
from paper_1607_04174_b200 import _lib
from paper_1607_04174_b200.device import DeviceGraph, ptr, round_up, stream_handle

pytestmark = pytest.mark.gpu


def _case(dims, m, b0, conn=None, mode="abs", seed=3):
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * (rng.random(n) < 0.2) + rng.normal(0, 0.05, n), 0, 1)
    lap0 = O.build_laplacian(img, dims, b0, mode, conn)
    vals, vecs = np.linalg.eigh(lap0.matrix.toarray())
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=b0, eigen=swb.EigenBasis(np.asfortranarray(vecs[:, :m]),
                                                                                  vals[:m]),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    dp = swb.to_device(pack, image=image, connectivity=conn, weight_mode=mode)
    return rng, n, image, dp


def _update_c(dp, b0, b1):
    import torch
    n, m, ldv = dp.n_vertices, dp.m, dp.ldv
    lat = dp.lattice.c_struct()
    V_out = torch.empty_like(dp.V)
    lam = torch.empty(m, dtype=torch.float64, device="cuda")
    order = torch.empty(m, dtype=torch.int64, device="cuda")
    dsq = torch.empty(n, dtype=torch.float64, device="cuda")
    vtg = torch.empty(m, dtype=torch.float64, device="cuda")
    dnorm = torch.empty(1, dtype=torch.float64, device="cuda")
    deg = torch.empty(2, dtype=torch.int32, device="cuda")
    nbytes = _lib.size("swb_update_workspace_bytes", C.byref(lat), m)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    _lib.call("swb_update_first_order", C.byref(lat), ptr(dp.image_dev), b0, b1, None, None, ptr(dp.V), ldv,
              ptr(dp.values_dev), m, 0.5, ptr(V_out), ptr(lam), ptr(order), ptr(dsq), ptr(vtg), ptr(dnorm), ptr(deg),
              ptr(ws), nbytes, stream_handle())
    return V_out, lam, order, dsq, vtg, dnorm, deg


def _solve_c(dp_lat, graph, V, values, vtg, m, seeds, labs, k, gamma=0.0, priors=None):
    import torch
    n = V.shape[0]
    lat = dp_lat.c_struct()
    s = len(seeds)
    sidx = torch.tensor(np.asarray(seeds, dtype=np.int64), device="cuda")
    slab = torch.tensor(np.asarray(labs, dtype=np.int32), device="cuda")
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    top2 = torch.empty(n, dtype=torch.float64, device="cuda")
    ldu = round_up(k, 2)
    U = torch.empty((n, ldu), dtype=torch.float64, device="cuda")
    pri = None
    if priors is not None:
        pri = torch.from_numpy(np.ascontiguousarray(priors, dtype=np.float64)).cuda()
    nbytes = _lib.size("swb_rw_solve_workspace_bytes", C.byref(lat), m, m, s, k, int(priors is not None))
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    rc = C.c_double(0.0)
    _lib.call("swb_rw_solve", C.byref(lat), ptr(graph.what), ptr(graph.diag), ptr(graph.d_sqrt_dev), ptr(V),
              V.shape[1], ptr(values), ptr(vtg), m, m, ptr(sidx) if s else None, ptr(slab) if s else None, s, k,
              float(gamma), ptr(pri), k if pri is not None else 0, ptr(labels), ptr(top2), ptr(U), ldu,
              C.byref(rc), ptr(ws), nbytes, stream_handle())
    return labels.cpu().numpy(), U[:, :k].cpu().numpy(), rc.value


@pytest.mark.parametrize("dims,conn", [((12, 10, 8), 6), ((30, 26), 8)])
def test_composite_update_and_solve_match_api(cuda_ok, dims, conn):
    rng, n, image, dp = _case(dims, 36, 12.0, conn=conn)
    up = swb.update_basis(dp, image, 17.0, method="first_order")
    V_out, lam, order, dsq, vtg, dnorm, deg = _update_c(dp, 12.0, 17.0)
    assert deg.cpu().numpy().tolist() == [0, 0]
    m = dp.m
    np.testing.assert_array_equal(order.cpu().numpy(), up.order_dev.cpu().numpy())
    np.testing.assert_allclose(lam.cpu().numpy(), up.lambda_hat, rtol=1e-14, atol=1e-16)
    np.testing.assert_allclose(V_out[:, :m].cpu().numpy(), up.V[:, :m].cpu().numpy(), rtol=0, atol=1e-14)
    np.testing.assert_allclose(vtg.cpu().numpy(), up.vtg.cpu().numpy(), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(float(dnorm.item()), up.dnorm, rtol=1e-14)
    seeds = np.sort(rng.choice(n, 14, replace=False))
    labs = np.arange(14) % 2
    f = swb.solve_fast(up, up.laplacian, swb.LabelProblem(num_labels=2, seeds=swb.SeedPartition(n, seeds, labs)),
                       want_field=True)
    g = DeviceGraph.build(dp.image_dev, dp.lattice, 17.0)
    labels, U, rc = _solve_c(dp.lattice, g, V_out, lam, vtg, m, seeds, labs, 2)
    np.testing.assert_allclose(U, f.values, atol=1e-12)
    np.testing.assert_array_equal(labels, swb.hard_labels(f).labels)
    assert rc > 1e-14


def test_composite_solve_priors_many_labels(cuda_ok):
    rng, n, image, dp = _case((12, 10, 8), 40, 12.0)
    k = 27
    pri = rng.random((n, k))
    pri /= pri.sum(axis=1, keepdims=True)
    prob = swb.LabelProblem(num_labels=k, seeds=swb.SeedPartition(n, [], []), priors=pri, gamma=1.0)
    f = swb.solve_fast(dp, None, prob, want_field=True)
    g = DeviceGraph.build(dp.image_dev, dp.lattice, 12.0)
    labels, U, rc = _solve_c(dp.lattice, g, dp.V, dp.values_dev, dp.ensure_vtg(), dp.m, [], [], k, gamma=1.0,
                             priors=pri)
    np.testing.assert_allclose(U, f.values, atol=1e-12)
    np.testing.assert_array_equal(labels, swb.hard_labels(f).labels)


def test_composite_solve_rejects_unsorted_or_duplicate_seeds(cuda_ok):
    """The seed kernels binary-search seed_idx, so swb_rw_solve validates the
    SeedPartition contract (sorted, unique, in range; graphs.py:51-98) and
    returns InvalidParam instead of silently wrong labels."""
    import torch
    rng, n, image, dp = _case((20, 18), 24, 12.0, conn=4)
    g = DeviceGraph.build(dp.image_dev, dp.lattice, 12.0)
    seeds = np.sort(rng.choice(n, 10, replace=False))
    labs = np.arange(10) % 2
    _solve_c(dp.lattice, g, dp.V, dp.values_dev, dp.ensure_vtg(), dp.m, seeds, labs, 2)   # valid: passes
    for bad_s, bad_l in [(seeds[::-1].copy(), labs), (np.concatenate([seeds[:9], seeds[8:9]]), labs),
                         (np.concatenate([seeds[:9], [n]]), labs), (seeds, np.where(labs == 1, 2, 0))]:
        with pytest.raises(swb.InvalidParam):
            _solve_c(dp.lattice, g, dp.V, dp.values_dev, dp.ensure_vtg(), dp.m, bad_s, bad_l, 2)
    flag = torch.empty(1, dtype=torch.float64, device="cuda")
    sidx = torch.tensor(seeds, device="cuda")
    slab = torch.tensor(labs.astype(np.int32), device="cuda")
    _lib.call("swb_check_seeds", ptr(sidx), ptr(slab), 10, n, 2, ptr(flag), stream_handle())
    assert float(flag.item()) == 0.0
    sidx_bad = torch.tensor(seeds[::-1].copy(), device="cuda")
    _lib.call("swb_check_seeds", ptr(sidx_bad), ptr(slab), 10, n, 2, ptr(flag), stream_handle())
    assert float(flag.item()) == 1.0


@pytest.mark.parametrize("dims,conn,k,m_use", [((12, 10, 8), 6, 2, 36), ((30, 26), 8, 3, 29), ((16, 14, 6), 6, 11, 36)])
def test_composite_fused_update_and_solve(cuda_ok, dims, conn, k, m_use):
    """swb_update_and_solve (one call: update + gamma = 0 solve with the
    reconstruction riding in the rotation) vs swb_update_first_order +
    swb_rw_solve on the same inputs: V' bit for bit (same digit products),
    eigenvalues / order / vtg identical, fields to 1e-12, labels off near-ties."""
    import torch
    rng, n, image, dp = _case(dims, 36, 12.0, conn=conn)
    V_out, lam, order, dsq, vtg, dnorm, deg = _update_c(dp, 12.0, 17.0)
    seeds = np.sort(rng.choice(n, 4 * k + 6, replace=False))
    labs = np.arange(seeds.size) % k
    g = DeviceGraph.build(dp.image_dev, dp.lattice, 17.0)
    lat = dp.lattice.c_struct()
    m, ldv = dp.m, dp.ldv
    s = seeds.size
    sidx = torch.tensor(seeds, dtype=torch.int64, device="cuda")
    slab = torch.tensor(labs, dtype=torch.int32, device="cuda")
    # the reference pair at m_use: swb_rw_solve on the updated basis
    nbytes = _lib.size("swb_rw_solve_workspace_bytes", C.byref(lat), m, m_use, s, k, 0)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    ldu = round_up(k, 2)
    labels1 = torch.empty(n, dtype=torch.int32, device="cuda")
    top2_1 = torch.empty(n, dtype=torch.float64, device="cuda")
    U1 = torch.empty((n, ldu), dtype=torch.float64, device="cuda")
    rc1 = C.c_double(0.0)
    _lib.call("swb_rw_solve", C.byref(lat), ptr(g.what), ptr(g.diag), ptr(g.d_sqrt_dev), ptr(V_out), ldv, ptr(lam),
              ptr(vtg), m, m_use, ptr(sidx), ptr(slab), s, k, 0.0, None, 0, ptr(labels1), ptr(top2_1), ptr(U1), ldu,
              C.byref(rc1), ptr(ws), nbytes, stream_handle())
    # fused
    V2 = torch.empty_like(dp.V)
    lam2 = torch.empty(m, dtype=torch.float64, device="cuda")
    order2 = torch.empty(m, dtype=torch.int64, device="cuda")
    dsq2 = torch.empty(n, dtype=torch.float64, device="cuda")
    vtg2 = torch.empty(m, dtype=torch.float64, device="cuda")
    labels2 = torch.empty(n, dtype=torch.int32, device="cuda")
    top2_2 = torch.empty(n, dtype=torch.float64, device="cuda")
    U2 = torch.empty((n, ldu), dtype=torch.float64, device="cuda")
    nbytes = _lib.size("swb_update_and_solve_workspace_bytes", C.byref(lat), m, m_use, s, k, ldv)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    rc2 = C.c_double(0.0)
    _lib.call("swb_update_and_solve", C.byref(lat), ptr(dp.image_dev), 12.0, 17.0, None, None, ptr(dp.V), ldv,
              ptr(dp.values_dev), m, 0.5, ptr(V2), ptr(lam2), ptr(order2), ptr(dsq2), ptr(vtg2), m_use, ptr(sidx),
              ptr(slab), s, k, ptr(labels2), ptr(top2_2), ptr(U2), ldu, C.byref(rc2), ptr(ws), nbytes,
              stream_handle())
    assert torch.equal(V2[:, :m], V_out[:, :m])
    assert torch.equal(lam2, lam) and torch.equal(order2, order) and torch.equal(vtg2, vtg)
    np.testing.assert_allclose(U2[:, :k].cpu().numpy(), U1[:, :k].cpu().numpy(), rtol=0, atol=1e-12)
    t = top2_1.cpu().numpy()
    l1, l2 = labels1.cpu().numpy(), labels2.cpu().numpy()
    assert not ((l1 != l2) & (t >= 1e-9)).any()
    np.testing.assert_allclose(rc2.value, rc1.value, rtol=1e-6)
