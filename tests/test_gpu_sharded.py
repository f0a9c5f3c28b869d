"""The z-slab sharded path on one GPU: 1-4 shards emulated in one process
(LocalComm: collectives are device copies / sums), real kernels with slab
row ranges and halos, checked against the single-GPU API path."""

import numpy as np
import pytest

import paper_1607_04174_b200 as swb
from oracle import rw_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("dims,conn,mode", [((12, 10, 16), 6, "sq"), ((24, 32), 8, "sq"), ((20, 24), 4, "abs")])
def test_sharded_matches_single_gpu(cuda_ok, world, dims, conn, mode):
    import torch
    from paper_1607_04174_b200.sharded import (CudaBackend, LocalComm, make_shards_from_global, sharded_solve,
                                                sharded_update)
    rng = np.random.default_rng(world + len(dims))
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * (rng.random(n) < 0.3) + rng.normal(0, 0.05, n), 0, 1)
    lap0 = O.build_laplacian(img, dims, 10.0, mode, conn)
    vals, vecs = np.linalg.eigh(lap0.matrix.toarray())
    m = 24
    V, lam = vecs[:, :m], vals[:m]
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=10.0, eigen=swb.EigenBasis(np.asfortranarray(V), lam),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    dp = swb.to_device(pack, image=image, connectivity=conn, weight_mode=mode)
    up = swb.update_basis(dp, image, 14.0)
    seeds = np.sort(rng.choice(n, 12, replace=False))
    labs = np.arange(12) % 2
    ref = swb.solve_fast(up, up.laplacian, swb.LabelProblem(num_labels=2, seeds=swb.SeedPartition(n, seeds, labs)),
                         want_field=True)
    shards = make_shards_from_global(dp.V, dp.values_dev, None, dp.lattice, dp.image_dev, 10.0, world)
    # poison halos: the exchange must fill them
    for sh in shards:
        if sh.plan.halo_lo:
            sh.V[:sh.plan.unit] = 1e30
        if sh.plan.halo_hi:
            sh.V[-sh.plan.unit:] = 1e30
    be, comm = CudaBackend(), LocalComm()
    sharded_update(shards, comm, be, 14.0)
    out = sharded_solve(shards, comm, be, seeds, labs, 2, want_u=True)
    V_sh = torch.cat([sh.own()[:, :m] for sh in shards]).cpu().numpy()
    np.testing.assert_allclose(V_sh, up.V[:, :m].cpu().numpy(), atol=1e-12)
    np.testing.assert_allclose(shards[0].values.cpu().numpy(), up.lambda_hat, rtol=1e-12, atol=1e-15)
    U = torch.cat([o[2] for o in out]).cpu().numpy()
    np.testing.assert_allclose(U, ref.values, atol=1e-10)
    labels = torch.cat([o[0] for o in out]).cpu().numpy()
    gap = O.top2_gap(ref.values)
    assert not ((labels != swb.hard_labels(ref).labels) & (gap > 1e-9)).any()


@pytest.mark.parametrize("dims,conn,mode", [((12, 10, 16), 6, "sq"), ((24, 32), 8, "sq")])
def test_sharded_through_c_comm_matches_local(cuda_ok, dims, conn, mode):
    """The sharded update + solve with the collectives through the library's
    own NCCL entry points (swb_comm_*: unique id, init, all-reduce, halo
    Send/Recv) -- one rank (one GPU is what the sandbox has) -- equals the
    in-process LocalComm run bit for bit."""
    import torch
    from paper_1607_04174_b200.sharded import (CComm, CudaBackend, LocalComm, make_shards_from_global,
                                                sharded_solve, sharded_update)
    rng = np.random.default_rng(7)
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * (rng.random(n) < 0.3) + rng.normal(0, 0.05, n), 0, 1)
    lap0 = O.build_laplacian(img, dims, 10.0, mode, conn)
    vals, vecs = np.linalg.eigh(lap0.matrix.toarray())
    m = 24
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=10.0,
                            eigen=swb.EigenBasis(np.asfortranarray(vecs[:, :m]), vals[:m]),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    dp = swb.to_device(pack, image=image, connectivity=conn, weight_mode=mode)
    seeds = np.sort(rng.choice(n, 12, replace=False))
    labs = np.arange(12) % 2
    outs = []
    for comm in (LocalComm(), CComm(0, 1)):
        shards = make_shards_from_global(dp.V, dp.values_dev, None, dp.lattice, dp.image_dev, 10.0, 1)
        be = CudaBackend()
        sharded_update(shards, comm, be, 14.0)
        out = sharded_solve(shards, comm, be, seeds, labs, 2, want_u=True)
        torch.cuda.synchronize()
        outs.append((shards[0].own()[:, :m].cpu().numpy(), out[0][2].cpu().numpy(), out[0][0].cpu().numpy()))
        if isinstance(comm, CComm):
            buf = torch.arange(10, dtype=torch.float64, device="cuda")
            comm.allreduce_sum([buf])
            assert buf.cpu().numpy().tolist() == list(range(10))
            comm.close()
    (va, ua, la), (vb, ub, lb) = outs
    np.testing.assert_array_equal(va, vb)
    np.testing.assert_array_equal(ua, ub)
    np.testing.assert_array_equal(la, lb)


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("dims,conn,mode", [((12, 10, 16), 6, "sq"), ((24, 32), 8, "sq")])
def test_sharded_fused_matches_single_gpu(cuda_ok, world, dims, conn, mode):
    """sharded_update_and_solve on 1/2/4 emulated shards vs the single-GPU
    update_and_solve: V' and eigenvalues to 1e-12, fields to 1e-10."""
    import torch
    from paper_1607_04174_b200.sharded import (CudaBackend, LocalComm, make_shards_from_global,
                                                sharded_update_and_solve)
    rng = np.random.default_rng(world + 3 * len(dims))
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * (rng.random(n) < 0.3) + rng.normal(0, 0.05, n), 0, 1)
    lap0 = O.build_laplacian(img, dims, 10.0, mode, conn)
    vals, vecs = np.linalg.eigh(lap0.matrix.toarray())
    m = 24
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=10.0,
                            eigen=swb.EigenBasis(np.asfortranarray(vecs[:, :m]), vals[:m]),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    dp = swb.to_device(pack, image=image, connectivity=conn, weight_mode=mode)
    seeds = np.sort(rng.choice(n, 14, replace=False))
    labs = np.arange(14) % 3
    prob = swb.LabelProblem(num_labels=3, seeds=swb.SeedPartition(n, seeds, labs))
    up, ref = swb.update_and_solve(dp, image, prob, 14.0, want_field=True)
    shards = make_shards_from_global(dp.V, dp.values_dev, None, dp.lattice, dp.image_dev, 10.0, world)
    for sh in shards:
        if sh.plan.halo_lo:
            sh.V[:sh.plan.unit] = 1e30
        if sh.plan.halo_hi:
            sh.V[-sh.plan.unit:] = 1e30
    out = sharded_update_and_solve(shards, LocalComm(), CudaBackend(), 14.0, seeds, labs, 3, want_u=True)
    V_sh = torch.cat([sh.own()[:, :m] for sh in shards]).cpu().numpy()
    np.testing.assert_allclose(V_sh, up.V[:, :m].cpu().numpy(), atol=1e-12)
    np.testing.assert_allclose(shards[0].values.cpu().numpy(), up.lambda_hat, rtol=1e-12, atol=1e-15)
    U = torch.cat([o[2] for o in out]).cpu().numpy()
    np.testing.assert_allclose(U, ref.values, atol=1e-10)
    labels = torch.cat([o[0] for o in out]).cpu().numpy()
    gap = O.top2_gap(ref.values)
    assert not ((labels != swb.hard_labels(ref).labels) & (gap > 1e-9)).any()
