"""Multi-rank z-slab orchestration on CPU: world_size 2 (and 3) over gloo with
the numpy shard backend, checked against the single-process oracle."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rw_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(dims, conn, mode, m, seed):
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * (rng.random(n) < 0.3) + rng.normal(0, 0.05, n), 0, 1)
    lap0 = O.build_laplacian(img, dims, 10.0, mode, conn)
    vals, vecs = np.linalg.eigh(lap0.matrix.toarray())
    seeds = np.sort(rng.choice(n, 10, replace=False))
    labs = np.arange(10) % 2
    priors = rng.random((n, 2))
    priors /= priors.sum(axis=1, keepdims=True)
    return img, vecs[:, :m], vals[:m], lap0, seeds, labs, priors


def _worker(rank, world, port, outdir, dims, conn, mode, m, gamma, fused=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from np_shard_backend import NumpyBackend
    from paper_1607_04174_b200.device import LatticeSpec
    from paper_1607_04174_b200.sharded import (DistComm, Shard, SlabPlan, sharded_solve, sharded_update,
                                                sharded_update_and_solve)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    img, V, lam, lap0, seeds, labs, priors = _problem(dims, conn, mode, m, 7)
    lattice = LatticeSpec.make(dims, conn, mode)
    be = NumpyBackend()
    comm = DistComm()
    plan = SlabPlan.make(dims, world, rank)
    Vl = torch.zeros((plan.local_rows, m + (m % 2)), dtype=torch.float64)
    Vl[:, :m] = torch.from_numpy(V[plan.row_base: plan.row_base + plan.local_rows])
    # poison the halo rows: the exchange must fill them
    if plan.halo_lo:
        Vl[:plan.unit] = 1e30
    if plan.halo_hi:
        Vl[-plan.unit:] = 1e30
    sh = Shard(plan, Vl, m, torch.from_numpy(lam.copy()), lattice, torch.from_numpy(img), be.graph(img, lattice, 10.0),
               10.0)
    if fused:
        (labels, _, U, rc), = sharded_update_and_solve([sh], comm, be, 14.0, seeds, labs, 2)
    else:
        sharded_update([sh], comm, be, 14.0)
        pri_own = [torch.from_numpy(priors[plan.own_begin: plan.own_end])] if gamma > 0 else None
        (labels, _, U, rc), = sharded_solve([sh], comm, be, seeds, labs, 2, gamma=gamma, priors=pri_own)
    parts = [None] * world
    dist.all_gather_object(parts, (plan.own_begin, sh.own()[:, :m].numpy(), U.numpy(), labels.numpy(),
                                   sh.values.numpy()))
    if rank == 0:
        parts.sort(key=lambda p: p[0])
        np.savez(os.path.join(outdir, "out.npz"), V=np.concatenate([p[1] for p in parts]),
                 U=np.concatenate([p[2] for p in parts]), labels=np.concatenate([p[3] for p in parts]),
                 lam=parts[0][4])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,conn,mode,gamma,fused", [(2, (8, 6, 10), 6, "abs", 0.0, False),
                                                              (3, (8, 6, 10), 6, "sq", 0.0, False),
                                                              (2, (12, 14), 8, "sq", 0.0, False),
                                                              (2, (8, 6, 10), 6, "abs", 0.5, False),
                                                              (2, (8, 6, 10), 6, "abs", 0.0, True),
                                                              (3, (12, 14), 8, "sq", 0.0, True)])
def test_sharded_update_and_solve_gloo(world, dims, conn, mode, gamma, fused):
    """fused: sharded_update_and_solve (the seed system before the rotation,
    the reconstruction as extra rotation columns) -- same results."""
    m = 16
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, dims, conn, mode, m, gamma, fused), nprocs=world,
                 join=True)
        out = np.load(os.path.join(d, "out.npz"))
    img, V, lam, lap0, seeds, labs, priors = _problem(dims, conn, mode, m, 7)
    lap1 = O.build_laplacian(img, dims, 14.0, mode, conn)
    V1, lam1, _, _, _ = O.first_order_update(V, lam, lap0, lap1)
    np.testing.assert_allclose(out["lam"], lam1, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(out["V"], V1, atol=1e-12)
    if gamma > 0:
        u = O.solve_fast(V1, lam1, lap1.d_sqrt, lap1.matrix, seeds, labs, 2, gamma=gamma, priors=priors)
    else:
        u = O.solve_fast(V1, lam1, lap1.d_sqrt, lap1.matrix, seeds, labs, 2)
    np.testing.assert_allclose(out["U"], u, atol=1e-10)
    np.testing.assert_array_equal(out["labels"], O.hard_labels(u))


def test_slab_plan_partition():
    from paper_1607_04174_b200.sharded import SlabPlan
    for world in (1, 2, 3, 4, 8):
        plans = [SlabPlan.make((16, 16, 37), world, r) for r in range(world)]
        assert plans[0].own_begin == 0 and plans[-1].own_end == 16 * 16 * 37
        for a, b in zip(plans, plans[1:]):
            assert a.own_end == b.own_begin
        assert not plans[0].halo_lo and not plans[-1].halo_hi
        for p in plans:
            assert p.row_base + p.local_rows >= p.own_end
            assert p.own_slice().stop - p.own_slice().start == p.own_end - p.own_begin


def test_sharded_solve_sorts_seeds_and_rejects_duplicates():
    """sharded_solve takes raw seed arrays: they are sorted (labels permuted
    alike) before the binary-searching seed kernels; duplicates raise."""
    from paper_1607_04174_b200 import errors
    from paper_1607_04174_b200.sharded import _sorted_seeds
    idx, lab = _sorted_seeds(np.array([9, 3, 7, 1]), np.array([0, 1, 2, 3]))
    assert idx.tolist() == [1, 3, 7, 9] and lab.tolist() == [3, 1, 2, 0]
    idx, lab = _sorted_seeds(torch.tensor([2, 5]), torch.tensor([1, 0]))
    assert idx.tolist() == [2, 5] and lab.tolist() == [1, 0]
    with pytest.raises(errors.InvalidParam):
        _sorted_seeds(np.array([4, 2, 4]), np.array([0, 1, 0]))
