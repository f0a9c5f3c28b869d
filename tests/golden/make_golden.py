"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container only (the reference is not present on the GPU
box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``specwalk`` from /root/reference/pkg/src (read-only), runs the
hot-path functions (refresh, solve_fast, select_m, hard_labels, seed_fit,
prior_residual, the graph/Laplacian primitives) on small seeded inputs, and
writes the inputs and outputs to ``tests/golden/*.npz``.  The committed
``.npz`` files are what the tests read; this script is kept so they can be
regenerated and audited.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF))

import specwalk as sw  # noqa: E402
from specwalk.adaptive import AdaptivePolicy, prior_residual, seed_fit, select_m  # noqa: E402
from specwalk.graphs import (LaplacianMode, laplacian_from_weights,  # noqa: E402
                             weights_from_edges)


def csr_parts(prefix, mat, out):
    mat = mat.tocsr()
    mat.sort_indices()
    out[prefix + "_data"] = mat.data
    out[prefix + "_indices"] = mat.indices.astype(np.int64)
    out[prefix + "_indptr"] = mat.indptr.astype(np.int64)


def seeds_of(ph, per_region, seed):
    k = ph.labels.num_labels()
    return sw.sample_region_seeds(ph.labels.labels, k, per_region,
                                  np.random.default_rng(seed))


def case_path3():
    out = {}
    image = sw.Image((3, 1), [0.0, 0.0, 0.0])
    pack = sw.precompute(image, 1.0, m=3)
    lap = sw.laplacian(sw.build_graph(image, 1.0), LaplacianMode.NORMALIZED)
    prob = sw.LabelProblem(num_labels=2, seeds=sw.SeedPartition(3, [0, 2], [0, 1]), gamma=0.0)
    u = sw.solve_fast(pack, lap, prob, m_use=3)
    out.update(dims=np.array([3, 1]), intensities=image.intensities, beta=1.0,
               V=np.asarray(pack.eigen.vectors), lam=pack.eigen.values, d_sqrt=pack.d_sqrt,
               seed_idx=np.array([0, 2]), seed_lab=np.array([0, 1]), U=u.values,
               labels=sw.hard_labels(u).labels)
    csr_parts("lap", lap.matrix, out)
    np.savez_compressed(OUT / "path3.npz", **out)


def case_phantom16():
    out = {}
    ph = sw.make_phantom("blobs2d", (16, 16), rng_seed=3, noise_sigma=0.05, num_regions=2)
    pack = sw.precompute(ph.image, 15.0, m=64)
    lap = sw.laplacian(sw.build_graph(ph.image, 15.0), LaplacianMode.NORMALIZED)
    n = ph.image.n_voxels
    out.update(dims=np.array(ph.image.dims), intensities=ph.image.intensities,
               truth=ph.labels.labels, beta=15.0, V=np.asarray(pack.eigen.vectors),
               lam=pack.eigen.values, d_sqrt=pack.d_sqrt, lap_d_sqrt=lap.d_sqrt)
    csr_parts("lap", lap.matrix, out)
    # refresh at several betas (refresh.py:63-82)
    for b in (15.0, 33.0, 45.0):
        r = sw.refresh(pack, ph.image, b)
        tag = f"refresh_{int(b)}"
        out[tag + "_lam"] = r.lambda_hat
        out[tag + "_order"] = r.order
        out[tag + "_d_sqrt"] = r.d_sqrt
        csr_parts(tag + "_lap", r.laplacian.matrix, out)
    # gamma = 0 solves at several m_use
    seeds = seeds_of(ph, 3, 0)
    out["seeds0_idx"], out["seeds0_lab"] = seeds.seed_indices, seeds.seed_labels
    prob = sw.LabelProblem(num_labels=2, seeds=seeds, gamma=0.0)
    for m_use in (24, 32, 64):
        u = sw.solve_fast(pack, lap, prob, m_use=m_use)
        out[f"solve0_m{m_use}_U"] = u.values
        out[f"solve0_m{m_use}_labels"] = sw.hard_labels(u).labels
    # gamma > 0 with priors
    rng = np.random.default_rng(17)
    priors = rng.random((n, 2))
    priors /= priors.sum(axis=1, keepdims=True)
    out["priors"] = priors
    seeds1 = seeds_of(ph, 4, 7)
    out["seeds1_idx"], out["seeds1_lab"] = seeds1.seed_indices, seeds1.seed_labels
    prob = sw.LabelProblem(num_labels=2, seeds=seeds1, priors=priors, gamma=0.5)
    u = sw.solve_fast(pack, lap, prob, m_use=40)
    out["solveg_m40_U"] = u.values
    # no seeds, constant priors (test_fastrw.py:103-110 shape)
    cpri = np.tile([0.3, 0.7], (n, 1))
    prob = sw.LabelProblem(num_labels=2, seeds=sw.SeedPartition(n, [], []), priors=cpri, gamma=2.0)
    out["solve_noseed_U"] = sw.solve_fast(pack, lap, prob, m_use=8).values
    # random priors, no seeds
    prob = sw.LabelProblem(num_labels=2, seeds=sw.SeedPartition(n, [], []), priors=priors, gamma=1.0)
    out["solve_noseed_rand_U"] = sw.solve_fast(pack, lap, prob, m_use=48).values
    # refreshed pack solve (beta 45)
    r = sw.refresh(pack, ph.image, 45.0)
    prob = sw.LabelProblem(num_labels=2, seeds=seeds, gamma=0.0)
    u = sw.solve_fast(r, r.laplacian, prob, m_use=40)
    out["solve_refresh45_m40_U"] = u.values
    # select_m variants (adaptive.py:133-185)
    for tag, pol, sd in (("default", AdaptivePolicy(), seeds),
                         ("loose", AdaptivePolicy(epsilon=1e9), seeds_of(ph, 3, 1)),
                         ("tight", AdaptivePolicy(epsilon=1e-9), seeds_of(ph, 50, 1)),
                         ("eps3e4", AdaptivePolicy(epsilon=3e-4), seeds_of(ph, 6, 5))):
        prob = sw.LabelProblem(num_labels=2, seeds=sd, gamma=0.0)
        m_use, info = select_m(pack, prob, pol)
        out[f"sel_{tag}_idx"], out[f"sel_{tag}_lab"] = sd.seed_indices, sd.seed_labels
        out[f"sel_{tag}_eps"] = pol.epsilon
        out[f"sel_{tag}_m"] = m_use
        out[f"sel_{tag}_sat"] = info["saturated"]
        out[f"sel_{tag}_steps_m"] = np.array([s["m"] for s in info["steps"]])
        out[f"sel_{tag}_steps_f"] = np.array([s["f"] for s in info["steps"]])
    pri4 = np.random.default_rng(3).random((n, 4))
    pri4 /= pri4.sum(axis=1, keepdims=True)
    out["pri4"] = pri4
    for tag, eps in (("p_loose", 10.0), ("p_tight", 1e-6), ("p_mid", 0.05)):
        prob = sw.LabelProblem(num_labels=4, seeds=sw.SeedPartition(n, [], []), priors=pri4, gamma=1.0)
        m_use, info = select_m(pack, prob, AdaptivePolicy(epsilon=eps))
        out[f"sel_{tag}_eps"] = eps
        out[f"sel_{tag}_m"] = m_use
        out[f"sel_{tag}_sat"] = info["saturated"]
        out[f"sel_{tag}_steps_m"] = np.array([s["m"] for s in info["steps"]])
        out[f"sel_{tag}_steps_g"] = np.array([s["g"] for s in info["steps"]])
    # smooth two-label priors: the prior test stops inside the schedule
    xs = np.arange(n) % 16
    p0 = 0.5 + 0.3 * np.cos(xs / 5.0)
    psm = np.stack([p0, 1.0 - p0], axis=1)
    out["psmooth"] = psm
    for tag, eps in (("ps_a", 0.05), ("ps_b", 0.01), ("ps_c", 0.002)):
        prob = sw.LabelProblem(num_labels=2, seeds=sw.SeedPartition(n, [], []), priors=psm, gamma=1.0)
        m_use, info = select_m(pack, prob, AdaptivePolicy(epsilon=eps))
        out[f"sel_{tag}_eps"] = eps
        out[f"sel_{tag}_m"] = m_use
        out[f"sel_{tag}_sat"] = info["saturated"]
        out[f"sel_{tag}_steps_m"] = np.array([s["m"] for s in info["steps"]])
        out[f"sel_{tag}_steps_g"] = np.array([s["g"] for s in info["steps"]])
    np.savez_compressed(OUT / "phantom16.npz", **out)


def case_blobs3d():
    out = {}
    ph = sw.make_phantom("blobs3d", (6, 5, 4), rng_seed=5, noise_sigma=0.05, num_regions=2)
    pack = sw.precompute(ph.image, 10.0, m=30)
    lap = sw.laplacian(sw.build_graph(ph.image, 10.0), LaplacianMode.NORMALIZED)
    n = ph.image.n_voxels
    out.update(dims=np.array(ph.image.dims), intensities=ph.image.intensities,
               beta=10.0, V=np.asarray(pack.eigen.vectors), lam=pack.eigen.values,
               d_sqrt=pack.d_sqrt)
    csr_parts("lap", lap.matrix, out)
    r = sw.refresh(pack, ph.image, 25.0)
    out["refresh_25_lam"], out["refresh_25_order"] = r.lambda_hat, r.order
    out["refresh_25_d_sqrt"] = r.d_sqrt
    csr_parts("refresh_25_lap", r.laplacian.matrix, out)
    seeds = seeds_of(ph, 3, 2)
    out["seeds_idx"], out["seeds_lab"] = seeds.seed_indices, seeds.seed_labels
    prob = sw.LabelProblem(num_labels=2, seeds=seeds, gamma=0.0)
    out["solve0_m20_U"] = sw.solve_fast(pack, lap, prob, m_use=20).values
    out["solve_refresh_m30_U"] = sw.solve_fast(r, r.laplacian, prob, m_use=30).values
    rng = np.random.default_rng(4)
    priors = rng.random((n, 3))
    priors /= priors.sum(axis=1, keepdims=True)
    out["priors3"] = priors
    seeds3 = sw.SeedPartition(n, [3, 50, 97], [0, 1, 2])
    prob = sw.LabelProblem(num_labels=3, seeds=seeds3, priors=priors, gamma=0.25)
    out["solveg3_m30_U"] = sw.solve_fast(pack, lap, prob, m_use=30).values
    np.savez_compressed(OUT / "blobs3d.npz", **out)


def _lattice_dims_edges(dims, conn):
    """Edge list for the non-default modes, built with the reference's own
    lattice_edges for the axis part and explicit diagonals for 8-conn."""
    heads, tails = sw.graphs.lattice_edges(dims)
    if conn == 8:
        nx, ny = dims
        grid = np.arange(nx * ny).reshape(dims, order="F")
        h1, t1 = grid[:-1, :-1].ravel(order="F"), grid[1:, 1:].ravel(order="F")
        h2, t2 = grid[1:, :-1].ravel(order="F"), grid[:-1, 1:].ravel(order="F")
        heads = np.concatenate([heads, h1, h2])
        tails = np.concatenate([tails, t1, t2])
    return heads, tails


def case_modes():
    """(dI)^2 weights, 8-connectivity and an edge cut: Laplacians from the
    reference primitives weights_from_edges + laplacian_from_weights."""
    out = {}
    dims = (14, 12)
    rng = np.random.default_rng(21)
    xs, ys = np.meshgrid(np.arange(dims[0]), np.arange(dims[1]), indexing="ij")
    img = np.where((xs - 6.5) ** 2 + (ys - 5.5) ** 2 <= 16, 0.7, 0.3)
    img = np.clip(img + rng.normal(0, 0.05, dims), 0, 1).reshape(-1, order="F")
    n = img.size
    out["dims"], out["intensities"] = np.array(dims), img
    for conn in (4, 8):
        heads, tails = _lattice_dims_edges(dims, conn)
        for mode in ("abs", "sq"):
            for beta in (60.0, 90.0):
                d = img[heads] - img[tails]
                arg = np.abs(d) if mode == "abs" else d * d
                w = np.maximum(np.exp(-beta * arg), sw.graphs.W_MIN)
                lap = laplacian_from_weights(weights_from_edges(n, heads, tails, w),
                                             LaplacianMode.NORMALIZED)
                tag = f"c{conn}_{mode}_{int(beta)}"
                csr_parts(tag, lap.matrix, out)
                out[tag + "_d_sqrt"] = lap.d_sqrt
    # edge cut: remove edges crossing the boundary of a 4x4 block at (5, 3)
    heads, tails = _lattice_dims_edges(dims, 8)

    def inside(f):
        x, y = f % dims[0], f // dims[0]
        return (x >= 5) & (x < 9) & (y >= 3) & (y < 7)

    cut = inside(heads) != inside(tails)
    d = img[heads] - img[tails]
    w = np.maximum(np.exp(-60.0 * (d * d)), sw.graphs.W_MIN)
    w_cut = np.where(cut, 0.0, w)
    lap = laplacian_from_weights(weights_from_edges(n, heads, tails, w_cut),
                                 LaplacianMode.NORMALIZED)
    out["cut_mask"] = cut
    csr_parts("cut_c8_sq_60", lap.matrix, out)
    out["cut_c8_sq_60_d_sqrt"] = lap.d_sqrt
    # a solve on the cut Laplacian with an orthonormal basis of its eigvecs
    dense = lap.matrix.toarray()
    vals, vecs = np.linalg.eigh(0.5 * (dense + dense.T))
    V = vecs[:, :40]
    lam = vals[:40]
    out["cut_V"], out["cut_lam"] = V, lam
    seeds = sw.SeedPartition(n, [0, 15, 100, 80, 90, 60], [0, 0, 1, 1, 1, 0])
    prob = sw.LabelProblem(num_labels=2, seeds=seeds, gamma=0.0)

    class _Pack:
        def __init__(self):
            self.eigen = sw.EigenBasis(V, lam)
            self.d_sqrt = lap.d_sqrt
            self.dims = dims

    u = sw.solve_fast(_Pack(), lap, prob, m_use=40)
    out["cut_seeds_idx"], out["cut_seeds_lab"] = seeds.seed_indices, seeds.seed_labels
    out["cut_U"] = u.values
    np.savez_compressed(OUT / "modes.npz", **out)


def case_adaptive_kats():
    out = {}
    rng = np.random.default_rng(8)
    for i, (s, m, bound) in enumerate(((30, 12, 5.0), (12, 20, 3.0), (40, 8, 0.5),
                                       (8, 8, 1e3), (25, 10, 0.05))):
        q = rng.standard_normal((s, m))
        u = (rng.random(s) > 0.5).astype(float) * rng.random(s)
        out[f"sf{i}_q"], out[f"sf{i}_u"], out[f"sf{i}_b"] = q, u, bound
        out[f"sf{i}_f"] = seed_fit(q, u, bound)
    q = np.linalg.qr(rng.standard_normal((50, 14)))[0]
    p = rng.random(50)
    g1, r1 = prior_residual(q[:, :6], p)
    g2, r2 = prior_residual(q, p, cached=r1, cached_m=6)
    out.update(pr_q=q, pr_p=p, pr_g1=g1, pr_r1=r1, pr_g2=g2, pr_r2=r2)
    np.savez_compressed(OUT / "adaptive.npz", **out)


def case_errors():
    """Reference exception classes for boundary cases."""
    out = {}
    ph = sw.make_phantom("blobs2d", (8, 8), rng_seed=1, noise_sigma=0.05, num_regions=2)
    pack = sw.precompute(ph.image, 15.0, m=16)
    lap = sw.laplacian(sw.build_graph(ph.image, 15.0), LaplacianMode.NORMALIZED)
    seeds = seeds_of(ph, 2, 0)
    prob = sw.LabelProblem(num_labels=2, seeds=seeds, gamma=0.0)
    kinds = {}
    for tag, kwargs in (("m1", {"m_use": 1}), ("m0", {"m_use": 0}), ("m99", {"m_use": 99})):
        try:
            sw.solve_fast(pack, lap, prob, **kwargs)
            kinds[tag] = "ok"
        except Exception as exc:  # noqa: BLE001
            kinds[tag] = type(exc).__name__
    # every voxel seeded -> one-hot field, no solve
    alls = sw.SeedPartition(64, np.arange(64), (np.arange(64) % 2))
    u = sw.solve_fast(pack, lap, sw.LabelProblem(num_labels=2, seeds=alls, gamma=0.0), m_use=4)
    out["allseed_U"] = u.values
    out["V"], out["lam"], out["d_sqrt"] = np.asarray(pack.eigen.vectors), pack.eigen.values, pack.d_sqrt
    csr_parts("lap", lap.matrix, out)
    out["seeds_idx"], out["seeds_lab"] = seeds.seed_indices, seeds.seed_labels
    out["kinds_keys"] = np.array(list(kinds.keys()))
    out["kinds_vals"] = np.array(list(kinds.values()))
    # hard_labels tie KATs (test_images.py:77-81)
    f = sw.ProbabilityField((3, 1), [[0.5, 0.5], [0.2, 0.8], [1 / 3, 1 / 3]][:2] + [[0.6, 0.4]])
    out["ties_in"] = f.values
    out["ties_out"] = sw.hard_labels(f).labels
    np.savez_compressed(OUT / "errors.npz", **out)


def case_pack_file():
    """A reference-written .rwpk file + what the reference loads from it."""
    ph = sw.make_phantom("blobs2d", (12, 10), rng_seed=2, noise_sigma=0.05, num_regions=2)
    pack = sw.precompute(ph.image, 15.0, m=12)
    path = OUT / "small.rwpk"
    sw.save_pack(pack, path)
    loaded = sw.load_pack(path)
    seeds = seeds_of(ph, 3, 4)
    lap = sw.laplacian(sw.build_graph(ph.image, 15.0), LaplacianMode.NORMALIZED)
    prob = sw.LabelProblem(num_labels=2, seeds=seeds, gamma=0.0)
    u = sw.solve_fast(loaded, lap, prob)
    np.savez_compressed(OUT / "pack_file.npz", V=np.asarray(loaded.eigen.vectors), lam=loaded.eigen.values,
                        d_sqrt=loaded.d_sqrt, beta=loaded.beta, dims=np.array(loaded.dims),
                        intensities=ph.image.intensities, image_hash=np.frombuffer(loaded.provenance.image_hash,
                                                                                    dtype=np.uint8),
                        seeds_idx=seeds.seed_indices, seeds_lab=seeds.seed_labels, U=u.values,
                        xxh_empty=sw.xxh64(b""), xxh_a=sw.xxh64(b"a"))


def case_registration():
    """Reference similarity_priors + a full registration-style solve."""
    from specwalk.registration import DisplacementGrid, expected_displacement, similarity_priors
    out = {}
    ph = sw.make_phantom("shifted_pair", (14, 12), rng_seed=4, noise_sigma=0.02, num_regions=2, shift=(1, 0))
    grid = DisplacementGrid((3, 3))
    pri = similarity_priors(ph.image, ph.moving, grid, patch_radius=1)
    out.update(f2=ph.image.intensities, m2=ph.moving.intensities, dims2=np.array(ph.image.dims),
               pri2=pri.values, vec2=grid.vectors())
    ph3 = sw.make_phantom("shifted_pair", (8, 7, 6), rng_seed=5, noise_sigma=0.02, num_regions=2, shift=(1, 0, 0))
    grid3 = DisplacementGrid((3, 3, 3))
    pri3 = similarity_priors(ph3.image, ph3.moving, grid3, patch_radius=1)
    out.update(f3=ph3.image.intensities, m3=ph3.moving.intensities, dims3=np.array(ph3.image.dims),
               pri3=pri3.values, vec3=grid3.vectors())
    # solve with the priors on an eigen pack and read out the displacement
    pack = sw.precompute(ph3.image, 50.0, m=60)
    lap = sw.laplacian(sw.build_graph(ph3.image, 50.0), LaplacianMode.NORMALIZED)
    n = ph3.image.n_voxels
    prob = sw.LabelProblem(num_labels=grid3.K, seeds=sw.SeedPartition(n, [], []), priors=pri3.values, gamma=1.0)
    u = sw.solve_fast(pack, lap, prob, m_use=50)
    disp = expected_displacement(u, grid3)
    out.update(V3=np.asarray(pack.eigen.vectors), lam3=pack.eigen.values, d3=pack.d_sqrt, U3=u.values,
               disp3=disp.vectors)
    csr_parts("lap3", lap.matrix, out)
    np.savez_compressed(OUT / "registration.npz", **out)


def case_aggregation():
    """Reference super-vertex aggregation (aggregation.py:89-216): clusters,
    delta weights, coarsened bases (both variants), aggregate Laplacian,
    aggregate priors, the coarse solve and the propagated field."""
    from specwalk.aggregation import (CoarsenVariant, aggregate_priors, build_aggregation,
                                      coarsen_basis, delta_weights, propagate)
    from specwalk.registration import DisplacementGrid, similarity_priors
    out = {}
    for tag, dims, shift, grid_ext, radius, tol, beta, m, m_use in (
            ("2", (20, 18), (1, 0), (3, 3), 2, 0.35, 30.0, 40, 30),
            ("3", (9, 8, 7), (1, 0, 0), (3, 3, 3), 1, 0.5, 20.0, 36, 30)):
        ph = sw.make_phantom("shifted_pair", dims, rng_seed=7, noise_sigma=0.02, num_regions=2, shift=shift)
        grid = DisplacementGrid(grid_ext)
        pri = similarity_priors(ph.image, ph.moving, grid, patch_radius=1)
        pack = sw.precompute(ph.image, beta, m=m)
        agg = build_aggregation(pri, max_cluster_radius=radius, similarity_tol=tol)
        graph = sw.build_graph(ph.image, beta=pack.beta)
        out.update({f"img{tag}": ph.image.intensities, f"mov{tag}": ph.moving.intensities,
                    f"dims{tag}": np.array(dims), f"pri{tag}": pri.values, f"V{tag}": np.asarray(pack.eigen.vectors),
                    f"lam{tag}": pack.eigen.values, f"dsq{tag}": pack.d_sqrt, f"beta{tag}": beta,
                    f"cid{tag}": agg.cluster_ids, f"nsup{tag}": agg.n_super, f"radius{tag}": radius,
                    f"tol{tag}": tol, f"muse{tag}": m_use, f"delta{tag}": delta_weights(agg, graph)})
        for var in (CoarsenVariant.DELTA, CoarsenVariant.NAIVE):
            v = var.value[0]
            basis, pbar = coarsen_basis(pack, agg, graph, var, m_use=m_use)
            out[f"q{v}{tag}"] = basis.q_bar
            out[f"lb{v}{tag}"] = basis.lambda_bar
            out[f"dsqbar{v}{tag}"] = pbar.d_sqrt
            csr_parts(f"lapbar{v}{tag}", pbar.laplacian.matrix, out)
        p_bar = aggregate_priors(pri.values, agg)
        p_bar /= p_bar.sum(axis=1, keepdims=True)
        _, pbar = coarsen_basis(pack, agg, graph, CoarsenVariant.DELTA, m_use=m_use)
        prob = sw.LabelProblem(num_labels=grid.K, seeds=sw.SeedPartition(agg.n_super, [], []), priors=p_bar,
                               gamma=1.0)
        u_bar = sw.solve_fast(pbar, pbar.laplacian, prob, m_use=pbar.m)
        u = propagate(u_bar.values, agg)
        out.update({f"pbar{tag}": p_bar, f"ubar{tag}": u_bar.values, f"u{tag}": u.values})
    np.savez_compressed(OUT / "aggregation.npz", **out)


if __name__ == "__main__":
    case_path3()
    case_phantom16()
    case_blobs3d()
    case_modes()
    case_adaptive_kats()
    case_errors()
    case_pack_file()
    case_registration()
    case_aggregation()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
