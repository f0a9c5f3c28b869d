"""Registration data term + displacement readout on the GPU (reference
registration.py:27-136) — the c5 caller of the hot path.

  DisplacementGrid       registration.py:27-55 (odd extents, x-fastest labels)
  similarity_priors      registration.py:95-129 -> swb_similarity_priors
  expected_displacement  registration.py:132-136 (U @ grid vectors, DMMA GEMM)
  register               registration.py:153-229, the pack (fast) branch
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .api import _mark, image_device
from .device import WORKSPACE, ptr, require_cuda, round_up, stream_handle
from .errors import DimsMismatch, InvalidParam
from .types import num_voxels


@dataclass(frozen=True)
class DisplacementGrid:
    extents: tuple
    step: int = 1

    def __post_init__(self):
        extents = tuple(int(e) for e in self.extents)
        if any(e < 1 or e % 2 == 0 for e in extents):
            raise InvalidParam("grid extents must be odd and positive")
        if self.step < 1:
            raise InvalidParam("grid step must be >= 1")
        object.__setattr__(self, "extents", extents)

    @property
    def K(self) -> int:
        return num_voxels(self.extents)

    def vectors(self) -> np.ndarray:
        """(K, d) displacement vectors; label 0 at the most negative corner, x fastest."""
        half = np.array([(e - 1) // 2 for e in self.extents])
        idx = np.arange(self.K)
        out = np.empty((self.K, len(self.extents)), dtype=np.int64)
        rem = idx
        for a, e in enumerate(self.extents):
            out[:, a] = rem % e
            rem = rem // e
        return (out - half) * self.step

    def zero_label(self) -> int:
        return int(np.flatnonzero((self.vectors() == 0).all(axis=1))[0])


class DevicePriors:
    """N x K priors resident on the GPU (ProbabilityField surface on demand)."""

    def __init__(self, dims, values_dev, sigma_dev):
        self.dims = tuple(dims)
        self.values_dev = values_dev
        self.sigma_dev = sigma_dev

    @property
    def K(self) -> int:
        return self.values_dev.shape[1]

    @property
    def values(self) -> np.ndarray:
        return self.values_dev.cpu().numpy()

    @property
    def sigma(self) -> float:
        return float(self.sigma_dev.item())


def similarity_priors(fixed, moving, grid: DisplacementGrid, patch_radius: int = 2) -> DevicePriors:
    """registration.py:95-129 on the GPU."""
    torch = require_cuda()
    if tuple(fixed.dims) != tuple(moving.dims):
        raise DimsMismatch("fixed and moving dims differ")
    if patch_radius < 0:
        raise InvalidParam("patch_radius must be >= 0")
    dims = tuple(int(d) for d in fixed.dims)
    nd = len(dims)
    nx, ny = dims[0], dims[1]
    nz = dims[2] if nd == 3 else 1
    if len(grid.extents) != nd:
        raise InvalidParam("grid dimensionality does not match the images")
    n = nx * ny * nz
    k = grid.K
    _mark("priors")
    F = image_device(fixed)
    M = image_device(moving)
    D = _grid_table(grid, nd)
    out = torch.empty((n, k), dtype=torch.float64, device="cuda")
    sigma = torch.empty(1, dtype=torch.float64, device="cuda")
    ws = WORKSPACE.get("priors", _lib.size("swb_similarity_priors_workspace_bytes", n, k))
    _lib.call("swb_similarity_priors", ptr(F), ptr(M), nx, ny, nz, nd, ptr(D), k, int(patch_radius), ptr(out), k,
              ptr(sigma), ptr(ws), ws.numel(), stream_handle())
    return DevicePriors(dims, out, sigma)


def _grid_table(grid: DisplacementGrid, nd: int):
    """Device int32 (K, 3) displacement table and (K, round_up(d, 2)) f64
    vectors, cached per grid."""
    ent = _GRID_CACHE.get(grid)
    if ent is None:
        torch = require_cuda()
        vec = grid.vectors()
        disp = np.zeros((grid.K, 3), dtype=np.int32)
        disp[:, :nd] = vec
        B = np.zeros((grid.K, round_up(nd, 2)))
        B[:, :nd] = vec
        ent = (torch.from_numpy(disp).to("cuda"), torch.from_numpy(B).to("cuda"))
        _GRID_CACHE[grid] = ent
    return ent[0]


_GRID_CACHE: dict = {}


def expected_displacement_device(field, grid: DisplacementGrid):
    """U @ vectors on the DMMA NN GEMM; (N, round_up(d, 2)) device tensor,
    columns >= d zero."""
    torch = require_cuda()
    if field.K != grid.K:
        raise DimsMismatch("probability columns do not match grid labels")
    if hasattr(field, "_u"):                      # DeviceField: U stays in HBM
        U = field._u()
    else:                                         # host ProbabilityField
        U = torch.from_numpy(np.ascontiguousarray(field.values, dtype=np.float64)).to("cuda")
    _mark("displacement")
    d = len(grid.extents)
    _grid_table(grid, d)
    B = _GRID_CACHE[grid][1]
    ldb = B.shape[1]
    n = U.shape[0]
    out = torch.empty((n, ldb), dtype=torch.float64, device="cuda")
    Uc = U if U.stride(1) == 1 else U.contiguous()
    _lib.call("swb_gemm_nn", ptr(Uc), Uc.stride(0), ptr(B), ldb, n, grid.K, ldb, ptr(out), ldb, 0, stream_handle())
    return out


def expected_displacement(field, grid: DisplacementGrid) -> np.ndarray:
    """registration.py:132-136: probability-weighted mean displacement (N, d)."""
    return expected_displacement_device(field, grid)[:, :len(grid.extents)].cpu().numpy()


@dataclass
class RegisterReport:
    """registration.py:58-82 (the fields the fast branch fills)."""
    method: str = "fast"
    m_use: int = 0
    adaptive_saturated: bool = False
    priors_s: float = 0.0
    solve_s: float = 0.0
    aggregate_s: float = 0.0
    n_super: int = 0


def _lift_seeds(seeds, agg):
    """registration.py:232-246: landmark voxels -> their super-vertices."""
    from .errors import InvalidParam as _IP
    from .types import SeedPartition
    if seeds.n_seeds == 0:
        return SeedPartition(agg.n_super, [], [])
    super_ids = agg.cluster_ids[seeds.seed_indices]
    uniq, first = np.unique(super_ids, return_index=True)
    labels = seeds.seed_labels[first]
    clash = {}
    for sid, lab in zip(super_ids, seeds.seed_labels):
        if clash.setdefault(sid, lab) != lab:
            raise _IP("conflicting landmark labels inside one super-vertex")
    return SeedPartition(agg.n_super, uniq, labels)


def register(fixed, moving, pack, grid: DisplacementGrid | None = None, gamma: float = 1.0,
             patch_radius: int = 2, adaptive: bool = False, aggregate=None, m_use: int | None = None,
             coarsen_variant=None, landmarks=None, policy=None):
    """registration.py:153-229 with a pack: priors -> (aggregation) ->
    (select_m) -> solve_fast -> expected displacement, on the GPU.  The
    basic (no pack) branch is outside the hot path."""
    import time
    from dataclasses import replace

    from .aggregation import CoarsenVariant, aggregate_priors, build_aggregation, coarsen_basis, propagate
    from .api import select_m, solve_fast
    from .types import AdaptivePolicy, LabelProblem, LaplacianMode, SeedPartition
    if pack is None:
        raise InvalidParam("register() on the GPU needs a spectral pack (the basic solver is out of scope)")
    if grid is None:
        grid = DisplacementGrid((7,) * len(fixed.dims))
    if coarsen_variant is None:
        coarsen_variant = CoarsenVariant.DELTA
    rep = RegisterReport()
    t0 = time.perf_counter()
    pri = similarity_priors(fixed, moving, grid, patch_radius)
    rep.priors_s = time.perf_counter() - t0
    n = num_voxels(fixed.dims)
    seeds = landmarks if landmarks is not None else SeedPartition(n, [], [])
    prob = LabelProblem(num_labels=grid.K, seeds=seeds, priors=pri.values_dev, gamma=gamma,
                        laplacian_mode=LaplacianMode.NORMALIZED)
    policy = replace(policy, grid_extents=grid.extents) if policy is not None else \
        AdaptivePolicy(grid_extents=grid.extents)
    t0 = time.perf_counter()
    if aggregate is not None:
        similarity_tol, radius = aggregate
        t_agg = time.perf_counter()
        agg = build_aggregation(pri, max_cluster_radius=radius, similarity_tol=similarity_tol)
        _, pack_bar = coarsen_basis(pack, agg, None, coarsen_variant, m_use=m_use, image=fixed)
        rep.aggregate_s = time.perf_counter() - t_agg
        rep.n_super = agg.n_super
        p_bar = aggregate_priors(pri, agg)
        p_bar = p_bar / p_bar.sum(dim=1, keepdim=True)
        if agg.n_super == 1:
            u = propagate(p_bar, agg)
            rep.m_use = pack_bar.m
        else:
            prob_bar = LabelProblem(num_labels=grid.K, seeds=_lift_seeds(seeds, agg), priors=p_bar.contiguous(),
                                    gamma=gamma, laplacian_mode=LaplacianMode.NORMALIZED)
            mb = pack_bar.m
            if adaptive:
                mb, info = select_m(pack_bar, prob_bar, policy)
                rep.adaptive_saturated = info["saturated"]
            u_bar = solve_fast(pack_bar, pack_bar.laplacian, prob_bar, m_use=mb, want_field=True)
            rep.m_use = mb
            u = propagate(u_bar, agg)
        rep.method = f"aggregate-{coarsen_variant.value}"
    else:
        lap = getattr(pack, "laplacian", None)
        chosen = m_use if m_use is not None else pack.m
        if adaptive:
            chosen, info = select_m(pack, prob, policy)
            rep.adaptive_saturated = info["saturated"]
        if lap is None:
            from .device import DeviceGraph, LatticeSpec
            lap = DeviceGraph.build(image_device(fixed), LatticeSpec.make(tuple(fixed.dims)), float(pack.beta))
        u = solve_fast(pack, lap, prob, m_use=chosen, want_field=True)
        rep.m_use = chosen
        rep.method = "fast"
    rep.solve_s = time.perf_counter() - t0
    return u, expected_displacement(u, grid), rep
