"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference ships no images or packs, so every benchmark
and parity input is generated here from ``np.random.default_rng`` with the
config index as the seed and sub-streams ``[cfg, purpose]``:

  c1  2-D 128^2 disk (r=30, 0.7 on 0.3) + N(0, 0.05^2), 4-conn, (dI)^2
      weights, beta 90 -> 120, M=50, L=2, 20 seeds / label
  c2  2-D 512^2, three disks {0.2, 0.5, 0.8} on 0, 8-conn, beta 60, M=200,
      L=3, 50 seeds / label, cut = edges crossing a 32x32 block boundary
  c3  3-D 128^3 ellipsoid (40/30/25, 0.65 in 0.35) + N(0, 0.08^2), 6-conn,
      beta 100 -> 140, M<=150, L=2, 5 rounds of +100 seeds / label
  c4  3-D 256^3, 4 spheres r~U(20,50), I~U(0.2,0.9) + N(0, 0.05^2), 6-conn,
      beta 80 -> 110, M=400, L=4, 200 seeds / label
  c5  3-D 96^3 registration pair: fixed = trilinear upsampling of 8^3 U(0,1)
      noise; moving = fixed sampled at x + u(x), u a smooth seeded field
      (trilinear 4^3 U(-1,1) per component, scaled to max |u_i| = 3);
      6-conn, reference default |dI| weights, beta 50 -> 70, M=300, 125
      labels (5x5x5 displacement grid, spacing 1), gamma 1, patch radius 2,
      the reference data term (mean |f - m| over the patch; BASELINE's text
      says "SSD", the reference registration.py:95-129 uses the absolute
      difference, which parity follows)
Labels for seeding: the objects (disks / spheres / ellipsoid+background);
voxels outside every object carry label -1 when the config's label count
names only the objects (c2, c4) and are never seeded.

Bases for the 3-D configs are QR-orthonormalised seeded Gaussians with
eigenvalues sorted U(1e-4, 1e-1) (the reference 3-D precompute is infeasible,
SURVEY.md §0.5); they are generated on the GPU (CholeskyQR2 on the DMMA
GEMMs) so the 54 GB c4 basis never touches the host.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

CONFIGS = {
    "c1": dict(dims=(128, 128), connectivity=4, weight_mode="sq", beta0=90.0, beta1=120.0, m=50, labels=2,
               seeds_per_label=20),
    "c2": dict(dims=(512, 512), connectivity=8, weight_mode="sq", beta0=60.0, beta1=60.0, m=200, labels=3,
               seeds_per_label=50, cut_block=32),
    "c3": dict(dims=(128, 128, 128), connectivity=6, weight_mode="sq", beta0=100.0, beta1=140.0, m=150,
               labels=2, seeds_per_label=100, rounds=5, epsilon=1e-3),
    "c4": dict(dims=(256, 256, 256), connectivity=6, weight_mode="sq", beta0=80.0, beta1=110.0, m=400,
               labels=4, seeds_per_label=200),
    "c5": dict(dims=(96, 96, 96), connectivity=6, weight_mode="abs", beta0=50.0, beta1=70.0, m=300, labels=125,
               seeds_per_label=0, grid=(5, 5, 5), gamma=1.0, patch_radius=2, max_disp=3.0),
}
CFG_INDEX = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}


@dataclass
class Workload:
    name: str
    dims: tuple
    intensities: np.ndarray
    truth: np.ndarray          # label per voxel, -1 = never seeded
    params: dict = field(default_factory=dict)


def _grid(dims):
    axes = [np.arange(n, dtype=np.float64) for n in dims]
    return np.meshgrid(*axes, indexing="ij")


def _flat(a):
    return np.asarray(a).reshape(-1, order="F")


def make_image(name: str, dims=None) -> Workload:
    p = dict(CONFIGS[name])
    dims = tuple(dims) if dims is not None else p["dims"]
    rng = np.random.default_rng([CFG_INDEX[name], 0])
    if name == "c1":
        x, y = _grid(dims)
        cx, cy = (dims[0] - 1) / 2, (dims[1] - 1) / 2
        r = 30.0 * min(dims) / 128.0
        inside = (x - cx) ** 2 + (y - cy) ** 2 <= r * r
        img = np.where(inside, 0.7, 0.3) + rng.normal(0, 0.05, dims)
        truth = inside.astype(np.int64)
    elif name == "c2":
        x, y = _grid(dims)
        img = np.zeros(dims)
        truth = -np.ones(dims, dtype=np.int64)
        placed = []
        scale = min(dims) / 512.0
        for k, level in enumerate((0.2, 0.5, 0.8)):
            for _ in range(1000):
                r = rng.uniform(40, 90) * scale
                c = rng.uniform(r, np.array(dims) - r)
                if all(np.hypot(*(c - c2)) > r + r2 + 2 for c2, r2 in placed):
                    break
            placed.append((c, r))
            m = (x - c[0]) ** 2 + (y - c[1]) ** 2 <= r * r
            img[m] = level
            truth[m] = k
        img = img + rng.normal(0, 0.05, dims)
    elif name == "c3":
        x, y, z = _grid(dims)
        c = (np.array(dims) - 1) / 2
        s = np.array([40.0, 30.0, 25.0]) * min(dims) / 128.0
        inside = ((x - c[0]) / s[0]) ** 2 + ((y - c[1]) / s[1]) ** 2 + ((z - c[2]) / s[2]) ** 2 <= 1.0
        img = np.where(inside, 0.65, 0.35) + rng.normal(0, 0.08, dims)
        truth = inside.astype(np.int64)
    elif name == "c4":
        x, y, z = _grid(dims)
        img = np.zeros(dims)
        truth = -np.ones(dims, dtype=np.int64)
        scale = min(dims) / 256.0
        for k in range(4):
            r = rng.uniform(20, 50) * scale
            c = rng.uniform(r, np.array(dims) - r)
            level = rng.uniform(0.2, 0.9)
            m = (x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 <= r * r
            img[m] = level
            truth[m] = k
        img = img + rng.normal(0, 0.05, dims)
    elif name == "c5":
        coarse = rng.uniform(0.0, 1.0, (8, 8, 8))
        img = _upsample(coarse, dims)
        u = np.stack([_upsample(rng.uniform(-1.0, 1.0, (4, 4, 4)), dims) for _ in range(3)], axis=-1)
        u *= p["max_disp"] / max(np.abs(u).max(), 1e-12)
        pts = np.stack(_grid(dims), axis=-1) + u
        moving = _trilinear(coarse, pts, dims)
        p["moving"] = _flat(moving)
        p["true_displacement"] = u.reshape(-1, 3, order="F")
        truth = np.zeros(dims, dtype=np.int64)
    else:
        raise ValueError(name)
    img = np.clip(img, 0.0, 1.0)
    p["dims"] = dims
    return Workload(name, dims, _flat(img), _flat(truth), p)


def _axis_weights(n_fine: int, n_coarse: int) -> np.ndarray:
    """(n_fine, n_coarse) linear-interpolation matrix, corners aligned."""
    t = np.linspace(0.0, n_coarse - 1.0, n_fine)
    i0 = np.minimum(np.floor(t).astype(int), n_coarse - 2)
    f = t - i0
    w = np.zeros((n_fine, n_coarse))
    w[np.arange(n_fine), i0] = 1.0 - f
    w[np.arange(n_fine), i0 + 1] += f
    return w


def _upsample(coarse: np.ndarray, dims) -> np.ndarray:
    """Trilinear upsampling of a coarse 3-D grid onto dims (corners aligned)."""
    a, b, c = (_axis_weights(n, m) for n, m in zip(dims, coarse.shape))
    return np.einsum("ia,jb,kc,abc->ijk", a, b, c, coarse, optimize=True)


def _trilinear(coarse: np.ndarray, pts: np.ndarray, dims) -> np.ndarray:
    """The upsampled field evaluated at continuous fine-grid points (clamped)."""
    out = np.zeros(pts.shape[:-1])
    idx, frac = [], []
    for ax, (n, m) in enumerate(zip(dims, coarse.shape)):
        t = np.clip(pts[..., ax], 0.0, n - 1.0) * (m - 1.0) / (n - 1.0)
        i0 = np.minimum(np.floor(t).astype(int), m - 2)
        idx.append(i0)
        frac.append(t - i0)
    for dx in (0, 1):
        for dy in (0, 1):
            for dz in (0, 1):
                w = ((frac[0] if dx else 1 - frac[0]) * (frac[1] if dy else 1 - frac[1]) *
                     (frac[2] if dz else 1 - frac[2]))
                out += w * coarse[idx[0] + dx, idx[1] + dy, idx[2] + dz]
    return out


def sample_region_seeds(labels: np.ndarray, num_labels: int, per_region: int, rng):
    """Uniform seeds inside each ground-truth region (restates the
    reference bench.py:89-102 sampler: label order, choice w/o replacement)."""
    chosen, chosen_labels = [], []
    for k in range(num_labels):
        region = np.flatnonzero(labels == k)
        if region.size == 0:
            continue
        take = min(per_region, region.size)
        chosen.append(rng.choice(region, size=take, replace=False))
        chosen_labels.append(np.full(take, k))
    idx = np.concatenate(chosen)
    lab = np.concatenate(chosen_labels)
    order = np.argsort(idx, kind="stable")
    return idx[order], lab[order]


def block_cut_voxel_mask(dims, connectivity: int, x0: int, y0: int, size: int = 32) -> np.ndarray:
    """c2's topology change as the API's voxel mask (N x ndir, uint8): the
    forward edge (v, v + d) is cut when exactly one endpoint lies inside the
    block [x0, x0+size) x [y0, y0+size) (2-D; voxels x-fastest, the
    direction order of LatticeSpec.forward_offsets)."""
    nx, ny = dims
    x, y = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    x, y = x.ravel(order="F"), y.ravel(order="F")
    inside = lambda a, b: (a >= x0) & (a < x0 + size) & (b >= y0) & (b < y0 + size)  # noqa: E731
    offs = [(1, 0), (0, 1)] if connectivity == 4 else [(1, 0), (0, 1), (1, 1), (-1, 1)]
    out = np.zeros((nx * ny, len(offs)), dtype=np.uint8)
    for d, (dx, dy) in enumerate(offs):
        xn, yn = x + dx, y + dy
        ok = (xn >= 0) & (xn < nx) & (yn >= 0) & (yn < ny)
        out[:, d] = ok & (inside(x, y) != inside(xn, yn))
    return out


def cut_for(w: Workload):
    """(mask, x0, y0): the seeded block position of a cut-edge config (c2),
    or None."""
    size = w.params.get("cut_block")
    if not size:
        return None
    rng = np.random.default_rng([CFG_INDEX[w.name], 7])
    nx, ny = w.dims
    x0, y0 = int(rng.integers(0, nx - size)), int(rng.integers(0, ny - size))
    return block_cut_voxel_mask(w.dims, w.params["connectivity"], x0, y0, size), x0, y0


def seeds_for(w: Workload, round_index: int = 0):
    rng = np.random.default_rng([CFG_INDEX[w.name], 1, round_index])
    return sample_region_seeds(w.truth, w.params["labels"], w.params["seeds_per_label"], rng)


def synthetic_lambda(name: str, m: int) -> np.ndarray:
    rng = np.random.default_rng([CFG_INDEX[name], 2])
    return np.sort(rng.uniform(1e-4, 1e-1, m))


def orthonormal_basis_device(n: int, m: int, seed: int, ldv: int | None = None):
    """QR-orthonormalised seeded Gaussian N x m on the GPU (row-major, ld
    round_up(m, 8)): CholeskyQR2 with the library's DMMA Gram / NN GEMMs."""
    import torch

    from . import _lib
    from .device import WORKSPACE, ptr, round_up, stream_handle
    ldv = ldv or round_up(m, 8)
    g = torch.Generator(device="cuda")
    g.manual_seed(int(seed))
    V = torch.empty((n, ldv), dtype=torch.float64, device="cuda")
    chunk = 1 << 24
    flat = V.view(-1)
    for s in range(0, flat.numel(), chunk):
        e = min(flat.numel(), s + chunk)
        flat[s:e].normal_(generator=g)
    if ldv > m:
        V[:, m:].zero_()
    W = torch.empty_like(V)
    st = stream_handle()
    ldg = round_up(m, 2)
    for _ in range(2):
        G = torch.zeros((m, ldg), dtype=torch.float64, device="cuda")
        ws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", n, m, m))
        _lib.call("swb_gemm_tn", ptr(V), ldv, ptr(V), ldv, n, m, m, 1, ptr(G), ldg, ptr(ws), ws.numel(), st)
        R = torch.linalg.cholesky(G[:, :m], upper=True)
        Rinv = torch.zeros((m, ldg), dtype=torch.float64, device="cuda")
        Rinv[:, :m] = torch.linalg.solve_triangular(R, torch.eye(m, dtype=torch.float64, device="cuda"),
                                                    upper=True)
        _lib.call("swb_gemm_nn", ptr(V), ldv, ptr(Rinv), ldg, n, m, m, ptr(W), ldv, 0, st)
        if ldv > m:
            W[:, m:].zero_()
        V, W = W, V
    del W
    return V


def orthonormal_basis_slab(plan, m: int, seed: int, comm, ldv: int | None = None):
    """Rows [row_base, row_base + local_rows) of the same global orthonormal
    basis for any rank count: a per-plane seeded Gaussian, orthonormalised by
    a distributed CholeskyQR2 (local DMMA Gram + one all-reduce).  Halo rows
    are left zero (the update's halo exchange fills them)."""
    import torch

    from . import _lib
    from .device import WORKSPACE, ptr, round_up, stream_handle
    ldv = ldv or round_up(m, 8)
    V = torch.zeros((plan.local_rows, ldv), dtype=torch.float64, device="cuda")
    own = V[plan.own_slice()]
    g = torch.Generator(device="cuda")
    for k, u in enumerate(range(plan.u0, plan.u1)):
        g.manual_seed(int(seed) * 1_000_003 + u)
        own[k * plan.unit:(k + 1) * plan.unit, :m].normal_(generator=g)
    rows = plan.own_end - plan.own_begin
    W = torch.zeros_like(own)
    st = stream_handle()
    ldg = round_up(m, 2)
    for _ in range(2):
        G = torch.zeros((m, ldg), dtype=torch.float64, device="cuda")
        ws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", rows, m, m))
        _lib.call("swb_gemm_tn", ptr(own), ldv, ptr(own), ldv, rows, m, m, 1, ptr(G), ldg, ptr(ws), ws.numel(), st)
        comm.allreduce_sum([G])
        R = torch.linalg.cholesky(G[:, :m], upper=True)
        Rinv = torch.zeros((m, ldg), dtype=torch.float64, device="cuda")
        Rinv[:, :m] = torch.linalg.solve_triangular(R, torch.eye(m, dtype=torch.float64, device="cuda"), upper=True)
        _lib.call("swb_gemm_nn", ptr(own), ldv, ptr(Rinv), ldg, rows, m, m, ptr(W), ldv, 0, st)
        own.copy_(W)
    del W
    return V
