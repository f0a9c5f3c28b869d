"""Registration data term + displacement readout on the GPU (reference
registration.py:27-136) — the c5 caller of the hot path.

  DisplacementGrid       registration.py:27-55 (odd extents, x-fastest labels)
  similarity_priors      registration.py:95-129 -> swb_similarity_priors
  expected_displacement  registration.py:132-136 (U @ grid vectors, DMMA GEMM)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
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
    vec = grid.vectors()
    if vec.shape[1] != nd:
        raise InvalidParam("grid dimensionality does not match the images")
    disp = np.zeros((grid.K, 3), dtype=np.int32)
    disp[:, :nd] = vec
    n = nx * ny * nz
    k = grid.K
    F = torch.from_numpy(np.array(fixed.intensities, dtype=np.float64)).to("cuda")
    M = torch.from_numpy(np.array(moving.intensities, dtype=np.float64)).to("cuda")
    D = torch.from_numpy(disp).to("cuda")
    out = torch.empty((n, k), dtype=torch.float64, device="cuda")
    sigma = torch.empty(1, dtype=torch.float64, device="cuda")
    ws = WORKSPACE.get("priors", _lib.size("swb_similarity_priors_workspace_bytes", n, k))
    _lib.call("swb_similarity_priors", ptr(F), ptr(M), nx, ny, nz, nd, ptr(D), k, int(patch_radius), ptr(out), k,
              ptr(sigma), ptr(ws), ws.numel(), stream_handle())
    return DevicePriors(dims, out, sigma)


def expected_displacement(field, grid: DisplacementGrid) -> np.ndarray:
    """registration.py:132-136: probability-weighted mean displacement (N, d)."""
    torch = require_cuda()
    if field.K != grid.K:
        raise DimsMismatch("probability columns do not match grid labels")
    if hasattr(field, "_u"):                      # DeviceField: U stays in HBM
        U = field._u()
    else:                                         # host ProbabilityField
        U = torch.from_numpy(np.ascontiguousarray(field.values, dtype=np.float64)).to("cuda")
    vec = grid.vectors().astype(np.float64)
    d = vec.shape[1]
    ldb = round_up(d, 2)
    B = torch.zeros((grid.K, ldb), dtype=torch.float64, device="cuda")
    B[:, :d] = torch.from_numpy(vec)
    n = U.shape[0]
    out = torch.empty((n, ldb), dtype=torch.float64, device="cuda")
    Uc = U if U.stride(1) == 1 else U.contiguous()
    _lib.call("swb_gemm_nn", ptr(Uc), Uc.stride(0), ptr(B), ldb, n, grid.K, ldb, ptr(out), ldb, 0, stream_handle())
    return out[:, :d].cpu().numpy()
