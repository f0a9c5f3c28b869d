"""Host-side data types of the reference API, restated for the drop-in.

Field names, validation and defaults follow the reference so that objects
built for ``specwalk`` work here and vice versa (duck typing on the same
attributes):

  Image             images.py:33-73        SeedPartition  graphs.py:51-98
  LabelMap          images.py:76-96        LabelProblem   solver.py:22-52
  ProbabilityField  images.py:99-125       EigenBasis     linalg.py:26-38
  SpectralPack      fastrw.py:126-152      PackSet        fastrw.py:155-177
  AdaptivePolicy    adaptive.py:23-62

These are plain host containers (numpy); the GPU-resident counterparts live
in ``device.py``.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import InvalidParam, SingularSystem

SENTINEL_UNLABELED = 65535
W_MIN = 1e-8
M_CAP = 4096
MAX_SEEDS = 10_000
DEFAULT_EPSILON = 0.1
DEFAULT_STRIDE = 4


class LaplacianMode(Enum):
    UNNORMALIZED = "unnormalized"
    NORMALIZED = "normalized"


def num_voxels(dims) -> int:
    return int(np.prod(dims))


def _frozen(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    a.setflags(write=False)
    return a


@dataclass(frozen=True)
class Image:
    """Scalar intensity grid (2-D or 3-D), flat x-fastest."""

    dims: tuple
    intensities: np.ndarray
    spacing: tuple = ()
    intensity_range: tuple = (0.0, 1.0)

    def __post_init__(self):
        dims = tuple(int(n) for n in self.dims)
        if len(dims) not in (2, 3) or any(n <= 0 for n in dims):
            raise InvalidParam(f"dims must be 2 or 3 positive extents, got {dims}")
        spacing = tuple(float(s) for s in self.spacing) if self.spacing else (1.0,) * len(dims)
        if len(spacing) != len(dims):
            raise InvalidParam("spacing length must match dims")
        vals = np.asarray(self.intensities, dtype=np.float64).ravel()
        if vals.size != num_voxels(dims):
            raise InvalidParam(f"expected {num_voxels(dims)} intensities, got {vals.size}")
        if not np.all(np.isfinite(vals)):
            raise InvalidParam("intensities must be finite")
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "spacing", spacing)
        object.__setattr__(self, "intensities", _frozen(vals))

    @property
    def n_voxels(self) -> int:
        return self.intensities.size

    @property
    def ndim(self) -> int:
        return len(self.dims)

    def content_hash(self) -> bytes:
        return content_hash(self)


def content_hash(image) -> bytes:
    """images.py:66-73: sha256 of rank, dims, spacing and f32 intensities."""
    h = hashlib.sha256()
    h.update(struct.pack("<B", len(image.dims)))
    h.update(np.asarray(image.dims, dtype="<u8").tobytes())
    h.update(np.asarray(image.spacing, dtype="<f8").tobytes())
    h.update(np.asarray(image.intensities).astype("<f4").tobytes())
    return h.digest()


@dataclass(frozen=True)
class LabelMap:
    dims: tuple
    labels: np.ndarray

    def __post_init__(self):
        dims = tuple(int(n) for n in self.dims)
        lab = np.asarray(self.labels).astype(np.int64, copy=False).ravel()
        if lab.size != num_voxels(dims):
            raise InvalidParam("label count does not match dims")
        if np.any(lab < 0):
            raise InvalidParam("labels must be non-negative")
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "labels", _frozen(lab))

    def num_labels(self) -> int:
        real = self.labels[self.labels != SENTINEL_UNLABELED]
        return int(real.max()) + 1 if real.size else 0


@dataclass(frozen=True)
class ProbabilityField:
    """Row-stochastic N x K label probabilities (validated as images.py:106-117)."""

    dims: tuple
    values: np.ndarray

    def __post_init__(self):
        dims = tuple(int(n) for n in self.dims)
        vals = np.asarray(self.values, dtype=np.float64)
        if vals.ndim != 2 or vals.shape[0] != num_voxels(dims):
            raise InvalidParam(f"values must be (N, K) with N={num_voxels(dims)}")
        if not np.allclose(vals.sum(axis=1), 1.0, atol=1e-6):
            raise InvalidParam("rows must sum to 1 within 1e-6")
        if vals.size and (vals.min() < -1e-6 or vals.max() > 1 + 1e-6):
            raise InvalidParam("entries must lie in [-1e-6, 1+1e-6]")
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "values", _frozen(vals))

    @property
    def K(self) -> int:
        return self.values.shape[1]

    def clamped(self) -> np.ndarray:
        return np.clip(self.values, 0.0, 1.0)


@dataclass(frozen=True)
class SeedPartition:
    """Seeded voxels, sorted ascending and unique (graphs.py:51-98)."""

    n_vertices: int
    seed_indices: np.ndarray
    seed_labels: np.ndarray

    def __post_init__(self):
        idx = np.asarray(self.seed_indices, dtype=np.int64).ravel()
        lab = np.asarray(self.seed_labels, dtype=np.int64).ravel()
        if idx.size != lab.size:
            raise InvalidParam("seed_indices and seed_labels must have equal length")
        if idx.size:
            order = np.argsort(idx, kind="stable")
            idx, lab = idx[order], lab[order]
            if idx[0] < 0 or idx[-1] >= self.n_vertices:
                raise IndexError(f"seed index out of range 0..{self.n_vertices - 1}")
            if np.any(np.diff(idx) == 0):
                raise InvalidParam("seed indices must be unique")
            if lab.min() < 0:
                raise InvalidParam("seed labels must be non-negative")
        object.__setattr__(self, "seed_indices", idx)
        object.__setattr__(self, "seed_labels", lab)

    @property
    def n_seeds(self) -> int:
        return self.seed_indices.size

    @property
    def num_labels(self) -> int:
        return int(self.seed_labels.max()) + 1 if self.n_seeds else 0

    def nonseed_indices(self) -> np.ndarray:
        mask = np.ones(self.n_vertices, dtype=bool)
        mask[self.seed_indices] = False
        return np.flatnonzero(mask)

    def one_hot(self, num_labels: int | None = None) -> np.ndarray:
        k = num_labels if num_labels is not None else self.num_labels
        u = np.zeros((self.n_seeds, k))
        u[np.arange(self.n_seeds), self.seed_labels] = 1.0
        return u


@dataclass(frozen=True)
class LabelProblem:
    """Online inputs of one solve (solver.py:22-52)."""

    num_labels: int
    seeds: SeedPartition
    priors: np.ndarray | None = None
    gamma: float = 0.0
    laplacian_mode: LaplacianMode = LaplacianMode.NORMALIZED

    def __post_init__(self):
        if self.gamma < 0:
            raise InvalidParam("gamma must be >= 0")
        if self.gamma == 0 and self.seeds.n_seeds == 0:
            raise SingularSystem("gamma = 0 with no seeds leaves the system singular")
        if self.priors is None:
            if self.gamma != 0:
                raise InvalidParam("gamma > 0 requires priors")
        else:
            p = self.priors
            if not _is_device_array(p):
                p = np.asarray(p, dtype=np.float64)
                if p.ndim != 2 or p.shape[1] != self.num_labels:
                    raise InvalidParam("priors must be (N, K)")
                if not np.allclose(p.sum(axis=1), 1.0, atol=1e-6):
                    raise InvalidParam("prior rows must sum to 1 within 1e-6")
            object.__setattr__(self, "priors", p)
        if self.seeds.n_seeds and self.seeds.seed_labels.max() >= self.num_labels:
            raise InvalidParam("seed label out of range")

    @property
    def K(self) -> int:
        return self.num_labels


def _is_device_array(x) -> bool:
    return type(x).__module__.startswith("torch")


@dataclass(frozen=True)
class EigenBasis:
    vectors: np.ndarray
    values: np.ndarray

    @property
    def m(self) -> int:
        return np.asarray(self.values).size

    def prefix(self, m: int) -> "EigenBasis":
        return EigenBasis(self.vectors[:, :m], self.values[:m])


@dataclass(frozen=True)
class PackProvenance:
    image_hash: bytes
    eig_tol: float | None = None
    built_at: float | None = None


@dataclass(frozen=True)
class SpectralPack:
    """Host spectral pack (fastrw.py:133-152): V column-major N x m."""

    dims: tuple
    spacing: tuple
    beta: float
    eigen: EigenBasis
    d_sqrt: np.ndarray
    provenance: PackProvenance
    neighborhood: str = "lattice"
    laplacian_mode: LaplacianMode = LaplacianMode.NORMALIZED

    @property
    def m(self) -> int:
        return self.eigen.m

    @property
    def n_vertices(self) -> int:
        return np.asarray(self.d_sqrt).size


@dataclass(frozen=True)
class PackSet:
    """Packs for one image at strictly ascending beta (fastrw.py:155-177)."""

    packs: tuple

    def __post_init__(self):
        if not self.packs:
            raise InvalidParam("PackSet needs at least one pack")
        betas = [p.beta for p in self.packs]
        if any(b2 <= b1 for b1, b2 in zip(betas, betas[1:])):
            raise InvalidParam("pack betas must be strictly ascending")
        ref = self.packs[0]
        for p in self.packs[1:]:
            if tuple(p.dims) != tuple(ref.dims):
                raise InvalidParam("packs must share dims")
            if p.provenance.image_hash != ref.provenance.image_hash:
                raise InvalidParam("packs must come from the same image")
        object.__setattr__(self, "packs", tuple(self.packs))

    @property
    def betas(self) -> list:
        return [p.beta for p in self.packs]


@dataclass
class AdaptivePolicy:
    """Thresholds and schedule for the online basis size (adaptive.py:23-62)."""

    epsilon: float = DEFAULT_EPSILON
    stride: int = DEFAULT_STRIDE
    m_start: int | None = None
    m_step: int | None = None
    grid_extents: tuple | None = None

    def __post_init__(self):
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")
        if self.stride < 1:
            raise ValueError("stride must be >= 1")

    def seed_threshold(self, n_seeds: int) -> float:
        return n_seeds * self.epsilon ** 2

    def prior_threshold(self, n_vertices: int) -> float:
        return n_vertices * self.epsilon ** 2

    def schedule(self, pack_m: int, k: int) -> list:
        step = self.m_step if self.m_step is not None else max(1, pack_m // 8)
        start = self.m_start if self.m_start is not None else max(k, pack_m // 8)
        start = min(max(start, k, 1), pack_m)
        out = list(range(start, pack_m + 1, max(1, step)))
        if not out or out[-1] != pack_m:
            out.append(pack_m)
        return out

    def label_subset(self, k: int) -> np.ndarray:
        if self.grid_extents is None or self.stride == 1:
            return np.arange(k)
        coords = [np.arange(0, n, self.stride) for n in self.grid_extents]
        mesh = np.meshgrid(*coords, indexing="ij")
        strides = np.cumprod([1, *self.grid_extents[:-1]])
        flat = sum(c * s for c, s in zip(mesh, strides))
        return np.sort(flat.ravel())
