"""specwalk-b200: the online hot path of the adaptable-precomputation random
walker (arXiv 1607.04174) rebuilt for NVIDIA B200 (sm_100a).

The public names mirror the reference package ``specwalk`` for the hot path
(refresh / refresh_from_set / solve_fast / select_m / hard_labels and the
data types they take), plus ``update_basis`` (first-order eigenpair update
for beta or topology changes), ``update_and_solve`` (the update and the
solve on the updated basis with the reconstruction folded into the
rotation) and ``segment``.  All numerics run in the
hand-written CUDA library ``libspecwalk_b200.so`` through its C ABI
(include/specwalk_b200.h); there is no CPU fallback.
"""

from .errors import (BackendUnavailable, ChecksumMismatch, DegenerateGraph, DeviceError, DimsMismatch,
                     EmptyBasis, FormatError, ImageMismatch, InsufficientBasis, InvalidParam, IoError,
                     NotConverged, SingularSmallSystem, SingularSystem, SpecwalkError, ZeroVector)
from .types import (AdaptivePolicy, EigenBasis, Image, LabelMap, LabelProblem, LaplacianMode, PackProvenance,
                    PackSet, ProbabilityField, SeedPartition, SpectralPack, SENTINEL_UNLABELED)
from .device import DeviceGraph, DevicePack, LatticeSpec, to_device
from .api import (DeviceField, RefreshedPack, UpdatedPack, evict_device_pack, hard_labels, nearest_pack, refresh,
                  refresh_from_set, segment, select_m, solve_fast, update_and_solve, update_basis)
from .dropin import install
from .capture import CapturedStep
from .packs import load_pack, save_pack, xxh64
from .registration import DevicePriors, DisplacementGrid, expected_displacement, register, similarity_priors
from .precompute import precompute, smallest_eigs_device

__version__ = "0.1.0"


def library_path():
    from ._lib import library_path as _p
    return _p()
