"""ctypes binding of libspecwalk_b200.so (the C ABI in include/specwalk_b200.h).

The shared library is built in-tree by ``build_ext.py`` (nvcc, sm_100a).  The
product path has no fallback: if the library or a CUDA device is missing the
calls raise instead of computing anything on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import errors

# SWB_LIB: load another build of the library (A/B measurement of compile-time
# variants, tools/build_variant.py); default the in-tree build
_LIB_PATH = Path(os.environ.get("SWB_LIB") or Path(__file__).resolve().parent / "libspecwalk_b200.so")

c_i64 = C.c_int64
c_i32 = C.c_int32
c_dbl = C.c_double
c_vp = C.c_void_p
c_sz = C.c_size_t


class Lattice(C.Structure):
    """swb_lattice (include/specwalk_b200.h)."""

    _fields_ = [("nx", c_i64), ("ny", c_i64), ("nz", c_i64),
                ("connectivity", c_i32), ("weight_mode", c_i32)]


# name -> (restype, argtypes)
SIGNATURES = {
    "swb_abi_version": (C.c_int, []),
    "swb_status_string": (C.c_char_p, [C.c_int]),
    "swb_last_cuda_error": (C.c_char_p, []),
    "swb_launch_count": (C.c_ulonglong, []),
    "swb_comm_last_error": (C.c_char_p, []),
    "swb_comm_nccl_version": (C.c_int, [C.POINTER(C.c_int)]),
    "swb_comm_unique_id": (C.c_int, [c_vp]),
    "swb_comm_init": (C.c_int, [c_vp, C.c_int, C.c_int, C.POINTER(c_vp)]),
    "swb_comm_destroy": (C.c_int, [c_vp]),
    "swb_comm_rank": (C.c_int, [c_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "swb_comm_allreduce_f64": (C.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "swb_comm_halo_exchange": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_i64, C.c_int, C.c_int, c_vp]),
    "swb_num_directions": (C.c_int, [C.POINTER(Lattice)]),
    "swb_graph_build": (C.c_int, [C.POINTER(Lattice), c_vp, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "swb_stencil_workspace_bytes": (c_sz, [C.POINTER(Lattice), c_i64]),
    "swb_stencil_rayleigh": (C.c_int, [C.POINTER(Lattice), c_vp, c_i64, c_i64, c_i64, c_i64, c_i64,
                                       c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "swb_stencil_delta": (C.c_int, [C.POINTER(Lattice), c_vp, c_i64, c_i64, c_i64, c_i64, c_i64,
                                    c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp,
                                    c_vp, c_sz, c_vp]),
    "swb_stencil_apply": (C.c_int, [C.POINTER(Lattice), c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp,
                                    c_vp, c_dbl, c_dbl, c_vp, c_i64, c_dbl, c_vp, c_i64, c_vp, c_vp, c_vp,
                                    c_sz, c_vp]),
    "swb_column_workspace_bytes": (c_sz, [c_i64]),
    "swb_ritz_residuals": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "swb_column_dots": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "swb_column_update": (C.c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "swb_column_products": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "swb_build_aggregation": (C.c_int, [c_vp, c_i64, c_i64, c_vp, c_i32, c_i32, c_dbl, c_vp, c_vp]),
    "swb_delta_weights": (C.c_int, [C.POINTER(Lattice), c_vp, c_vp, c_vp]),
    "swb_cluster_rows": (C.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "swb_csr_spmm": (C.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "swb_edge_weights": (C.c_int, [C.POINTER(Lattice), c_vp, c_dbl, c_vp, c_vp, c_vp]),
    "swb_canonical_signs": (C.c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_sz, c_vp]),
    "swb_update_workspace_bytes": (c_sz, [C.POINTER(Lattice), c_i64]),
    "swb_update_first_order": (C.c_int, [C.POINTER(Lattice), c_vp, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64,
                                         c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "swb_update_and_solve_workspace_bytes": (c_sz, [C.POINTER(Lattice), c_i64, c_i64, c_i64, c_i64, c_i64]),
    "swb_update_and_solve": (C.c_int, [C.POINTER(Lattice), c_vp, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64,
                                       c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp,
                                       c_vp, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "swb_oz_gemm_nn_split": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64,
                                       c_vp, C.c_size_t, c_vp]),
    "swb_rw_solve_workspace_bytes": (c_sz, [C.POINTER(Lattice), c_i64, c_i64, c_i64, c_i64, C.c_int]),
    "swb_rw_solve": (C.c_int, [C.POINTER(Lattice), c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp,
                               c_vp, c_i64, c_i64, c_dbl, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_sz,
                               c_vp]),
    "swb_gemm_tn_workspace_bytes": (c_sz, [c_i64, c_i64, c_i64]),
    "swb_gemm_tn": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, C.c_int, c_vp, c_i64,
                              c_vp, c_sz, c_vp]),
    "swb_gemm_nn": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, C.c_int, c_vp]),
    "swb_gemm_nn_ex": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, C.c_int, c_dbl,
                                 c_vp]),
    "swb_oz_gemm_nn_workspace_bytes": (C.c_size_t, [c_i64, c_i64, c_i64]),
    "swb_oz_gemm_nn": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, C.c_size_t,
                                 c_vp]),
    "swb_oz_split_cols": (C.c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, C.c_size_t, c_vp]),
    "swb_oz_split_rows": (C.c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, C.c_int, c_vp, C.c_size_t, c_vp]),
    "swb_oz_gemm_planes": (C.c_int, [c_i64, c_i64, c_i64, c_i64, C.c_int, c_vp, c_i64, c_vp, C.c_size_t, c_vp]),
    "swb_oz_gemm_planes_ex": (C.c_int, [c_i64, c_i64, c_i64, c_i64, C.c_int, c_vp, c_i64, c_i64, c_vp, c_i64,
                                        c_vp, c_vp, C.c_size_t, c_vp]),
    "swb_oz_gemm_nn_workspace_bytes_full": (C.c_size_t, [c_i64, c_i64, c_i64]),
    "swb_oz_layout_info": (C.c_int, [c_i64, c_i64, c_i64, c_vp]),
    "swb_gemm_tn_sym_emit": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_sz, c_vp, c_i64,
                                       c_vp, c_sz, c_vp]),
    "swb_small_dense_solve": (C.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "swb_ell_rows_gather": (C.c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "swb_ell_rows_scatter": (C.c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "swb_build_caug": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "swb_oz_gemm_planes_split": (C.c_int, [c_i64, c_i64, c_i64, c_i64, C.c_int, c_vp, c_i64, c_i64, c_vp, c_i64,
                                           c_vp, C.c_size_t, c_vp]),
    "swb_finalize_label": (C.c_int, [c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_dbl, c_vp, c_vp, c_i64, c_vp, c_vp,
                                     c_vp]),
    "swb_oz_chunk_rows": (c_i64, [c_i64, c_i64, c_i64]),
    "swb_int8_peak_probe": (C.c_int, [C.c_int, C.POINTER(C.c_double), c_vp]),
    "swb_int8_scheme_probe": (C.c_int, [C.c_int, C.POINTER(C.c_double), c_vp]),
    "swb_int8_probe_ex": (C.c_int, [C.c_int, C.c_int, C.c_uint, C.POINTER(C.c_double), c_vp]),
    "swb_oz_gemm_nn_raw": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, C.c_size_t,
                                     c_vp]),
    "swb_update_coeffs": (C.c_int, [C.c_int, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_dbl, c_vp, c_i64,
                                    c_vp, c_vp, c_vp]),
    "swb_seed_rows": (C.c_int, [C.POINTER(Lattice), c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "swb_seed_project": (C.c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64,
                                   c_vp, c_vp, c_i64, c_vp, c_dbl, c_i64, c_vp, c_i64, c_vp, c_vp,
                                   c_vp, c_vp, c_vp]),
    "swb_gecon_wb_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "swb_gecon_wb": (C.c_int, [c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "swb_norm1": (C.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "swb_check_seeds": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "swb_small_solve_workspace_bytes": (c_sz, [c_i64, c_i64, c_i64]),
    "swb_small_solve": (C.c_int, [c_dbl, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp,
                                  c_dbl, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_sz,
                                  c_vp]),
    "swb_small_solve_ex": (C.c_int, [c_dbl, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp,
                                     c_dbl, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_sz,
                                     c_vp, c_vp, c_vp]),
    "swb_check_rcond": (C.c_int, [c_dbl]),
    "swb_lu_workspace_bytes": (c_sz, [c_i64]),
    "swb_lu_factor": (C.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "swb_lu_rcond": (C.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "swb_lu_solve_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "swb_lu_solve": (C.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_sz, c_vp]),
    "swb_reconstruct_label": (C.c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_dbl,
                                        c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "swb_gather_rows": (C.c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "swb_scatter_rows": (C.c_int, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "swb_apply_seeds": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp,
                                  c_vp]),
    "swb_seed_fit_workspace_bytes": (c_sz, [c_i64, c_i64, c_i64, c_i64]),
    "swb_seed_fit_schedule": (C.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64,
                                        c_i32, c_dbl, c_vp, c_vp, c_sz, c_vp]),
    "swb_prior_hat": (C.c_int, [c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "swb_argmax_rows": (C.c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "swb_fp64_peak_probe": (C.c_int, [C.c_int, c_vp, C.POINTER(c_dbl), c_vp]),
    "swb_xxh64_state_bytes": (c_sz, []),
    "swb_xxh64_init": (None, [c_vp, C.c_uint64]),
    "swb_xxh64_update": (None, [c_vp, c_vp, c_sz]),
    "swb_xxh64_digest": (C.c_uint64, [c_vp]),
    "swb_f32_colmajor_to_f64_rowmajor": (C.c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "swb_f64_colmajor_to_f64_rowmajor": (C.c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp]),
    "swb_f64_rowmajor_to_f32_colmajor": (C.c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "swb_similarity_priors_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "swb_similarity_priors": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_i64, c_i32, c_vp, c_i64, c_i32, c_vp, c_i64,
                                        c_vp, c_vp, c_sz, c_vp]),
    "swb_sumsq": (C.c_int, [c_vp, c_i64, c_vp, c_vp, c_sz, c_vp]),
    "swb_gather_columns": (C.c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp]),
}

_lib = None


def library_path() -> Path:
    return _LIB_PATH


def load() -> C.CDLL:
    """Load (once) and type the shared library.  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise errors.BackendUnavailable(
            f"{_LIB_PATH.name} is not built; run `python -m paper_1607_04174_b200.build_ext`"
            " (there is no CPU fallback)")
    lib = C.CDLL(str(_LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str = "") -> None:
    """Map an ABI status onto the reference exception taxonomy."""
    if status == 0:
        return
    lib = load()
    name = lib.swb_status_string(status).decode()
    msg = f"{what}: {name}" if what else name
    if status == 5:
        msg += f" ({lib.swb_last_cuda_error().decode()})"
    elif status == 7:
        msg += f" ({lib.swb_comm_last_error().decode()})"
    raise errors.from_status(status, msg)


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)


def size(name: str, *args) -> int:
    return int(getattr(load(), name)(*args))
