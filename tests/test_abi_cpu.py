"""CPU-side checks of the C ABI: the library loads without a GPU and exports
every symbol declared in include/specwalk_b200.h (no compute calls)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_1607_04174_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "specwalk_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(swb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.library_path()))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_table_matches_header():
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_status_strings_match_reference_taxonomy():
    lib = _lib.load()
    names = {i: lib.swb_status_string(i).decode() for i in range(7)}
    assert names[0] == "ok"
    assert names[1] == "InvalidParam"
    assert names[2] == "InsufficientBasis"
    assert names[3] == "SingularSmallSystem"
    assert names[4] == "DegenerateGraph"
    assert lib.swb_abi_version() == 1


def test_status_maps_to_exceptions():
    from paper_1607_04174_b200 import errors
    with pytest.raises(errors.InvalidParam):
        _lib.check(1)
    with pytest.raises(errors.InsufficientBasis):
        _lib.check(2)
    with pytest.raises(errors.SingularSmallSystem):
        _lib.check(3)
    with pytest.raises(errors.DegenerateGraph):
        _lib.check(4)


def test_host_side_validation_without_device():
    lib = _lib.load()
    lat = _lib.Lattice(4, 4, 1, 5, 0)        # no such neighbourhood
    assert lib.swb_num_directions(ctypes.byref(lat)) == -1
    lat = _lib.Lattice(4, 4, 1, 8, 0)
    assert lib.swb_num_directions(ctypes.byref(lat)) == 4
    lat = _lib.Lattice(4, 4, 4, 6, 1)
    assert lib.swb_num_directions(ctypes.byref(lat)) == 3
    # rcond gate of fastrw.py:340
    assert lib.swb_check_rcond(1e-3) == 0
    assert lib.swb_check_rcond(1e-15) == 3
    assert lib.swb_check_rcond(float("nan")) == 3
    # invalid arguments are rejected before any device work
    assert lib.swb_gemm_nn(None, 0, None, 0, 10, 4, 4, None, 4, 0, None) == 1
    assert lib.swb_update_coeffs(7, None, 0, None, None, None, 4, 0.5, None, 0, None, None, None) == 1


def test_workspace_queries():
    lib = _lib.load()
    assert lib.swb_gemm_tn_workspace_bytes(16_777_216, 400, 400) > 0
    assert lib.swb_small_solve_workspace_bytes(800, 400, 4) > 801 * 801 * 8
    assert lib.swb_lu_workspace_bytes(801) >= 801 * 8


def test_c2_cut_mask_matches_oracle_block_cut():
    """The bench's c2 topology change (workloads.block_cut_voxel_mask) is the
    oracle's block cut (edges with exactly one endpoint inside the block)."""
    import numpy as np
    from oracle import rw_oracle as O
    from paper_1607_04174_b200 import workloads as W
    from paper_1607_04174_b200.device import LatticeSpec
    for conn in (4, 8):
        dims = (23, 19)
        lat = LatticeSpec.make(dims, conn, "sq")
        want = lat.edge_mask_to_voxel_mask(O.block_cut_mask(dims, 5, 3, size=8, connectivity=conn))
        got = W.block_cut_voxel_mask(dims, conn, 5, 3, size=8)
        assert np.array_equal(got, want)


def test_comm_entry_points_without_device():
    """swb_comm_* (csrc/comm.cu): NCCL is dlopen'ed on first use; version and
    unique-id need no GPU; bad arguments are InvalidParam before any NCCL call."""
    lib = _lib.load()
    v = ctypes.c_int()
    rc = lib.swb_comm_nccl_version(ctypes.byref(v))
    if rc == 7:
        pytest.skip(f"NCCL not loadable here: {lib.swb_comm_last_error().decode()}")
    assert rc == 0 and v.value >= 21800
    buf = (ctypes.c_uint8 * 128)()
    assert lib.swb_comm_unique_id(buf) == 0 and any(bytes(buf))
    h = ctypes.c_void_p()
    assert lib.swb_comm_init(buf, 0, 0, ctypes.byref(h)) == 1
    assert lib.swb_comm_init(buf, 2, 2, ctypes.byref(h)) == 1
    assert lib.swb_comm_init(None, 1, 0, ctypes.byref(h)) == 1
    assert lib.swb_comm_allreduce_f64(None, None, None, 4, None) == 1
    assert lib.swb_comm_halo_exchange(None, None, 8, 4, 4, 0, 0, None) == 1
    assert lib.swb_comm_destroy(None) == 0
    assert lib.swb_status_string(7).decode() == "CommError"
