"""`.rwpk` ingest: native XXH64 (CPU) and GPU load / save against a pack
file written by the unmodified reference (tests/golden/small.rwpk)."""

import numpy as np
import pytest

from conftest import GOLDEN, load_golden


def test_xxh64_reference_vectors():
    from paper_1607_04174_b200.packs import xxh64
    # reference tests/test_fastrw.py:21-25
    assert xxh64(b"") == 0xEF46DB3751D8E999
    assert xxh64(b"a") == 0xD24EC4F1A98C6E5B
    z = load_golden("pack_file")
    assert xxh64(b"") == int(z["xxh_empty"]) and xxh64(b"a") == int(z["xxh_a"])
    data = bytes(range(256)) * 37
    import ctypes as C
    from paper_1607_04174_b200 import _lib
    lib = _lib.load()
    st = C.create_string_buffer(lib.swb_xxh64_state_bytes())
    lib.swb_xxh64_init(st, 0)
    for a, b in ((0, 5), (5, 100), (100, 131), (131, len(data))):
        lib.swb_xxh64_update(st, data[a:b], b - a)
    assert lib.swb_xxh64_digest(st) == xxh64(data)


def test_pack_file_checksum_matches_native():
    import struct
    from paper_1607_04174_b200.packs import xxh64
    raw = (GOLDEN / "small.rwpk").read_bytes()
    body = raw[:-40]
    assert xxh64(body) == struct.unpack("<Q", raw[-40:-32])[0]


@pytest.mark.gpu
def test_load_pack_to_device_matches_reference(cuda_ok, tmp_path):
    import paper_1607_04174_b200 as swb
    from oracle import rw_oracle as O
    z = load_golden("pack_file")
    dp = swb.load_pack(GOLDEN / "small.rwpk")
    assert dp.dims == tuple(z["dims"]) and dp.beta == float(z["beta"]) and dp.m == z["lam"].size
    np.testing.assert_array_equal(dp.V[:, :dp.m].cpu().numpy(), z["V"])
    np.testing.assert_array_equal(dp.values, z["lam"])
    np.testing.assert_array_equal(dp.d_sqrt, z["d_sqrt"])
    assert dp.provenance.image_hash == z["image_hash"].tobytes()
    out = tmp_path / "resaved.rwpk"
    swb.save_pack(dp, out)
    assert out.read_bytes() == (GOLDEN / "small.rwpk").read_bytes()
    lap = O.build_laplacian(z["intensities"], tuple(z["dims"]), float(z["beta"]))
    prob = swb.LabelProblem(num_labels=2, seeds=swb.SeedPartition(z["d_sqrt"].size, z["seeds_idx"], z["seeds_lab"]))
    f = swb.solve_fast(dp, lap, prob, want_field=True)
    np.testing.assert_allclose(f.values, z["U"], atol=1e-10)


@pytest.mark.gpu
def test_load_pack_errors(cuda_ok, tmp_path):
    import paper_1607_04174_b200 as swb
    raw = bytearray((GOLDEN / "small.rwpk").read_bytes())
    bad = bytearray(raw)
    bad[len(bad) - 45] ^= 0x01
    (tmp_path / "bad.rwpk").write_bytes(bytes(bad))
    with pytest.raises(swb.ChecksumMismatch):
        swb.load_pack(tmp_path / "bad.rwpk")
    (tmp_path / "magic.rwpk").write_bytes(b"XXXX" + bytes(raw[4:]))
    with pytest.raises(swb.FormatError):
        swb.load_pack(tmp_path / "magic.rwpk")
    (tmp_path / "trunc.rwpk").write_bytes(bytes(raw[: len(raw) // 2]))
    with pytest.raises(swb.FormatError):
        swb.load_pack(tmp_path / "trunc.rwpk")
    with pytest.raises(swb.IoError):
        swb.load_pack(tmp_path / "missing.rwpk")


@pytest.mark.gpu
@pytest.mark.parametrize("beta_online,method,adaptive", [(None, "rayleigh", False), (20.0, "rayleigh", False),
                                                         (20.0, "first_order", True)])
def test_segment_flow(cuda_ok, beta_online, method, adaptive):
    import paper_1607_04174_b200 as swb
    from oracle import rw_oracle as O
    z = load_golden("pack_file")
    image = swb.Image(tuple(z["dims"]), z["intensities"])
    dp = swb.load_pack(GOLDEN / "small.rwpk", image=image)
    seeds = swb.SeedPartition(image.n_voxels, z["seeds_idx"], z["seeds_lab"])
    labels, field, rep = swb.segment(image, [dp], seeds, beta_online=beta_online, method=method,
                                     adaptive=adaptive, want_field=True)
    V, lam = z["V"], z["lam"]
    lap0 = O.build_laplacian(z["intensities"], tuple(z["dims"]), float(z["beta"]))
    if beta_online is None:
        Vu, lu, lap, dsq = V, lam, lap0, z["d_sqrt"]
    elif method == "rayleigh":
        lap = O.build_laplacian(z["intensities"], tuple(z["dims"]), beta_online)
        lu, order = O.refresh(V, lap)
        Vu, dsq = V[:, order], lap.d_sqrt
    else:
        lap = O.build_laplacian(z["intensities"], tuple(z["dims"]), beta_online)
        Vu, lu, _, _, _ = O.first_order_update(V, lam, lap0, lap)
        dsq = lap.d_sqrt
    m = rep["m_use"]
    if adaptive:
        m_o, _ = O.select_m(Vu, dsq, z["seeds_idx"], z["seeds_lab"], 2)
        assert m == m_o
    u = O.solve_fast(Vu, lu, dsq, lap.matrix, z["seeds_idx"], z["seeds_lab"], 2, m_use=m)
    np.testing.assert_allclose(field.values, u, atol=1e-9)
    assert rep["refreshed"] == (beta_online is not None)


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [4096, 3 * 4 * 144 + 7, 1 << 30])
def test_streamed_load_and_save_multi_block(cuda_ok, tmp_path, monkeypatch, chunk):
    """Ingest / save stream the payload in column blocks through pinned
    staging buffers (staging.py); with tiny blocks (one column, a ragged
    three-column block, one block) the loaded basis and the re-saved bytes
    are identical to the reference-written file."""
    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200 import staging
    monkeypatch.setattr(staging, "CHUNK_BYTES", chunk)
    z = load_golden("pack_file")
    dp = swb.load_pack(GOLDEN / "small.rwpk")
    np.testing.assert_array_equal(dp.V[:, :dp.m].cpu().numpy(), z["V"])
    out = tmp_path / "resaved.rwpk"
    swb.save_pack(dp, out)
    assert out.read_bytes() == (GOLDEN / "small.rwpk").read_bytes()


@pytest.mark.gpu
def test_streamed_load_detects_corrupt_payload(cuda_ok, tmp_path, monkeypatch):
    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200 import staging
    monkeypatch.setattr(staging, "CHUNK_BYTES", 4096)
    raw = bytearray((GOLDEN / "small.rwpk").read_bytes())
    raw[-40 - 1000] ^= 0x10                     # one bit inside the eigenvector block
    bad = tmp_path / "bad.rwpk"
    bad.write_bytes(bytes(raw))
    with pytest.raises(swb.ChecksumMismatch):
        swb.load_pack(bad)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_upload_basis_streams_column_major_blocks(cuda_ok, monkeypatch, dtype):
    from paper_1607_04174_b200 import staging
    from paper_1607_04174_b200.device import upload_basis
    monkeypatch.setattr(staging, "CHUNK_BYTES", 5000)
    rng = np.random.default_rng(1)
    V = np.asfortranarray(rng.standard_normal((777, 37)).astype(dtype))
    got = upload_basis(V, 33).cpu().numpy()
    assert got.shape == (777, 40)
    np.testing.assert_array_equal(got[:, :33], V[:, :33].astype(np.float64))
    assert not got[:, 33:].any()
