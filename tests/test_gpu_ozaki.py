"""The FP64 GEMM on INT8 tensor cores (csrc/ozaki.cu): the int32 digit-product
group sums are checked exactly against a numpy restatement of the digit
split, and the FP64 result against numpy's matmul within the scheme's error
bound 2^-50 * K * max|A[r,:]| * max|B[:,c]| (the FP64 GEMM bound with row /
column maxima)."""

import numpy as np
import pytest

from paper_1607_04174_b200 import _lib

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _ptr(t):
    return t.data_ptr()


def _digits(M, axis):
    """Row (axis=1) or column (axis=0) scaled balanced 7-digit split of
    csrc/ozaki.cu: X = rint(x 2^54), base-256 digits in [-128, 127]."""
    amax = np.abs(M).max(axis=axis, keepdims=True)
    e = np.where(amax > 0, np.frexp(amax)[1], 0)
    e = np.maximum(e, -960)
    X = np.rint(M * np.ldexp(1.0, 54 - e)).astype(np.int64)
    digs = [None] * 7
    for s in range(6, 0, -1):
        d = ((X & 0xFF) ^ 0x80) - 0x80
        digs[s] = d
        X = (X - d) >> 8
    digs[0] = X
    assert np.abs(X).max(initial=0) <= 65
    return digs, e


def _groups(A, B):
    da, _ = _digits(A, 1)
    db, _ = _digits(B, 0)
    return [sum(da[i] @ db[g - i] for i in range(g + 1)) for g in range(7)]


def _run(A, B, raw=False):
    rows, K = A.shape
    M2 = B.shape[1]
    dA = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    dB = torch.from_numpy(np.ascontiguousarray(B)).cuda()
    nbytes = _lib.size("swb_oz_gemm_nn_workspace_bytes", rows, K, M2)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    if raw:
        rows_p = (rows + 127) // 128 * 128
        np_ = (M2 + 63) // 64 * 64  # OZ_BN = 64 column tiles
        r = torch.zeros(7 * rows_p * np_, dtype=torch.int32, device="cuda")
        _lib.call("swb_oz_gemm_nn_raw", _ptr(dA), K, _ptr(dB), M2, rows, K, M2, _ptr(r), _ptr(ws), nbytes, None)
        torch.cuda.synchronize()
        return r.cpu().numpy().reshape(7, rows_p, np_)[:, :rows, :M2]
    ldo = M2 + (M2 & 1)
    out = torch.full((rows, ldo), np.nan, dtype=torch.float64, device="cuda")
    _lib.call("swb_oz_gemm_nn", _ptr(dA), K, _ptr(dB), M2, rows, K, M2, _ptr(out), ldo, _ptr(ws), nbytes, None)
    torch.cuda.synchronize()
    return out.cpu().numpy()[:, :M2]


@pytest.mark.parametrize("rows,K,M2", [(128, 32, 64), (300, 70, 50), (1000, 400, 400)])
def test_group_sums_exact(cuda_ok, rows, K, M2):
    rng = np.random.default_rng(rows + K)
    A = rng.standard_normal((rows, K))
    B = rng.standard_normal((K, M2))
    got = _run(A, B, raw=True)
    want = _groups(A, B)
    for g in range(7):
        assert np.array_equal(got[g], want[g]), f"group {g}"


def _bound(A, B):
    ra = np.abs(A).max(axis=1, keepdims=True)
    cb = np.abs(B).max(axis=0, keepdims=True)
    return 2.0 ** -50 * A.shape[1] * ra * cb


@pytest.mark.parametrize("rows,K,M2", [(1, 1, 1), (129, 33, 65), (5000, 400, 400), (777, 96, 130),
                                       # the digit split's instance boundaries (K <= 256 / <= 448 / <= 512)
                                       (300, 256, 256), (300, 257, 100), (260, 448, 64), (260, 449, 64),
                                       (200, 512, 512)])
def test_fp64_product_within_bound(cuda_ok, rows, K, M2):
    rng = np.random.default_rng(7 * rows + K)
    A = rng.standard_normal((rows, K)) * np.exp(rng.uniform(-3, 3, (rows, 1)))
    B = rng.standard_normal((K, M2)) * np.exp(rng.uniform(-3, 3, (1, M2)))
    got = _run(A, B)
    want = A @ B
    assert np.all(np.abs(got - want) <= _bound(A, B))


def test_rotation_shaped_orthonormal(cuda_ok):
    """The update's shape: orthonormal V (unit columns) times a near-identity
    rotation; error at the FP64 GEMM level."""
    rng = np.random.default_rng(3)
    V, _ = np.linalg.qr(rng.standard_normal((20000, 96)))
    C = np.eye(96) + 1e-2 * rng.standard_normal((96, 96))
    got = _run(V, C)
    want = V @ C
    assert np.abs(got - want).max() < 1e-14
    assert np.all(np.abs(got - want) <= _bound(V, C))


def test_zero_rows_and_columns(cuda_ok):
    A = np.zeros((200, 40))
    A[5] = 1.5
    B = np.zeros((40, 70))
    B[:, 3] = -2.0
    got = _run(A, B)
    assert np.array_equal(got, A @ B)


def test_parts_match_composite_across_chunks(cuda_ok, monkeypatch):
    """device.rotate_rows (split B once, then per row chunk: split A, GEMM)
    equals the one-call swb_oz_gemm_nn, and a ragged last chunk is handled:
    the chunk size is forced small by a row count just over one chunk."""
    from paper_1607_04174_b200.device import rotate_rows
    rng = np.random.default_rng(11)
    rows, K = (1 << 20) + 37, 24
    A = torch.from_numpy(rng.standard_normal((rows, K))).cuda()
    B = torch.from_numpy(np.eye(K) + 0.1 * rng.standard_normal((K, K))).cuda()
    assert _lib.size("swb_oz_chunk_rows", rows, K, K) < rows
    o1 = torch.empty((rows, K), dtype=torch.float64, device="cuda")
    rotate_rows(A, K, B, K, rows, K, o1, K)
    o2 = torch.from_numpy(_run(A.cpu().numpy(), B.cpu().numpy())).cuda()
    assert torch.equal(o1, o2)
    monkeypatch.setenv("SWB_ROTATION", "dmma")
    o3 = torch.empty_like(o1)
    rotate_rows(A, K, B, K, rows, K, o3, K)
    assert (o1 - o3).abs().max().item() < 1e-13


def test_update_int8_rotation_matches_dmma(cuda_ok, monkeypatch):
    """The first-order update with the INT8 rotation agrees with the DMMA
    rotation to the FP64 GEMM level."""
    import paper_1607_04174_b200 as swb
    from oracle import rw_oracle as O
    rng = np.random.default_rng(5)
    dims = (21, 17, 9)
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * (rng.random(n) > 0.5) + rng.normal(0, 0.05, n), 0, 1)
    lap = O.build_laplacian(img, dims, 20.0, "abs", 6)
    vals, vecs = np.linalg.eigh(lap.matrix.toarray())
    m = 37
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=20.0,
                            eigen=swb.EigenBasis(np.asfortranarray(vecs[:, :m]), vals[:m]), d_sqrt=lap.d_sqrt,
                            provenance=swb.PackProvenance(image.content_hash()))
    dp = swb.to_device(pack, image=image)
    a = swb.update_basis(dp, image, 27.0, method="first_order")
    monkeypatch.setenv("SWB_ROTATION", "dmma")
    b = swb.update_basis(dp, image, 27.0, method="first_order")
    assert np.array_equal(a.lambda_hat, b.lambda_hat)
    assert (a.V[:, :m] - b.V[:, :m]).abs().max().item() < 1e-13


def test_int8_probe_runs(cuda_ok):
    import ctypes as C
    ops = C.c_double()
    _lib.check(_lib.load().swb_int8_peak_probe(10, C.byref(ops), None))
    torch.cuda.synchronize()
    assert ops.value > 0


def test_int8_scheme_probe_runs(cuda_ok):
    import ctypes as C
    ops = C.c_double()
    _lib.check(_lib.load().swb_int8_scheme_probe(10, C.byref(ops), None))
    torch.cuda.synchronize()
    assert ops.value == 2.0 * torch.cuda.get_device_properties(0).multi_processor_count * 10 * 28 * 128 * 64 * 32


def test_k_limit(cuda_ok):
    """K = 512 is the largest K whose group sums are exact int32; K = 513 is
    rejected (callers use the DMMA GEMM there)."""
    rng = np.random.default_rng(512)
    A = rng.standard_normal((300, 512))
    B = rng.standard_normal((512, 70))
    got = _run(A, B)
    assert np.all(np.abs(got - A @ B) <= _bound(A, B))
    assert _lib.size("swb_oz_gemm_nn_workspace_bytes", 300, 513, 70) > 0
    dA = torch.zeros((300, 513), dtype=torch.float64, device="cuda")
    dB = torch.zeros((513, 70), dtype=torch.float64, device="cuda")
    out = torch.zeros((300, 70), dtype=torch.float64, device="cuda")
    nb = _lib.size("swb_oz_gemm_nn_workspace_bytes", 300, 513, 70)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    rc = _lib.load().swb_oz_gemm_nn(_ptr(dA), 513, _ptr(dB), 70, 300, 513, 70, _ptr(out), 70, _ptr(ws), nb, None)
    assert rc != 0


def test_rotation_at_scale_matches_dmma(cuda_ok):
    """The c4 rotation shape at 2M+37 rows x K = 400 (three row chunks, the
    last ragged; V with unit-scale orthonormal-like columns, C near the
    identity): the INT8 digit-product GEMM agrees with the FP64 DMMA GEMM to
    the FP64 level everywhere."""
    from paper_1607_04174_b200.device import rotate_rows
    rows, K = (2 << 20) + 37, 400
    g = torch.Generator(device="cuda").manual_seed(4)
    V = torch.randn((rows, K), dtype=torch.float64, device="cuda", generator=g) / rows ** 0.5
    C = torch.eye(K, dtype=torch.float64, device="cuda") + 0.05 * torch.randn((K, K), dtype=torch.float64,
                                                                              device="cuda", generator=g)
    o1 = torch.empty_like(V)
    rotate_rows(V, K, C, K, rows, K, o1, K)
    o2 = torch.empty_like(V)
    _lib.call("swb_gemm_nn", _ptr(V), K, _ptr(C), K, rows, K, K, _ptr(o2), K, 0, None)
    torch.cuda.synchronize()
    scale = V.abs().max().item() * C.abs().max().item() * K
    assert (o1 - o2).abs().max().item() <= 2.0 ** -50 * scale
    assert torch.isfinite(o1).all()
