"""The rotation's digit planes emitted by the projection's diagonal tiles
(swb_gemm_tn_sym_emit, row scales from the previous rotation's recorded row
maxima) instead of the split pass: the planes and row scales are byte-for-
byte those of swb_oz_split_rows, over several row chunks and for tile widths
80 (K = 400, 200) and 64 (K = 256); the chained update through them matches
the split path (P, V' to rounding: the projection's CTA partition differs)."""

import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _pack(dims, m, seed):
    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200 import workloads as W
    from paper_1607_04174_b200.device import DevicePack, LatticeSpec
    rng = np.random.default_rng(seed)
    n = int(np.prod(dims))
    img = np.clip(0.5 + 0.3 * (rng.random(n) < 0.3) + rng.normal(0, 0.05, n), 0, 1)
    image = swb.Image(dims, img)
    lattice = LatticeSpec.make(dims, 6 if len(dims) == 3 else 4, "sq")
    V = W.orthonormal_basis_device(n, m, seed=seed)
    lam = torch.sort(torch.rand(m, dtype=torch.float64, device="cuda") * 0.1 + 1e-4).values
    img_dev = torch.from_numpy(img).cuda()
    g0 = swb.DeviceGraph.build(img_dev, lattice, 60.0)
    prov = swb.PackProvenance(image_hash=image.content_hash())
    dp = DevicePack(V, m, lam, g0.d_sqrt_dev, g0.dnorm, dims, (), 60.0, prov, lattice, image_dev=img_dev, graph=g0)
    from paper_1607_04174_b200 import api
    api._image_entry(image)[2] = img_dev
    return image, dp


@pytest.mark.parametrize("n,m", [(2_500_000, 400), (300_000, 200), (700_000, 256)])
def test_emitted_planes_equal_split(cuda_ok, n, m):
    from paper_1607_04174_b200 import _lib
    from paper_1607_04174_b200.device import oz_full_workspace, ptr
    torch.manual_seed(3)
    X = torch.randn(n, m, dtype=torch.float64, device="cuda") * torch.rand(n, 1, dtype=torch.float64, device="cuda")
    X[7].zero_()                                             # a zero row: scale 2^-28, zero digits
    Y = torch.randn(n, m, dtype=torch.float64, device="cuda")
    amax = X.abs().max(dim=1).values.contiguous().view(torch.int64)
    m2 = m + 3
    full = oz_full_workspace(n, m, m2)
    P1 = torch.empty(m, m, dtype=torch.float64, device="cuda")
    P2 = torch.empty_like(P1)
    tws = torch.empty(_lib.size("swb_gemm_tn_workspace_bytes", n, m, m), dtype=torch.uint8, device="cuda")
    _lib.call("swb_gemm_tn_sym_emit", ptr(X), m, ptr(Y), m, n, m, ptr(P1), m, ptr(tws), tws.numel(), ptr(amax), m2,
              ptr(full), full.numel(), None)
    _lib.call("swb_gemm_tn", ptr(X), m, ptr(Y), m, n, m, m, 1, ptr(P2), m, ptr(tws), tws.numel(), None)
    np.testing.assert_allclose(P1.cpu().numpy(), P2.cpu().numpy(), rtol=1e-12, atol=1e-9)
    info = (C.c_int64 * 5)()
    _lib.call("swb_oz_layout_info", n, m, m2, info)
    chunk, nkc, off0, a_sl, stride = list(info)
    nb = _lib.size("swb_oz_gemm_nn_workspace_bytes", n, m, m2)
    ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
    for i in range((n + chunk - 1) // chunk):
        r0 = i * chunk
        nr = min(chunk, n - r0)
        _lib.call("swb_oz_split_rows", C.c_void_p(X.data_ptr() + 8 * r0 * m), m, nr, n, m, m2, i & 1, ptr(ws),
                  ws.numel(), None)
        torch.cuda.synchronize()
        used = (nr + 127) // 128 * nkc * 7 * 4096            # row blocks x K chunks x 28 KB stages
        e = full[off0 + i * stride: off0 + i * stride + used]
        sref = ws[off0 + (i & 1) * stride: off0 + (i & 1) * stride + used]
        assert torch.equal(e, sref), f"planes differ in chunk {i}"
        se = full[off0 + i * stride + a_sl: off0 + i * stride + a_sl + 8 * nr].view(torch.float64)
        ss = ws[off0 + (i & 1) * stride + a_sl: off0 + (i & 1) * stride + a_sl + 8 * nr].view(torch.float64)
        assert torch.equal(se, ss), f"row scales differ in chunk {i}"


@pytest.mark.parametrize("dims,m", [((256, 256, 20), 400), ((128, 128, 8), 200)])
def test_chained_update_through_emitted_planes(cuda_ok, dims, m):
    import paper_1607_04174_b200 as swb
    image, dp = _pack(dims, m, 11)
    os.environ["SWB_EMIT"] = "1"
    try:
        up1 = swb.update_basis(dp, image, 80.0, keep_P=True)      # split path (no maxima yet), records them
    finally:
        os.environ.pop("SWB_EMIT", None)
    amax = torch.from_numpy(np.abs(up1.V[:, :m].cpu().numpy()).max(axis=1)).cuda()
    assert torch.equal(up1.row_amax_dev.view(torch.float64), amax)
    ref = swb.update_basis(up1, image, 60.0, keep_P=True)           # split path (default)
    os.environ["SWB_EMIT"] = "1"
    try:
        em = swb.update_basis(up1, image, 60.0, keep_P=True)        # planes from the projection
    finally:
        os.environ.pop("SWB_EMIT", None)
    np.testing.assert_allclose(em.P.cpu().numpy(), ref.P.cpu().numpy(), rtol=0, atol=1e-13)
    np.testing.assert_allclose(em.V[:, :m].cpu().numpy(), ref.V[:, :m].cpu().numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(em.lambda_hat, ref.lambda_hat, rtol=1e-13, atol=1e-16)
