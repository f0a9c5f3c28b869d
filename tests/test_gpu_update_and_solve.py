"""update_and_solve: the first-order update and the RW solve on the updated
basis with the reconstruction folded into the rotation (the coefficients
ride as extra columns of C in the INT8 GEMM's padding).  Checked against the
two separate calls (update_basis + solve_fast) on the same device pack -- V'
and the eigenvalues bit for bit, fields to 1e-12, labels off near-ties --
and against the oracle at the bench shapes (c4 slab, c2 cut, c1)."""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = Path(__file__).resolve().parent.parent


def _device_pack(swb, s):
    from oracle import rw_oracle as O
    p = s["params"]
    dims, img, V, lam = s["dims"], s["img"], s["V"], s["lam"]
    lap0 = O.build_laplacian(img, dims, p["beta0"], p["weight_mode"], p["connectivity"])
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=p["beta0"], eigen=swb.EigenBasis(V, lam),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    dp = swb.to_device(pack, image=image, connectivity=p["connectivity"], weight_mode=p["weight_mode"])
    return image, dp, lap0


def _check_against_separate(swb, dp, image, prob, beta, cut=None, m_use=None):
    """update_and_solve vs update_basis + solve_fast on the same pack."""
    up1 = swb.update_basis(dp, image, beta, cut_edges=cut)
    f1 = swb.solve_fast(up1, None, prob, m_use, want_field=True)
    up2, f2 = swb.update_and_solve(dp, image, prob, beta, cut_edges=cut, m_use=m_use, want_field=True)
    m = up1.m
    # the rotation's columns [0, K) are the same digit products: V' bit for bit
    assert torch.equal(up1.V[:, :m], up2.V[:, :m])
    np.testing.assert_array_equal(up1.lambda_hat, up2.lambda_hat)
    np.testing.assert_array_equal(up1.order, up2.order)
    u1, u2 = f1.values, f2.values
    np.testing.assert_allclose(u2, u1, rtol=0, atol=1e-12)
    l1, l2 = swb.hard_labels(f1).labels, swb.hard_labels(f2).labels
    top2 = f1.top2_dev.cpu().numpy()
    assert not ((l1 != l2) & (top2 >= 1e-9)).any()
    return up2, f2


def test_c4_slab_fused_matches_separate_and_oracle(cuda_ok):
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_1607_04174_b200 as swb
    from oracle import rw_oracle as O
    s = bench.cpu_sample("c4", None, 400)
    p = s["params"]
    image, dp, lap0 = _device_pack(swb, s)
    prob = swb.LabelProblem(num_labels=p["labels"], seeds=swb.SeedPartition(s["n"], s["seeds"], s["labs"]))
    up, f = _check_against_separate(swb, dp, image, prob, p["beta1"])
    lap1 = O.build_laplacian(s["img"], s["dims"], p["beta1"], p["weight_mode"], p["connectivity"])
    Vo, lamo, _, _, _ = O.first_order_update(s["V"], s["lam"], lap0, lap1)
    u_ref = O.solve_fast(Vo, lamo, lap1.d_sqrt, lap1.matrix, s["seeds"], s["labs"], p["labels"])
    np.testing.assert_allclose(f.values, u_ref, rtol=0, atol=1e-9)
    gap = O.top2_gap(u_ref)
    assert not ((swb.hard_labels(f).labels != O.hard_labels(u_ref)) & (gap >= 1e-9)).any()


def test_c2_cut_fused_matches_separate(cuda_ok):
    """The c2 full-size topology update (block cut), K = 200: 200 + 3 extra
    columns fit the padding of the 256-column tile."""
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_1607_04174_b200 as swb
    from paper_1607_04174_b200 import workloads as W
    s = bench.cpu_sample("c2", None, 200)
    p = s["params"]
    image, dp, _ = _device_pack(swb, s)
    x0, y0 = s["cut"]
    mask = W.block_cut_voxel_mask(s["dims"], p["connectivity"], x0, y0, size=p["cut_block"])
    prob = swb.LabelProblem(num_labels=p["labels"], seeds=swb.SeedPartition(s["n"], s["seeds"], s["labs"]))
    _check_against_separate(swb, dp, image, prob, p["beta0"], cut=mask)


def test_c1_fused_matches_separate_with_m_use(cuda_ok):
    """c1 (K = 50: 50 + 2 columns in one 64-column tile) at a truncated
    m_use, plus a basis size that is a multiple of 64 (the extra columns
    then need a tile of their own)."""
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_1607_04174_b200 as swb
    s = bench.cpu_sample("c1", None, 50)
    p = s["params"]
    image, dp, _ = _device_pack(swb, s)
    prob = swb.LabelProblem(num_labels=p["labels"], seeds=swb.SeedPartition(s["n"], s["seeds"], s["labs"]))
    _check_against_separate(swb, dp, image, prob, p["beta1"])
    _check_against_separate(swb, dp, image, prob, p["beta1"], m_use=37)
    s64 = bench.cpu_sample("c1", None, 64)
    image, dp64, _ = _device_pack(swb, s64)
    _check_against_separate(swb, dp64, image, prob, p["beta1"])


def test_fused_many_labels_and_fallbacks(cuda_ok):
    """L > 8 (the in-place many-label finalize), no seeds and gamma > 0
    (both take the separate calls)."""
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_1607_04174_b200 as swb
    s = bench.cpu_sample("c1", None, 50)
    p = s["params"]
    image, dp, _ = _device_pack(swb, s)
    rng = np.random.default_rng(5)
    n = s["n"]
    seeds = np.sort(rng.choice(n, 60, replace=False))
    labs = rng.integers(0, 12, seeds.size)
    labs[:12] = np.arange(12)
    prob = swb.LabelProblem(num_labels=12, seeds=swb.SeedPartition(n, seeds, labs))
    _check_against_separate(swb, dp, image, prob, p["beta1"])
    pri = rng.random((n, 3))
    pri /= pri.sum(1, keepdims=True)
    prob_g = swb.LabelProblem(num_labels=3, seeds=swb.SeedPartition(n, [], []), priors=pri, gamma=0.5)
    up, f = swb.update_and_solve(dp, image, prob_g, p["beta1"], want_field=True)
    f1 = swb.solve_fast(swb.update_basis(dp, image, p["beta1"]), None, prob_g, want_field=True)
    np.testing.assert_allclose(f.values, f1.values, rtol=0, atol=1e-12)


def test_fused_gamma_priors(cuda_ok):
    """gamma > 0 through update_and_solve: V'^T P^ formed as C^T (V^T P^)
    before the rotation; 27 labels with priors, without and with seeds."""
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_1607_04174_b200 as swb
    s = bench.cpu_sample("c1", None, 50)
    p = s["params"]
    image, dp, _ = _device_pack(swb, s)
    rng = np.random.default_rng(8)
    n = s["n"]
    pri = rng.random((n, 27)) ** 4
    pri /= pri.sum(1, keepdims=True)
    seeds = np.sort(rng.choice(n, 30, replace=False))
    for sp in (swb.SeedPartition(n, [], []), swb.SeedPartition(n, seeds, rng.integers(0, 27, seeds.size))):
        prob = swb.LabelProblem(num_labels=27, seeds=sp, priors=pri, gamma=1.0)
        _check_against_separate(swb, dp, image, prob, p["beta1"])


@pytest.mark.parametrize("L", [70, 125, 200, 300])
def test_fused_finalize_label_widths(cuda_ok, L):
    """The many-label finalize of update_and_solve at every dispatch width
    (register rows of <= 128 / <= 256 labels, the loop kernel beyond): c5 has
    125 labels."""
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_1607_04174_b200 as swb
    s = bench.cpu_sample("c1", None, 320)
    p = s["params"]
    image, dp, _ = _device_pack(swb, s)
    rng = np.random.default_rng(L)
    n = s["n"]
    pri = rng.random((n, L)) ** 4
    pri /= pri.sum(1, keepdims=True)
    seeds = np.sort(rng.choice(n, 40, replace=False))
    sp = swb.SeedPartition(n, seeds, rng.integers(0, L, seeds.size))
    prob = swb.LabelProblem(num_labels=L, seeds=sp, priors=pri, gamma=1.0)
    _check_against_separate(swb, dp, image, prob, p["beta1"])


def test_fused_on_the_dmma_rotation(cuda_ok):
    """SWB_ROTATION=dmma (and K > 512) rotate on the FP64 DMMA GEMM: the
    extra columns V (C coeff) then come from a second DMMA product."""
    import os
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_1607_04174_b200 as swb
    s = bench.cpu_sample("c1", None, 50)
    p = s["params"]
    image, dp, _ = _device_pack(swb, s)
    prob = swb.LabelProblem(num_labels=p["labels"], seeds=swb.SeedPartition(s["n"], s["seeds"], s["labs"]))
    os.environ["SWB_ROTATION"] = "dmma"
    try:
        up1 = swb.update_basis(dp, image, p["beta1"])
        f1 = swb.solve_fast(up1, None, prob, want_field=True)
        up2, f2 = swb.update_and_solve(dp, image, prob, p["beta1"], want_field=True)
    finally:
        os.environ.pop("SWB_ROTATION", None)
    assert torch.equal(up1.V[:, :up1.m], up2.V[:, :up2.m])
    np.testing.assert_allclose(f2.values, f1.values, rtol=0, atol=1e-12)


def test_fused_with_select_m(cuda_ok):
    """update_and_solve(policy=...): select_m on the updated basis (its seed
    rows formed before the rotation) picks the same m as select_m on the
    update_basis result, and the field matches solve_fast at that m (c3's
    adaptive workload on a 128 x 128 x 4 slab)."""
    sys.path.insert(0, str(ROOT))
    import bench
    import paper_1607_04174_b200 as swb
    s = bench.cpu_sample("c3", None, 150)
    p = s["params"]
    image, dp, _ = _device_pack(swb, s)
    prob = swb.LabelProblem(num_labels=p["labels"], seeds=swb.SeedPartition(s["n"], s["seeds"], s["labs"]))
    pol = swb.AdaptivePolicy(epsilon=p["epsilon"])
    up1 = swb.update_basis(dp, image, p["beta1"])
    m1, _ = swb.select_m(up1, prob, pol)
    f1 = swb.solve_fast(up1, None, prob, m1, want_field=True)
    up2, f2 = swb.update_and_solve(dp, image, prob, p["beta1"], policy=pol, want_field=True)
    assert f2.m_use == m1
    assert torch.equal(up1.V[:, :up1.m], up2.V[:, :up2.m])
    np.testing.assert_allclose(f2.values, f1.values, rtol=0, atol=1e-12)
