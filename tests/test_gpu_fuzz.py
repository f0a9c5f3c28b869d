"""Seeded randomized sweep of the whole interaction (first-order update with
beta and / or edge cuts, then a solve) against the oracle: lattice shapes
and connectivities, weight modes, basis sizes (odd / even / not a multiple
of the 64-column stencil block), gap guards, label counts, gamma = 0 with
seeds and gamma > 0 with priors.  Tolerances as in test_gpu_parity.py."""

import numpy as np
import pytest

import paper_1607_04174_b200 as swb
from oracle import rw_oracle as O

pytestmark = pytest.mark.gpu

SHAPES = [(17, 13), (40, 9), (9, 40), (7, 6, 5), (11, 8, 6), (5, 12, 9), (33, 31), (6, 6, 14)]


def _case(i):
    rng = np.random.default_rng(1000 + i)
    dims = SHAPES[i % len(SHAPES)]
    d3 = len(dims) == 3
    conn = 6 if d3 else (8 if i % 3 == 0 else 4)
    mode = "sq" if i % 2 else "abs"
    n = int(np.prod(dims))
    m = int(min(n - 1, [17, 33, 40, 65, 24, 50][i % 6]))
    k = 2 + i % 4
    gamma = 0.0 if i % 3 else 0.7
    b0 = float(rng.uniform(5, 40))
    b1 = b0 * float(rng.uniform(0.7, 1.5))
    guard = [0.5, 0.25, 0.75][i % 3]
    cut = None
    if not d3 and i % 4 == 1:
        x0, y0 = int(rng.integers(0, dims[0] - 4)), int(rng.integers(0, dims[1] - 4))
        cut = O.block_cut_mask(dims, x0, y0, size=4, connectivity=conn)
    return rng, dims, conn, mode, n, m, k, gamma, b0, b1, guard, cut


@pytest.mark.parametrize("i", range(24))
def test_update_and_solve_sweep(cuda_ok, i):
    rng, dims, conn, mode, n, m, k, gamma, b0, b1, guard, cut = _case(i)
    labels_img = (rng.random(n) * k).astype(int)
    img = np.clip(0.2 + 0.6 * labels_img / max(k - 1, 1) + rng.normal(0, 0.05, n), 0, 1)
    lap0 = O.build_laplacian(img, dims, b0, mode, conn)
    vals, vecs = np.linalg.eigh(lap0.matrix.toarray())
    V, lam = vecs[:, :m], vals[:m]
    image = swb.Image(dims, img)
    pack = swb.SpectralPack(dims=dims, spacing=(), beta=b0, eigen=swb.EigenBasis(np.asfortranarray(V), lam),
                            d_sqrt=lap0.d_sqrt, provenance=swb.PackProvenance(image.content_hash()))
    dp = swb.to_device(pack, image=image, connectivity=conn, weight_mode=mode)
    up = swb.update_basis(dp, image, b1, cut_edges=cut, method="first_order", gap_guard=guard, keep_P=True)
    lap1 = O.build_laplacian(img, dims, b1, mode, conn, cut_edges=cut)
    Vo, lamo, order, P, _ = O.first_order_update(V, lam, lap0, lap1, gap_guard=guard)
    np.testing.assert_allclose(up.P.cpu().numpy()[:, :m], P, rtol=0, atol=1e-12)
    np.testing.assert_allclose(up.lambda_hat, lamo, rtol=1e-9, atol=1e-13)
    if gamma == 0.0:
        s = min(n, 3 * k + 2)
        seeds = np.sort(rng.choice(n, s, replace=False))
        labs = np.arange(s) % k
        prob = swb.LabelProblem(num_labels=k, seeds=swb.SeedPartition(n, seeds, labs))
        u = O.solve_fast(Vo, lamo, lap1.d_sqrt, lap1.matrix, seeds, labs, k, m_use=m)
    else:
        pri = rng.random((n, k)) + 0.1
        pri /= pri.sum(axis=1, keepdims=True)
        seeds = np.sort(rng.choice(n, 2, replace=False))
        labs = np.array([0, k - 1])
        prob = swb.LabelProblem(num_labels=k, seeds=swb.SeedPartition(n, seeds, labs), priors=pri, gamma=gamma)
        u = O.solve_fast(Vo, lamo, lap1.d_sqrt, lap1.matrix, seeds, labs, k, gamma=gamma, priors=pri, m_use=m)
    f = swb.solve_fast(up, up.laplacian, prob, m_use=m, want_field=True)
    np.testing.assert_allclose(f.values, u, atol=1e-9)
    gap = O.top2_gap(u)
    lab = swb.hard_labels(f).labels
    assert not ((lab != O.hard_labels(u)) & (gap >= 1e-9)).any()
