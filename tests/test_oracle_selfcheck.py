"""Self-checks that pin the restated first-order update (CPU, no GPU).

The reference has no eigenvector update (`/root/reference/SPEC.md:446` lists
"true eigen-updates (perturbation theory)" as a non-goal), so the oracle's
`first_order_update` / `update_coefficients` (SURVEY §7 "Recommended update
definition") cannot be compared with a reference function.  These tests pin
it instead against mathematics the reference does provide:

* the diagonal of P = Vᵀ(ΔL̂)V equals the reference `refresh` shift
  λ̂ − λ (`/root/reference/pkg/src/specwalk/refresh.py:75-79`) for exact
  eigenpairs, where λ̂ is the reference's own Rayleigh quotient;
* for exact (dense `eigh`) bases of small graphs (N ≤ 400), the updated
  eigenvalues λ' and the updated eigenvectors V' converge to the dense
  eigenpairs of the new Laplacian as O(‖ΔL̂‖²): halving β' − β (or the cut
  strength t of an edge cut) divides the errors by ≈ 4, while the
  zeroth-order answer (V unchanged) only halves;
* the same on a truncated basis for the eigenvalues (the Rayleigh quotient
  is second-order accurate regardless of truncation);
* the gap guard: coefficients whose divided difference would exceed the
  guard are exactly zero and every kept |C_ji| is ≤ gap_guard.

The Laplacians come from the oracle's restatement of the reference graph
primitives, which `tests/test_oracle_golden.py` pins bit-exactly to the
reference (`graphs.py:101-159`).
"""

import numpy as np
import pytest

from oracle import rw_oracle as O


def _image(dims, seed):
    """Two-region image (a disk / ball at 0.7 on 0.3) plus N(0, 0.05²) noise."""
    rng = np.random.default_rng(seed)
    grids = np.meshgrid(*[np.arange(d) for d in dims], indexing="ij")
    r2 = sum((g - d / 2.0) ** 2 for g, d in zip(grids, dims))
    base = 0.3 + 0.4 * (r2 < (min(dims) / 3.0) ** 2)
    n = int(np.prod(dims))
    return np.clip(base.ravel(order="F") + rng.normal(0, 0.05, n), 0.0, 1.0)


def _dense_eigs(lap):
    lam, V = np.linalg.eigh(lap.matrix.toarray())
    return lam, V


def _scaled_cut_laplacian(img, dims, beta, mode, conn, cut, t):
    """Edge weights of the cut edges scaled by (1 - t); t = 1 is the cut."""
    heads, tails = O.lattice_edges(dims, conn)
    w = O.edge_weights(img, heads, tails, beta, mode)
    w = np.where(cut, (1.0 - t) * w, w)
    return O.normalized_laplacian(O.symmetric_weights(img.size, heads, tails, w))


CASES = [((14, 12), 4, "sq", 10.0, 0.2),
         ((14, 12), 4, "abs", 3.0, 0.1),
         ((12, 11), 8, "sq", 8.0, 0.2),
         ((6, 6, 5), 6, "abs", 4.0, 0.1),
         ((5, 5, 4), 6, "sq", 10.0, 0.4)]


@pytest.mark.parametrize("dims,conn,mode,beta,db", CASES)
def test_diag_P_equals_refresh_shift(dims, conn, mode, beta, db):
    """diag(Vᵀ ΔL̂ V) == λ̂ − λ for exact eigenpairs (refresh.py:75-79)."""
    img = _image(dims, sum(dims))
    lap0 = O.build_laplacian(img, dims, beta, mode, conn)
    lap1 = O.build_laplacian(img, dims, beta + db, mode, conn)
    lam, V = _dense_eigs(lap0)
    _, _, order, P, _ = O.first_order_update(V, lam, lap0, lap1)
    lam_hat_sorted, order_r = O.refresh(V, lap1)
    np.testing.assert_array_equal(order, order_r)
    lam_hat = np.empty_like(lam_hat_sorted)
    lam_hat[order_r] = lam_hat_sorted
    live = lam_hat > 0                                # the clamp at 0 (refresh.py:78)
    np.testing.assert_allclose(np.diag(P)[live], (lam_hat - lam)[live], rtol=0, atol=1e-13)


def _convergence(make_lap1, lap0, ts, m=None):
    """Errors of the first-order (and zeroth-order) update against the dense
    eigenpairs of each new Laplacian, over every column (all steps are small
    enough that ‖ΔL̂‖₂ is below the smallest spectral gap)."""
    lam, V = _dense_eigs(lap0)
    if m is not None:
        lam, V = lam[:m], V[:, :m]
    rows = []
    for t in ts:
        lap1 = make_lap1(t)
        Vo, lamo, order, P, Cf = O.first_order_update(V, lam, lap0, lap1)
        lam_e, V_e = _dense_eigs(lap1)
        lam_e, V_e = lam_e[:lamo.size], V_e[:, :lamo.size]
        dl = np.abs(np.linalg.eigvalsh((lap1.matrix - lap0.matrix).toarray())).max()
        el = np.abs(lamo - lam_e).max()
        s = np.sign(np.einsum("ij,ij->j", Vo, V_e))
        s[s == 0] = 1.0
        ev = np.linalg.norm(Vo - V_e * s, axis=0).max()
        # zeroth order: the old vectors, in the same (refresh) order
        V0 = V[:, order]
        s0 = np.sign(np.einsum("ij,ij->j", V0, V_e))
        s0[s0 == 0] = 1.0
        e0 = np.linalg.norm(V0 - V_e * s0, axis=0).max()
        rows.append((t, dl, el, ev, e0))
    return rows


def _assert_second_order(rows, check_vectors=True):
    for (t0, _, el0, ev0, e00), (t1, _, el1, ev1, e01) in zip(rows, rows[1:]):
        assert t1 == pytest.approx(t0 / 2)
        assert 3.2 < el0 / el1 < 4.8, rows             # O(|dL|^2) eigenvalues
        if check_vectors:
            assert 3.2 < ev0 / ev1 < 4.8, rows         # O(|dL|^2) eigenvectors
            assert 1.7 < e00 / e01 < 2.4, rows         # zeroth order is O(|dL|)
    if check_vectors:
        # at the smallest step the first-order vectors are far better than V
        assert rows[-1][3] < 0.05 * rows[-1][4]


@pytest.mark.parametrize("dims,conn,mode,beta,db", CASES)
def test_beta_update_converges_second_order(dims, conn, mode, beta, db):
    """λ', V' → dense eigenpairs of L̂(β') as O(‖ΔL̂‖²), full basis, N ≤ 400."""
    img = _image(dims, sum(dims))
    lap0 = O.build_laplacian(img, dims, beta, mode, conn)
    ts = [db / 2 ** k for k in range(3, 7)]
    rows = _convergence(lambda t: O.build_laplacian(img, dims, beta + t, mode, conn), lap0, ts)
    _assert_second_order(rows)


@pytest.mark.parametrize("dims,conn,block,t0", [((14, 12), 4, (3, 2, 6), 0.005), ((12, 11), 8, (4, 3, 5), 0.00125),
                                                ((9, 8), 4, (2, 2, 4), 0.005)])
def test_cut_update_converges_second_order(dims, conn, block, t0):
    """The edge-cut topology update with the cut edges' weights scaled by
    (1 − t): λ', V' → dense eigenpairs as O(t²)."""
    img = _image(dims, 7 + sum(dims))
    beta, mode = 6.0, "sq"
    x0, y0, size = block
    cut = O.block_cut_mask(dims, x0, y0, size=size, connectivity=conn)
    assert cut.any()
    lap0 = O.build_laplacian(img, dims, beta, mode, conn)
    ts = [t0 / 2 ** k for k in range(4)]
    rows = _convergence(lambda t: _scaled_cut_laplacian(img, dims, beta, mode, conn, cut, t), lap0, ts)
    _assert_second_order(rows)


def test_full_cut_equals_build_laplacian_cut():
    """t = 1 of the scaled cut is the oracle's cut Laplacian (weights 0)."""
    dims, conn = (14, 12), 8
    img = _image(dims, 3)
    cut = O.block_cut_mask(dims, 3, 2, size=6, connectivity=conn)
    a = _scaled_cut_laplacian(img, dims, 6.0, "sq", conn, cut, 1.0)
    b = O.build_laplacian(img, dims, 6.0, "sq", conn, cut_edges=cut)
    assert abs(a.matrix - b.matrix).max() == 0.0
    np.testing.assert_array_equal(a.d_sqrt, b.d_sqrt)


def test_truncated_basis_eigenvalues_second_order():
    """With M < N the Rayleigh quotients (λ' = λ̂) stay O(‖ΔL̂‖²) accurate."""
    dims, conn, mode, beta = (18, 16), 4, "sq", 10.0
    img = _image(dims, 11)
    lap0 = O.build_laplacian(img, dims, beta, mode, conn)
    ts = [0.2 / 2 ** k for k in range(4)]
    rows = _convergence(lambda t: O.build_laplacian(img, dims, beta + t, mode, conn), lap0, ts, m=40)
    _assert_second_order(rows, check_vectors=False)


def test_gap_guard_bounds_coefficients():
    """Kept |C_ji| ≤ gap_guard before column scaling; guarded pairs are 0."""
    dims = (14, 12)
    img = _image(dims, 5)
    lap0 = O.build_laplacian(img, dims, 3.0, "abs", 4)
    lap1 = O.build_laplacian(img, dims, 9.0, "abs", 4)      # a large step: many guarded pairs
    lam, V = _dense_eigs(lap0)
    _, _, order, P, Cf = O.first_order_update(V, lam, lap0, lap1)
    # undo sort + scaling: Cf = C[:, order] * s[order]
    C = np.empty_like(Cf)
    C[:, order] = Cf
    C = C / np.diag(C)[None, :]
    diff = lam[None, :] - lam[:, None]
    off = ~np.eye(lam.size, dtype=bool)
    guarded = off & (np.abs(P) > 0.5 * np.abs(diff))
    assert guarded.any()
    assert np.all(C[guarded] == 0.0)
    assert np.abs(C[off]).max() <= 0.5 + 1e-15
    np.testing.assert_allclose(np.linalg.norm(Cf, axis=0), 1.0, rtol=1e-14)
