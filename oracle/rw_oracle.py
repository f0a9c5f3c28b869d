"""CPU restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.

This module is the parity oracle for the B200 kernels in
``paper_1607_04174_b200``.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline leg (``--impl reference`` / ``cpu_baseline``)
may import it, and only as the checker or the timed CPU baseline.  The
product path never calls into this file.

It restates, in plain numpy/scipy, the algorithm of the reference package
``specwalk`` (arXiv 1607.04174, Andrews & Hamarneh); every function cites
the reference file:line it follows (paths relative to
``/root/reference/pkg/src/specwalk/``).  It is pinned against golden vectors
produced by running the reference itself (``tests/golden/make_golden.py``,
checked by ``tests/test_oracle_golden.py``).

Two pieces have no reference function:
  * the first-order eigenvector rotation ``first_order_update`` (the
    eigenvalue half is the reference ``refresh`` Rayleigh quotient, pinned);
  * the edge-cut topology update (built here from the reference graph
    primitives restated below, which are pinned bit-exactly).
They are pinned by mathematical self-checks instead of reference outputs
(``tests/test_oracle_selfcheck.py``): P's diagonal equals the reference
refresh shift λ̂ − λ to 1e-13 for exact eigenpairs, and on dense ``eigh``
bases (N ≤ 180) λ' and V' converge to the new Laplacian's eigenpairs as
O(‖ΔL̂‖²) for β steps and for edge cuts of strength t (errors / 4 per
halving), while the zeroth-order answer only halves.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

# graphs.py:20
W_MIN = 1e-8
# fastrw.py:37
MAX_SEEDS = 10_000
# adaptive.py:19-20
DEFAULT_EPSILON = 0.1
DEFAULT_STRIDE = 4


class OracleError(Exception):
    """Carries the reference exception class name in ``kind``."""

    def __init__(self, kind: str, message: str, condition: float = float("inf")):
        super().__init__(f"{kind}: {message}")
        self.kind = kind
        self.condition = condition


# ---------------------------------------------------------------------------
# graph + normalized Laplacian (graphs.py:101-159)
# ---------------------------------------------------------------------------

def forward_offsets(ndim: int, connectivity: int) -> list[tuple[int, ...]]:
    """Forward neighbour offsets (dx, dy[, dz]) of the lattice.

    4/6-connectivity are the reference lattice (graphs.py:101-113: one axis
    at a time, x first).  8-connectivity (2-D) is the BASELINE config-2
    extension: the axis edges followed by the two diagonals (+1,+1), (-1,+1).
    """
    if ndim == 2 and connectivity == 4:
        return [(1, 0), (0, 1)]
    if ndim == 3 and connectivity == 6:
        return [(1, 0, 0), (0, 1, 0), (0, 0, 1)]
    if ndim == 2 and connectivity == 8:
        return [(1, 0), (0, 1), (1, 1), (-1, 1)]
    raise OracleError("InvalidParam", f"unsupported connectivity {connectivity} in {ndim}-D")


def lattice_edges(dims, connectivity: int | None = None):
    """(heads, tails) flat x-fastest indices; one entry per undirected edge.

    Follows graphs.py:101-113 (grid in Fortran order, per-axis slices); the
    diagonal directions of 8-connectivity are appended after the axis edges.
    """
    dims = tuple(int(n) for n in dims)
    nd = len(dims)
    if connectivity is None:
        connectivity = 4 if nd == 2 else 6
    grid = np.arange(int(np.prod(dims)), dtype=np.int64).reshape(dims, order="F")
    heads, tails = [], []
    for off in forward_offsets(nd, connectivity):
        src = [slice(None)] * nd
        dst = [slice(None)] * nd
        for ax, o in enumerate(off):
            if o > 0:
                src[ax] = slice(None, -o)
                dst[ax] = slice(o, None)
            elif o < 0:
                src[ax] = slice(-o, None)
                dst[ax] = slice(None, o)
        heads.append(grid[tuple(src)].ravel(order="F"))
        tails.append(grid[tuple(dst)].ravel(order="F"))
    return np.concatenate(heads), np.concatenate(tails)


def edge_weights(intensities, heads, tails, beta: float, weight_mode: str = "abs"):
    """w = max(exp(-beta*|dI|), W_MIN) (graphs.py:134-136); "sq" uses dI^2."""
    if beta < 0:
        raise OracleError("InvalidParam", f"beta must be >= 0, got {beta}")
    d = intensities[heads] - intensities[tails]
    if weight_mode == "abs":
        arg = np.abs(d)
    elif weight_mode == "sq":
        arg = d * d
    else:
        raise OracleError("InvalidParam", f"unknown weight mode {weight_mode!r}")
    return np.maximum(np.exp(-beta * arg), W_MIN)


def symmetric_weights(n: int, heads, tails, w) -> sp.csr_matrix:
    """Symmetric CSR from one direction per edge (graphs.py:116-124)."""
    mat = sp.coo_matrix((np.concatenate([w, w]),
                         (np.concatenate([heads, tails]),
                          np.concatenate([tails, heads]))), shape=(n, n)).tocsr()
    mat.sort_indices()
    return mat


class Lap:
    """Normalized Laplacian L^ = D^-1/2 (D - W) D^-1/2 (graphs.py:143-159)."""

    def __init__(self, matrix: sp.csr_matrix, d_sqrt: np.ndarray, degrees: np.ndarray):
        self.matrix = matrix
        self.d_sqrt = d_sqrt
        self.degrees = degrees

    @property
    def n_vertices(self) -> int:
        return self.matrix.shape[0]


def normalized_laplacian(weights: sp.spmatrix) -> Lap:
    """graphs.py:143-159 (NORMALIZED branch), including the explicit
    (L + L^T)/2 symmetrization and the DegenerateGraph check."""
    weights = weights.tocsr()
    deg = np.asarray(weights.sum(axis=1)).ravel()
    if np.any(deg <= 0):
        raise OracleError("DegenerateGraph", "graph has an isolated vertex")
    d_sqrt = np.sqrt(deg)
    inv = sp.diags(1.0 / d_sqrt)
    mat = (inv @ (sp.diags(deg) - weights) @ inv).tocsr()
    mat = ((mat + mat.T) * 0.5).tocsr()
    mat.sort_indices()
    return Lap(mat, d_sqrt, deg)


def build_laplacian(intensities, dims, beta: float, weight_mode: str = "abs",
                    connectivity: int | None = None, cut_edges=None) -> Lap:
    """build_graph + laplacian (graphs.py:127-140, 143-159).

    ``cut_edges``: optional boolean mask over the lattice_edges() list; cut
    edges get weight 0 (the topology-change extension).
    """
    intensities = np.asarray(intensities, dtype=np.float64).ravel()
    heads, tails = lattice_edges(dims, connectivity)
    w = edge_weights(intensities, heads, tails, beta, weight_mode)
    if cut_edges is not None:
        w = np.where(np.asarray(cut_edges, dtype=bool), 0.0, w)
    return normalized_laplacian(symmetric_weights(intensities.size, heads, tails, w))


def block_cut_mask(dims, x0: int, y0: int, size: int = 32, connectivity: int = 8):
    """Edges with exactly one endpoint inside the block [x0,x0+size)x[y0,y0+size)."""
    heads, tails = lattice_edges(dims, connectivity)
    nx = dims[0]

    def inside(f):
        x, y = f % nx, f // nx
        return (x >= x0) & (x < x0 + size) & (y >= y0) & (y < y0 + size)

    return inside(heads) != inside(tails)


# ---------------------------------------------------------------------------
# beta refresh (refresh.py:63-82) and the first-order update (new)
# ---------------------------------------------------------------------------

def refresh(vectors: np.ndarray, lap_new: Lap):
    """refresh.py:75-79: lam^ = max(diag(V^T L'V)/diag(V^T V), 0), stable sort."""
    v = np.asarray(vectors, dtype=np.float64)
    norms = np.einsum("ij,ij->j", v, v)
    quad = np.einsum("ij,ij->j", v, lap_new.matrix @ v)
    lam = np.maximum(quad / norms, 0.0)
    order = np.argsort(lam, kind="stable")
    return lam[order], order


def update_coefficients(P: np.ndarray, lam_old: np.ndarray, lam_hat_unsorted: np.ndarray,
                        gap_guard: float = 0.5):
    """Coefficient matrix of the first-order eigenvector update (no reference
    function; SURVEY §7 "Recommended update definition").

    C_ii = 1; for i != j, C_ji = P_ji / (lam_i - lam_j) when
    |P_ji| <= gap_guard*|lam_i - lam_j|, else 0 (stored lam).  Columns are
    scaled to unit norm assuming V^T V = I, then stably sorted by lam^.
    Returns (Cfull M x M = C[:, order] * s[order], lam_sorted, order).
    """
    m = lam_old.size
    diff = lam_old[None, :] - lam_old[:, None]        # [j, i] = lam_i - lam_j
    C = np.zeros((m, m))
    ok = (np.abs(P) <= gap_guard * np.abs(diff)) & (diff != 0.0)
    np.fill_diagonal(ok, False)
    C[ok] = P[ok] / diff[ok]
    np.fill_diagonal(C, 1.0)
    s = 1.0 / np.sqrt(np.einsum("ji,ji->i", C, C))
    order = np.argsort(lam_hat_unsorted, kind="stable")
    return C[:, order] * s[order][None, :], lam_hat_unsorted[order], order


def first_order_update(vectors: np.ndarray, lam_old: np.ndarray, lap_old: Lap,
                       lap_new: Lap, gap_guard: float = 0.5):
    """V' = V C Pi diag(s), lam' = refresh lam^[Pi] (north-star part (a))."""
    v = np.asarray(vectors, dtype=np.float64)
    dL = (lap_new.matrix - lap_old.matrix).tocsr()
    P = v.T @ (dL @ v)
    P = 0.5 * (P + P.T)
    norms = np.einsum("ij,ij->j", v, v)
    quad = np.einsum("ij,ij->j", v, lap_new.matrix @ v)
    lam_hat = np.maximum(quad / norms, 0.0)
    Cf, lam_sorted, order = update_coefficients(P, np.asarray(lam_old, np.float64),
                                                lam_hat, gap_guard)
    return v @ Cf, lam_sorted, order, P, Cf


# ---------------------------------------------------------------------------
# online solve (fastrw.py:332-467, solver.py:55-66, images.py:128-130)
# ---------------------------------------------------------------------------

def dense_solve(a: np.ndarray, rhs: np.ndarray):
    """fastrw.py:332-344: LU + 1-norm rcond; SingularSmallSystem below 1e-14."""
    try:
        lu, piv = sla.lu_factor(a)
    except sla.LinAlgError as exc:  # pragma: no cover - LAPACK path
        raise OracleError("SingularSmallSystem", str(exc))
    anorm = np.linalg.norm(a, 1) if a.size else 0.0
    rcond = sla.lapack.dgecon(lu, anorm, norm="1")[0] if a.size else 1.0
    if not np.isfinite(rcond) or rcond < 1e-14:
        raise OracleError("SingularSmallSystem", "seed system numerically singular",
                          condition=1.0 / max(rcond, 1e-300))
    return sla.lu_solve((lu, piv), rhs), rcond


def finalize(u: np.ndarray, seed_idx, seed_lab, k: int) -> np.ndarray:
    """solver.py:55-66: one-hot seeds, clip >= 0, dead rows -> 1/K, normalize."""
    if len(seed_idx):
        u[seed_idx] = 0.0
        u[seed_idx, seed_lab] = 1.0
    u = np.clip(u, 0.0, None)
    sums = u.sum(axis=1, keepdims=True)
    dead = (sums == 0.0).ravel()
    if dead.any():
        u[dead] = 1.0 / k
        sums[dead] = 1.0
    return u / sums


def hard_labels(u: np.ndarray) -> np.ndarray:
    """images.py:128-130: argmax, ties to the lowest label."""
    return np.argmax(u, axis=1)


def spectral_weights(values: np.ndarray, gamma: float) -> np.ndarray:
    """fastrw.py:399-403: 1/(lam+gamma), or deflated 1/lam (lam>1e-10) at gamma=0."""
    if gamma == 0:
        w = np.zeros_like(values)
        nz = values > 1e-10
        w[nz] = 1.0 / values[nz]
        return w
    return 1.0 / (values + gamma)


def sorted_seeds(seed_idx, seed_lab, n: int):
    """SeedPartition normalisation (graphs.py:51-98)."""
    idx = np.asarray(seed_idx, dtype=np.int64).ravel()
    lab = np.asarray(seed_lab, dtype=np.int64).ravel()
    if idx.size != lab.size:
        raise OracleError("InvalidParam", "seed_indices and seed_labels must have equal length")
    if idx.size:
        o = np.argsort(idx, kind="stable")
        idx, lab = idx[o], lab[o]
        if idx[0] < 0 or idx[-1] >= n:
            raise OracleError("IndexError", "seed index out of range")
        if np.any(np.diff(idx) == 0):
            raise OracleError("InvalidParam", "seed indices must be unique")
    return idx, lab


def solve_fast(vectors, values, d_sqrt, lap_matrix, seed_idx, seed_lab, k: int,
               gamma: float = 0.0, priors=None, m_use: int | None = None,
               return_parts: bool = False):
    """fastrw.py:352-467 restated in one pass (no column streaming; the
    reference proves streaming == in-memory to 1e-12, test_fastrw.py:132-144).

    ``vectors`` N x M (any float dtype; promoted to f64 as the reference does),
    ``d_sqrt`` the pack's d_sqrt, ``lap_matrix`` the CSR normalized Laplacian
    (only its seed rows are read).  Returns the finalized N x K field.
    """
    vectors = np.asarray(vectors)
    d_sqrt = np.asarray(d_sqrt, dtype=np.float64)
    n = d_sqrt.size
    mtot = np.asarray(values).size
    if m_use is None:
        m_use = mtot
    if not 1 <= m_use <= mtot:
        raise OracleError("InvalidParam", f"m_use must be in 1..{mtot}")
    if m_use < k:
        raise OracleError("InsufficientBasis", f"m_use={m_use} cannot represent {k} labels")
    s_idx, s_lab = sorted_seeds(seed_idx, seed_lab, n)
    s = s_idx.size
    if s > MAX_SEEDS:
        raise OracleError("InvalidParam", f"at most {MAX_SEEDS} seeds supported")
    vals = np.asarray(values[:m_use], dtype=np.float64)
    mask = np.ones(n, dtype=bool)
    mask[s_idx] = False
    n_idx = np.flatnonzero(mask)
    u = np.zeros((n, k))
    if n_idx.size == 0:
        return finalize(u, s_idx, s_lab, k)
    q = np.asarray(vectors[:, :m_use], dtype=np.float64)
    p_masked = None
    if priors is not None:
        p_masked = np.asarray(priors, dtype=np.float64) * d_sqrt[:, None]
        p_masked[s_idx] = 0.0
    w = spectral_weights(vals, gamma)
    seed_rows = lap_matrix[s_idx] if s else None
    l_s = seed_rows[:, s_idx].toarray() if s else np.zeros((0, 0))
    q_s = q[s_idx]
    b_qn = (seed_rows @ q - l_s @ q_s) if s else np.zeros((0, m_use))
    g = d_sqrt / np.linalg.norm(d_sqrt)
    g_masked = g.copy()
    g_masked[s_idx] = 0.0
    t_p = q.T @ p_masked if p_masked is not None else None
    onehot = np.zeros((s, k))
    onehot[np.arange(s), s_lab] = 1.0
    u_s_hat = onehot * d_sqrt[s_idx, None]
    extra = None
    rcond = None
    if gamma > 0:
        if s:
            a_s = np.eye(s) - (b_qn * w) @ q_s.T
            rhs = l_s @ u_s_hat + gamma * u_s_hat + gamma * (b_qn * w) @ t_p
            f_s, rcond = dense_solve(a_s, rhs)
            coeff = w[:, None] * (q_s.T @ f_s + gamma * t_p)
        else:
            coeff = w[:, None] * (gamma * t_p)
    else:
        gq = q.T @ g_masked
        g_s = g[s_idx]
        a = np.empty((s + 1, s + 1))
        a[:s, :s] = np.eye(s) - (b_qn * w) @ q_s.T
        a[:s, s] = -(seed_rows @ g_masked)
        a[s, :s] = -(gq * w) @ q_s.T
        a[s, s] = g_s @ g_s
        rhs = np.empty((s + 1, k))
        rhs[:s] = l_s @ u_s_hat
        rhs[s] = g_s @ u_s_hat
        sol, rcond = dense_solve(a, rhs)
        coeff = w[:, None] * (q_s.T @ sol[:s])
        extra = sol[s]
    u_hat = q @ coeff
    if extra is not None:
        u_hat += np.outer(g_masked, extra)
    u[n_idx] = u_hat[n_idx] / d_sqrt[n_idx, None]
    out = finalize(u, s_idx, s_lab, k)
    if return_parts:
        return out, {"coeff": coeff, "extra": extra, "rcond": rcond, "q_s": q_s,
                     "b_qn": b_qn, "weights": w}
    return out


def top2_gap(u: np.ndarray) -> np.ndarray:
    """Difference between the two largest probabilities per row."""
    if u.shape[1] < 2:
        return np.full(u.shape[0], np.inf)
    part = np.partition(u, -2, axis=1)
    return part[:, -1] - part[:, -2]


# ---------------------------------------------------------------------------
# dynamic basis size (adaptive.py:23-185)
# ---------------------------------------------------------------------------

def schedule(pack_m: int, k: int, m_start=None, m_step=None) -> list[int]:
    """adaptive.py:45-52."""
    step = m_step if m_step is not None else max(1, pack_m // 8)
    start = m_start if m_start is not None else max(k, pack_m // 8)
    start = min(max(start, k, 1), pack_m)
    out = list(range(start, pack_m + 1, max(1, step)))
    if not out or out[-1] != pack_m:
        out.append(pack_m)
    return out


def label_subset(k: int, grid_extents=None, stride: int = DEFAULT_STRIDE) -> np.ndarray:
    """adaptive.py:54-62: strided sub-grid of displacement labels."""
    if grid_extents is None or stride == 1:
        return np.arange(k)
    coords = [np.arange(0, n, stride) for n in grid_extents]
    mesh = np.meshgrid(*coords, indexing="ij")
    strides = np.cumprod([1, *grid_extents[:-1]])
    flat = sum(c * st for c, st in zip(mesh, strides))
    return np.sort(flat.ravel())


def seed_fit(q_s: np.ndarray, u: np.ndarray, bound: float) -> float:
    """adaptive.py:72-110: min_{|a|<=bound} |Q_s a - u|^2 via thin SVD,
    then ridge bisection (<=200 steps, tol 1e-6*bound) if the bound binds."""
    q_s = np.asarray(q_s, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64).ravel()
    if bound <= 0:
        return float(u @ u)
    uu, sing, _ = np.linalg.svd(q_s, full_matrices=False)
    b = uu.T @ u
    perp = float(u @ u - b @ b)
    keep = sing > max(1e-13 * (sing[0] if sing.size else 0.0), 1e-300)
    sing, bk = sing[keep], b[keep]
    if sing.size == 0:
        return float(u @ u)

    def a2(mu):
        z = sing * bk / (sing ** 2 + mu)
        return float(z @ z)

    if a2(0.0) <= bound ** 2:
        return float(max(perp, 0.0))
    lo, hi = 0.0, float(sing[0] * np.linalg.norm(bk) / bound)
    while a2(hi) > bound ** 2:
        hi *= 2.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if a2(mid) > bound ** 2:
            lo = mid
        else:
            hi = mid
        if abs(np.sqrt(a2(hi)) - bound) <= 1e-6 * bound:
            break
    z = sing * bk / (sing ** 2 + hi)
    resid = bk - sing * z
    return float(max(perp + resid @ resid, 0.0))


def prior_residual(q: np.ndarray, p: np.ndarray, cached=None, cached_m: int = 0):
    """adaptive.py:113-130: r <- r - Q_new (Q_new^T r); returns (|r|^2, r)."""
    q = np.asarray(q, dtype=np.float64)
    if cached is not None:
        r = np.array(cached, dtype=np.float64, copy=True)
        fresh = q[:, cached_m:]
    else:
        r = np.array(p, dtype=np.float64, copy=True)
        fresh = q
    if fresh.shape[1]:
        r -= fresh @ (fresh.T @ r)
    return float(r @ r), r


def select_m(vectors, d_sqrt, seed_idx, seed_lab, k: int, priors=None,
             epsilon: float = DEFAULT_EPSILON, stride: int = DEFAULT_STRIDE,
             m_start=None, m_step=None, grid_extents=None):
    """adaptive.py:133-185.  Returns (m_use, info)."""
    d_sqrt = np.asarray(d_sqrt, dtype=np.float64)
    n = d_sqrt.size
    bound = float(np.sqrt(np.sum(d_sqrt ** 2)))
    s_idx, s_lab = sorted_seeds(seed_idx, seed_lab, n)
    pack_m = vectors.shape[1]
    u_s_hat = None
    if s_idx.size:
        onehot = np.zeros((s_idx.size, k))
        onehot[np.arange(s_idx.size), s_lab] = 1.0
        u_s_hat = onehot * d_sqrt[s_idx, None]
    tl = np.arange(0)
    p_hat = None
    if priors is not None:
        tl = label_subset(k, grid_extents, stride)
        p_hat = np.asarray(priors, dtype=np.float64)[:, tl] * d_sqrt[:, None]
    f_max = s_idx.size * epsilon ** 2
    g_max = n * epsilon ** 2
    resid = [None] * tl.size
    cached_m = 0
    info = {"steps": [], "saturated": False}
    for m in schedule(pack_m, k, m_start, m_step):
        step = {"m": m, "f": [], "g": []}
        ok = True
        if u_s_hat is not None:
            q_s = np.asarray(vectors[s_idx, :m], dtype=np.float64)
            for col in range(k):
                f = seed_fit(q_s, u_s_hat[:, col], bound)
                step["f"].append(f)
                ok = ok and f <= f_max
        if p_hat is not None:
            qm = np.asarray(vectors[:, :m], dtype=np.float64)
            for j in range(tl.size):
                gval, resid[j] = prior_residual(qm, p_hat[:, j], resid[j], cached_m)
                step["g"].append(gval)
                ok = ok and gval <= g_max
        cached_m = m
        info["steps"].append(step)
        if ok:
            return m, info
    info["saturated"] = True
    return pack_m, info


def nearest_beta(betas, new_beta: float) -> int:
    """refresh.py:91-96: index of the pack nearest on a log scale."""
    import math

    def dist(b):
        if b <= 0 or new_beta <= 0:
            return abs(b - new_beta)
        return abs(math.log(new_beta) - math.log(b))
    best = min(range(len(betas)), key=lambda i: dist(betas[i]))
    return best


# ---------------------------------------------------------------------------
# registration data term (registration.py:27-136)
# ---------------------------------------------------------------------------

def grid_vectors(extents, step: int = 1) -> np.ndarray:
    """registration.py:44-48: displacement table, x offset fastest."""
    extents = tuple(int(e) for e in extents)
    k = int(np.prod(extents))
    out = np.empty((k, len(extents)), dtype=np.int64)
    rem = np.arange(k)
    for a, e in enumerate(extents):
        out[:, a] = rem % e
        rem = rem // e
    return (out - np.array([(e - 1) // 2 for e in extents])) * step


def similarity_priors(fixed, moving, dims, vectors, patch_radius: int = 2):
    """registration.py:95-129: returns (priors N x K, sigma)."""
    dims = tuple(dims)
    d = len(dims)
    f = np.asarray(fixed, dtype=np.float64).reshape(dims, order="F")
    m = np.asarray(moving, dtype=np.float64).reshape(dims, order="F")

    def shifted(g, off):
        out = g
        for axis, o in enumerate(off):
            idx = np.clip(np.arange(g.shape[axis]) + int(o), 0, g.shape[axis] - 1)
            out = np.take(out, idx, axis=axis)
        return out

    offs = np.stack(np.meshgrid(*([np.arange(-patch_radius, patch_radius + 1)] * d), indexing="ij"),
                    axis=-1).reshape(-1, d)
    scores = np.empty((f.size, len(vectors)))
    for k, disp in enumerate(vectors):
        acc = np.zeros(dims)
        for off in offs:
            acc += np.abs(shifted(f, off) - shifted(m, off + disp))
        scores[:, k] = (acc / len(offs)).reshape(-1, order="F")
    sigma = max(scores.min(axis=1).mean(), 1e-8)
    logits = -((scores / sigma) ** 2)
    logits -= logits.max(axis=1, keepdims=True)
    vals = np.exp(logits)
    vals /= vals.sum(axis=1, keepdims=True)
    return vals, sigma


# ---------------------------------------------------------------------------
# super-vertex aggregation (aggregation.py:89-216)
# ---------------------------------------------------------------------------

def build_aggregation(priors, dims, max_cluster_radius: int, similarity_tol: float):
    """aggregation.py:89-127: greedy BFS region growing in flat index order.
    Returns (cluster_ids int64 (N,), n_super)."""
    from collections import deque
    dims = tuple(int(d) for d in dims)
    p = np.asarray(priors, dtype=np.float64)
    n = int(np.prod(dims))
    coords = np.stack(np.unravel_index(np.arange(n), dims, order="F"), axis=1)
    strides = np.cumprod([1, *dims[:-1]])
    cluster = np.full(n, -1, dtype=np.int64)
    nid = 0
    for start in range(n):
        if cluster[start] >= 0:
            continue
        cluster[start] = nid
        ps, cs = p[start], coords[start]
        q = deque([start])
        while q:
            x = q.popleft()
            cx = coords[x]
            for axis in range(len(dims)):
                for step in (-1, 1):
                    if not 0 <= cx[axis] + step < dims[axis]:
                        continue
                    y = x + step * strides[axis]
                    if cluster[y] >= 0:
                        continue
                    if np.abs(coords[y] - cs).max() > max_cluster_radius:
                        continue
                    if np.abs(p[y] - ps).sum() > similarity_tol:
                        continue
                    cluster[y] = nid
                    q.append(y)
        nid += 1
    return cluster, nid


def delta_weights(cluster_ids, dims):
    """aggregation.py:130-139: 2 per lattice neighbour in another cluster."""
    heads, tails = lattice_edges(dims)
    differs = cluster_ids[heads] != cluster_ids[tails]
    delta = np.zeros(int(np.prod(dims)))
    np.add.at(delta, heads[differs], 2.0)
    np.add.at(delta, tails[differs], 2.0)
    return delta


def eta_bar_t(cluster_ids, n_super):
    n = cluster_ids.size
    sizes = np.bincount(cluster_ids, minlength=n_super)
    return sp.csr_matrix((1.0 / sizes[cluster_ids], (cluster_ids, np.arange(n))), shape=(n_super, n))


def gram_schmidt(v, drop_tol: float = 1e-10):
    """linalg.py gram_schmidt: modified Gram-Schmidt, two passes, columns
    with residual norm < drop_tol dropped."""
    v = np.array(v, dtype=np.float64)
    kept = []
    for j in range(v.shape[1]):
        col = v[:, j].copy()
        for _ in range(2):
            for q in kept:
                col -= q @ col * q
        nrm = np.linalg.norm(col)
        if nrm < drop_tol:
            continue
        kept.append(col / nrm)
    return np.column_stack(kept) if kept else np.zeros((v.shape[0], 0))


def coarsen_basis(V, cluster_ids, n_super, intensities, dims, beta, variant="delta", m_use=None):
    """aggregation.py:154-204 -> (q_bar, lambda_bar, d_sqrt_bar, lap_bar)."""
    V = np.asarray(V, dtype=np.float64)
    if m_use is not None:
        V = V[:, :m_use]
    weighted = V * delta_weights(cluster_ids, dims)[:, None] if variant == "delta" else V
    raw = eta_bar_t(cluster_ids, n_super) @ weighted
    if n_super == 1:
        return np.ones((1, 1)), np.zeros(1), np.ones(1), None
    q = gram_schmidt(raw)
    heads, tails = lattice_edges(dims)
    w = edge_weights(np.asarray(intensities, dtype=np.float64), heads, tails, beta)
    wmat = symmetric_weights(cluster_ids.size, heads, tails, w).tocoo()
    ci, cj = cluster_ids[wmat.row], cluster_ids[wmat.col]
    cross = ci != cj
    wbar = sp.coo_matrix((wmat.data[cross], (ci[cross], cj[cross])), shape=(n_super, n_super)).tocsr()
    wbar.sum_duplicates()
    wbar.sort_indices()
    lap = normalized_laplacian(wbar)
    quad = np.einsum("ij,ij->j", q, lap.matrix @ q)
    lam = np.maximum(quad, 0.0)
    order = np.argsort(lam, kind="stable")
    return q[:, order], lam[order], lap.d_sqrt, lap


def aggregate_priors(priors, cluster_ids, n_super):
    """aggregation.py:207-209."""
    return eta_bar_t(cluster_ids, n_super) @ np.asarray(priors, dtype=np.float64)
