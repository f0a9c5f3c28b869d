"""Offline precompute on the GPU: the m smallest eigenpairs
of the normalised Laplacian, as a device pack ready for update_basis /
solve_fast.

Reference: ``precompute`` fastrw.py:200-221 (graph -> smallest_eigs ->
_snap_null_vector), ``smallest_eigs`` linalg.py:98-175 (block shift-invert
Krylov with a sparse LU, eigh Rayleigh-Ritz, residual test
||L y - theta y|| <= eig_tol * max(1, |theta|), NotConverged with the
converged prefix), ``_canonical_signs`` linalg.py:90-95,
``_snap_null_vector`` fastrw.py:180-197.

The reference's sparse LU is infeasible in 3-D (SURVEY finding: splu 64^3 =
796 s), so the GPU path replaces shift-invert Krylov by Chebyshev-filtered
subspace iteration, which needs only the operator:

  * filter: p_d(L^) X by the scaled three-term Chebyshev recurrence on the
    damped interval [a, 2] (a = the block's largest Ritz value, 2 >= the
    normalised-Laplacian spectrum), each step one fused stencil pass
    (swb_stencil_apply: out = a L^ Y + b Y + g Z);
  * orthonormalise: CholeskyQR2 with the DMMA Gram / NN GEMMs (shifted
    CholeskyQR3 if the Gram is not numerically definite);
  * Rayleigh-Ritz: H = X^T L^ X (stencil + symmetric DMMA projection), a
    k x k symmetric eigendecomposition, X <- X Z and L^X <- (L^X) Z;
  * the reference residual test on the first m Ritz pairs
    (swb_ritz_residuals), then canonical signs and the null-vector snap.
The block carries k = m + guard vectors (guard columns speed convergence of
the m-th pair).  Only k x k matrices leave the N-length kernels.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib
from .device import (WORKSPACE, DeviceGraph, DevicePack, LatticeSpec, ptr, require_cuda, round_up,
                     stream_handle)
from .errors import InvalidParam, NotConverged
from .types import PackProvenance

# reference constants (fastrw.py:36,39; linalg.py:21)
M_CAP = 4096
NULL_EIG_SNAP = 1e-3
EIG_TOL = 1e-6
SPECTRUM_TOP = 2.0   # lambda_max(L^) <= 2 for a normalised Laplacian


class _Op:
    """L^ on row-major N x k device blocks through the stencil apply pass."""

    def __init__(self, graph: DeviceGraph, k: int):
        self.graph = graph
        self.n = graph.lattice.n
        self.k = k
        self.lat = graph.lattice.c_struct()
        self.ws = WORKSPACE.get("stencil_apply", _lib.size("swb_stencil_workspace_bytes", C.byref(self.lat), k))
        self.applies = 0

    def __call__(self, X, out, a=1.0, b=0.0, Z=None, g=0.0):
        g_ = self.graph
        _lib.call("swb_stencil_apply", C.byref(self.lat), ptr(X), X.shape[1], 0, 0, self.n, self.k, ptr(g_.what),
                  ptr(g_.diag), ptr(g_.d_sqrt_dev), float(a), float(b), ptr(Z), Z.shape[1] if Z is not None else 0,
                  float(g), ptr(out), out.shape[1], None, None, ptr(self.ws), self.ws.numel(), stream_handle())
        self.applies += 1


def _gram(X, k):
    torch = require_cuda()
    ldg = round_up(k, 2)
    G = torch.empty((k, ldg), dtype=torch.float64, device="cuda")
    ws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", X.shape[0], k, k))
    _lib.call("swb_gemm_tn", ptr(X), X.shape[1], ptr(X), X.shape[1], X.shape[0], k, k, 1, ptr(G), ldg, ptr(ws),
              ws.numel(), stream_handle())
    return G


def _project(X, Y, k):
    """X^T Y (symmetric by construction: Y = L^ X)."""
    torch = require_cuda()
    ldg = round_up(k, 2)
    H = torch.empty((k, ldg), dtype=torch.float64, device="cuda")
    ws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", X.shape[0], k, k))
    _lib.call("swb_gemm_tn", ptr(X), X.shape[1], ptr(Y), Y.shape[1], X.shape[0], k, k, 1, ptr(H), ldg, ptr(ws),
              ws.numel(), stream_handle())
    return H[:, :k]


def _times(X, k, S, out):
    """out[:, :k] = X[:, :k] S (S k x k, DMMA NN)."""
    torch = require_cuda()
    ldb = round_up(k, 2)
    B = torch.zeros((k, ldb), dtype=torch.float64, device="cuda")
    B[:, :k] = S
    _lib.call("swb_gemm_nn", ptr(X), X.shape[1], ptr(B), ldb, X.shape[0], k, k, ptr(out), out.shape[1], 0,
              stream_handle())


def _orthonormalize(X, W, k):
    """CholeskyQR2 of X[:, :k] (result in X; W scratch).  Falls back to a
    shifted first pass (CholeskyQR3) when the Gram is not definite."""
    torch = require_cuda()
    eye = torch.eye(k, dtype=torch.float64, device="cuda")
    passes = 2
    i = 0
    while i < passes:
        G = _gram(X, k)[:, :k]
        R, info = torch.linalg.cholesky_ex(G, upper=True)
        if int(info.item()) != 0:
            # shifted CholeskyQR: G + s I is definite; two more passes follow
            s = 11.0 * (X.shape[0] * k + k * (k + 1)) * np.finfo(np.float64).eps * float(torch.trace(G).item())
            R = torch.linalg.cholesky(G + s * eye, upper=True)
            passes = i + 3
        Rinv = torch.linalg.solve_triangular(R, eye, upper=True)
        _times(X, k, Rinv, W)
        X[:, :k].copy_(W[:, :k])
        i += 1


def _rayleigh_ritz(op, X, Y, W, k):
    """X <- X Z, Y <- L^ X (rotated); returns ascending Ritz values."""
    torch = require_cuda()
    op(X, Y)
    H = _project(X, Y, k)
    H = 0.5 * (H + H.T)
    theta, Z = torch.linalg.eigh(H)
    _times(X, k, Z, W)
    X[:, :k].copy_(W[:, :k])
    _times(Y, k, Z, W)
    Y[:, :k].copy_(W[:, :k])
    return theta


def _residuals(X, Y, theta, k):
    torch = require_cuda()
    res2 = torch.empty(k, dtype=torch.float64, device="cuda")
    ws = WORKSPACE.get("columns", _lib.size("swb_column_workspace_bytes", k))
    _lib.call("swb_ritz_residuals", ptr(X), X.shape[1], ptr(Y), Y.shape[1], ptr(theta.contiguous()), X.shape[0], k,
              ptr(res2), ptr(ws), ws.numel(), stream_handle())
    return torch.sqrt(torch.clamp(res2, min=0.0))


def _chebyshev(op, X, Y, W, a, b, a0, degree):
    """p_d(L^) X with p damping [a, b] (scaled recurrence); result returned
    as one of the three buffers (the others are scratch)."""
    e = (b - a) / 2.0
    c = (b + a) / 2.0
    sigma = e / (a0 - c)
    tau = 2.0 / sigma
    x0, y1, y2 = X, Y, W
    op(x0, y1, a=sigma / e, b=-c * sigma / e)
    for _ in range(2, degree + 1):
        sig_new = 1.0 / (tau - sigma)
        op(y1, y2, a=2.0 * sig_new / e, b=-2.0 * sig_new * c / e, Z=x0, g=-sigma * sig_new)
        x0, y1, y2 = y1, y2, x0
        sigma = sig_new
    return y1, x0, y2


def _null_snap(V, m, values, d_sqrt_dev, dnorm):
    """_snap_null_vector (fastrw.py:180-197) on the device basis."""
    torch = require_cuda()
    if values[0] > NULL_EIG_SNAP:
        return values
    values = values.copy()
    g = d_sqrt_dev / dnorm
    V[:, 0].copy_(g)
    values[0] = 0.0
    if m > 1:
        rest = V[:, 1:]
        ws = WORKSPACE.get("columns", _lib.size("swb_column_workspace_bytes", m - 1))
        h = torch.empty(m - 1, dtype=torch.float64, device="cuda")
        st = stream_handle()
        for _ in range(2):
            _lib.call("swb_column_dots", ptr(rest), V.shape[1], ptr(g), V.shape[0], m - 1, ptr(h), ptr(ws),
                      ws.numel(), st)
            _lib.call("swb_column_update", ptr(rest), V.shape[1], V.shape[0], m - 1, ptr(g), ptr(h), None, st)
        _lib.call("swb_column_dots", ptr(rest), V.shape[1], None, V.shape[0], m - 1, ptr(h), ptr(ws), ws.numel(), st)
        scale = 1.0 / torch.sqrt(h)
        _lib.call("swb_column_update", ptr(rest), V.shape[1], V.shape[0], m - 1, None, None, ptr(scale), st)
    return values


def smallest_eigs_device(graph: DeviceGraph, m: int, eig_tol: float = EIG_TOL, seed: int = 0, *,
                         guard: int | None = None, degree: int = 24, max_iter: int = 400):
    """m smallest eigenpairs of L^ (graph) -> (V N x round_up(m, 8) device,
    values host, info).  Raises NotConverged (partial = (V, values) prefix)
    at the iteration cap, like smallest_eigs (linalg.py:160-166)."""
    torch = require_cuda()
    n = graph.lattice.n
    if not 1 <= m <= n:
        raise InvalidParam(f"need 1 <= m <= {n}, got {m}")
    if guard is None:
        guard = max(8, m // 8)
    k = min(n, m + guard)
    ldk = round_up(k, 8)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(int(seed))
    X = torch.zeros((n, ldk), dtype=torch.float64, device="cuda")
    X[:, :k].normal_(generator=gen)
    Y = torch.zeros_like(X)
    W = torch.zeros_like(X)
    op = _Op(graph, k)
    _orthonormalize(X, W, k)
    theta = _rayleigh_ritz(op, X, Y, W, k)
    it = 0
    history = []
    converged = 0
    while True:
        res = _residuals(X, Y, theta, k)
        th = theta.cpu().numpy()
        r = res.cpu().numpy()
        ok = r[:m] <= eig_tol * np.maximum(1.0, np.abs(th[:m]))
        converged = m if ok.all() else int(np.argmin(ok))
        history.append((it, converged, float(r[:m].max())))
        if converged >= m or k >= n and it > 0:
            break
        if it >= max_iter:
            break
        # damp [theta_k, 2]; amplify below (scaled Chebyshev, Zhou & Saad)
        a = float(th[k - 1])
        a0 = min(float(th[0]), a - 1e-12)
        out, s1, s2 = _chebyshev(op, X, Y, W, a, SPECTRUM_TOP, a0, degree)
        X, Y, W = out, s1, s2
        _orthonormalize(X, W, k)
        theta = _rayleigh_ritz(op, X, Y, W, k)
        it += 1
    info = {"iterations": it, "k": k, "degree": degree, "applies": op.applies, "history": history}
    take = m if converged >= m else converged
    values = theta.cpu().numpy()[:take].copy()
    # the Ritz block becomes the pack's basis in place (its leading dimension
    # stays round_up(k, 8); columns >= take are zeroed): at BASELINE scale the
    # three N x k blocks already fill most of HBM
    del Y, W
    V = X
    V[:, take:].zero_()
    if take:
        ws = WORKSPACE.get("columns", _lib.size("swb_column_workspace_bytes", take))
        _lib.call("swb_canonical_signs", ptr(V), V.shape[1], n, take, ptr(ws), ws.numel(), stream_handle())
    if converged < m:
        raise NotConverged(f"only {converged}/{m} eigenpairs converged (iteration cap {max_iter})",
                           partial=(V, values), converged=converged)
    return V, values, info


def precompute(image, beta: float, m: int, eig_tol: float = EIG_TOL, seed: int = 0, *, connectivity=None,
               weight_mode: str = "abs", guard: int | None = None, degree: int = 24,
               max_iter: int = 400) -> DevicePack:
    """precompute (fastrw.py:200-221) on the GPU -> DevicePack.  A
    NotConverged run keeps the converged prefix (with a warning), as the
    reference does."""
    import warnings

    from .api import image_device, image_hash
    torch = require_cuda()
    n = image.n_voxels if hasattr(image, "n_voxels") else int(np.prod(image.dims))
    if not 1 <= m <= min(n, M_CAP):
        raise InvalidParam(f"need 1 <= m <= min(N, {M_CAP}), got {m}")
    lattice = LatticeSpec.make(tuple(image.dims), connectivity, weight_mode)
    img_dev = image_device(image)
    graph = DeviceGraph.build(img_dev, lattice, beta)
    try:
        V, values, info = smallest_eigs_device(graph, m, eig_tol, seed, guard=guard, degree=degree,
                                               max_iter=max_iter)
    except NotConverged as exc:
        V, values = exc.partial
        if len(values) == 0:
            raise
        warnings.warn(f"eigensolver converged {exc.converged} of {m} pairs; pack truncated")
        info = {"converged": exc.converged}
    mm = len(values)
    values = _null_snap(V, mm, values, graph.d_sqrt_dev, graph.dnorm)
    prov = PackProvenance(image_hash=image_hash(image), eig_tol=eig_tol, built_at=time.time())
    pack = DevicePack(V, mm, torch.from_numpy(values).to("cuda"), graph.d_sqrt_dev, graph.dnorm, tuple(image.dims),
                      tuple(getattr(image, "spacing", ()) or ()), float(beta), prov, lattice, image_dev=img_dev,
                      graph=graph)
    pack.solver_info = info
    return pack
