"""Super-vertex aggregation and eigenvector coarsening on the GPU (SURVEY
§8f #4; reference aggregation.py:28-216).

  build_aggregation   aggregation.py:89-127  -> swb_build_aggregation
                      (native, sequential by definition: flat scan order +
                      FIFO BFS; numpy pairwise L1 so decisions match exactly)
  delta_weights       aggregation.py:130-139 -> swb_delta_weights (GPU)
  coarsen_basis       aggregation.py:154-204: eta_bar^T (delta V) by
                      swb_cluster_rows, two-pass Gram-Schmidt on the DMMA
                      GEMMs, the aggregate Laplacian, re-valued columns by
                      the aggregate Rayleigh quotients (swb_csr_spmm +
                      swb_column_products), stable sort
  aggregate_priors    aggregation.py:207-209 -> swb_cluster_rows
  propagate           aggregation.py:212-219 -> swb_gather_rows

The aggregate graph itself (N-bar super-vertices, irregular) is assembled on
the host from the GPU's raw lattice edge weights with the reference's own
sparse-assembly order (coo -> csr, sum duplicates, normalised Laplacian), so
the coarse Laplacian matches the reference's to the last ulp of the edge
weights' exp(); every N-length and N-bar x m operation runs on the GPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from .device import WORKSPACE, DevicePack, LatticeSpec, ptr, require_cuda, round_up, stream_handle
from .errors import DegenerateGraph, DimsMismatch, EmptyBasis, InvalidParam
from .types import PackProvenance, ProbabilityField, num_voxels

GS_DROP_TOL = 1e-10   # linalg.py:23


class CoarsenVariant(Enum):
    NAIVE = "naive"
    DELTA = "delta"


@dataclass(frozen=True)
class Aggregation:
    """Hard assignment of voxels to super-vertices (aggregation.py:34-57)."""

    dims: tuple
    cluster_ids: np.ndarray
    n_super: int

    @property
    def sizes(self) -> np.ndarray:
        return np.bincount(self.cluster_ids, minlength=self.n_super)

    def device(self):
        """(cluster ids int32, member order int64, offsets int64) on the GPU, cached."""
        cache = self.__dict__.get("_dev")
        if cache is None:
            torch = require_cuda()
            order = np.argsort(self.cluster_ids, kind="stable")
            off = np.zeros(self.n_super + 1, dtype=np.int64)
            np.cumsum(self.sizes, out=off[1:])
            cache = (torch.from_numpy(self.cluster_ids.astype(np.int32)).to("cuda"),
                     torch.from_numpy(order.astype(np.int64)).to("cuda"), torch.from_numpy(off).to("cuda"))
            object.__setattr__(self, "_dev", cache)
        return cache


@dataclass
class CoarseBasis:
    """aggregation.py:60-71 (q_bar on the device; host view on demand)."""

    q_bar_dev: object
    lambda_bar: np.ndarray
    delta: object
    variant: CoarsenVariant

    @property
    def m(self) -> int:
        return self.lambda_bar.size

    @property
    def q_bar(self) -> np.ndarray:
        return self.q_bar_dev[:, :self.m].cpu().numpy()


class CoarseLaplacian:
    """Reference Laplacian surface of the aggregate graph (host CSR)."""

    def __init__(self, matrix, d_sqrt):
        self.matrix = matrix
        self.d_sqrt = d_sqrt

    @property
    def n_vertices(self) -> int:
        return self.matrix.shape[0]

    @property
    def mode(self):
        from .types import LaplacianMode
        return LaplacianMode.NORMALIZED


class PropagatedField:
    """Voxel probabilities copied from super-vertex rows (device)."""

    def __init__(self, dims, U_dev, k):
        self.dims = tuple(dims)
        self.U_dev = U_dev
        self._k = k

    @property
    def K(self) -> int:
        return self._k

    def _u(self):
        return self.U_dev

    @property
    def values(self) -> np.ndarray:
        return self.U_dev[:, :self._k].cpu().numpy()

    def field(self) -> ProbabilityField:
        return ProbabilityField(self.dims, self.values)


def _priors_host(priors):
    if hasattr(priors, "values_dev"):
        return priors.values_dev.cpu().numpy(), tuple(priors.dims)
    return np.ascontiguousarray(priors.values, dtype=np.float64), tuple(priors.dims)


def build_aggregation(priors, max_cluster_radius: int, similarity_tol: float) -> Aggregation:
    """aggregation.py:89-127 (priors: ProbabilityField / DevicePriors)."""
    p, dims = _priors_host(priors)
    n = num_voxels(dims)
    if p.shape[0] != n:
        raise DimsMismatch("prior rows do not match dims")
    cid = np.empty(n, dtype=np.int32)
    ns = C.c_int64(0)
    d = np.asarray(dims, dtype=np.int64)
    _lib.call("swb_build_aggregation", p.ctypes.data, p.shape[1], p.shape[1], d.ctypes.data, len(dims),
              int(max_cluster_radius), float(similarity_tol), cid.ctypes.data, C.byref(ns))
    return Aggregation(dims=dims, cluster_ids=cid.astype(np.int64), n_super=int(ns.value))


def delta_weights(agg: Aggregation, dims=None):
    """aggregation.py:130-139 on the GPU (the default-connectivity lattice of
    the aggregation's dims, like the reference's lattice_edges(dims))."""
    torch = require_cuda()
    if dims is not None and tuple(dims) != agg.dims:
        raise DimsMismatch("aggregation and graph dims differ")
    cid, _, _ = agg.device()
    lat = LatticeSpec.make(agg.dims).c_struct()
    out = torch.empty(num_voxels(agg.dims), dtype=torch.float64, device="cuda")
    _lib.call("swb_delta_weights", C.byref(lat), ptr(cid), ptr(out), stream_handle())
    return out


def _cluster_rows(agg: Aggregation, X, m, w=None):
    torch = require_cuda()
    _, order, off = agg.device()
    out = torch.zeros((agg.n_super, round_up(m, 2)), dtype=torch.float64, device="cuda")
    _lib.call("swb_cluster_rows", ptr(X), X.stride(0), m, ptr(w), ptr(order), ptr(off), agg.n_super, ptr(out),
              out.shape[1], stream_handle())
    return out


def _copy_column(src, j, dst, k):
    """dst[:, k] = src[:, j] (device column copy through swb_gather_columns)."""
    torch = require_cuda()
    cmap = torch.tensor([j], dtype=torch.int32, device="cuda")
    view = dst[:, k:]
    _lib.call("swb_gather_columns", ptr(src), src.stride(0), src.shape[0], ptr(cmap), 1, ptr(view), dst.stride(0),
              stream_handle())


def _gram_schmidt(raw, m):
    """Two-pass Gram-Schmidt (linalg.py gram_schmidt) on the device:
    each column is orthogonalised twice against the kept ones (DMMA TN + NN),
    dropped if its norm falls below GS_DROP_TOL, else normalised."""
    torch = require_cuda()
    nb = raw.shape[0]
    ldq = round_up(max(m, 1), 8)
    Q = torch.zeros((nb, ldq), dtype=torch.float64, device="cuda")
    col = torch.zeros((nb, 2), dtype=torch.float64, device="cuda")
    h = torch.zeros((ldq, 2), dtype=torch.float64, device="cuda")
    nrm2 = torch.empty(1, dtype=torch.float64, device="cuda")
    st = stream_handle()
    cws = WORKSPACE.get("columns", _lib.size("swb_column_workspace_bytes", 1))
    nk = 0
    for j in range(m):
        _copy_column(raw, j, col, 0)
        for _ in range(2):
            if nk:
                tws = WORKSPACE.get("gemm_tn_gs", _lib.size("swb_gemm_tn_workspace_bytes", nb, nk, 1))
                _lib.call("swb_gemm_tn", ptr(Q), ldq, ptr(col), 2, nb, nk, 1, 0, ptr(h), 2, ptr(tws), tws.numel(), st)
                _lib.call("swb_gemm_nn_ex", ptr(Q), ldq, ptr(h), 2, nb, nk, 1, ptr(col), 2, 1, -1.0, st)
        _lib.call("swb_column_dots", ptr(col), 2, None, nb, 1, ptr(nrm2), ptr(cws), cws.numel(), st)
        nrm = float(np.sqrt(nrm2.item()))
        if nrm < GS_DROP_TOL:
            continue
        scale = torch.full((1,), 1.0 / nrm, dtype=torch.float64, device="cuda")
        _lib.call("swb_column_update", ptr(col), 2, nb, 1, None, None, ptr(scale), st)
        _copy_column(col, 0, Q, nk)
        nk += 1
    return Q, nk


def _symmetric_lattice_weights(w, lattice: LatticeSpec):
    """Host CSR of the lattice weight matrix in the reference construction
    order (graphs.py:116-124): per direction the forward entries, then the
    mirrored ones, coo -> csr."""
    import scipy.sparse as sp
    n = lattice.n
    dims = lattice.dims
    nd = len(dims)
    grid = np.arange(n, dtype=np.int64).reshape(dims, order="F")
    heads, tails, vals = [], [], []
    wv = w.reshape(n, lattice.ndir)
    for d, off in enumerate(lattice.forward_offsets()):
        src = [slice(None)] * nd
        dst = [slice(None)] * nd
        for ax, o in enumerate(off):
            if o > 0:
                src[ax], dst[ax] = slice(None, -o), slice(o, None)
            elif o < 0:
                src[ax], dst[ax] = slice(-o, None), slice(None, o)
        h = grid[tuple(src)].ravel(order="F")
        heads.append(h)
        tails.append(grid[tuple(dst)].ravel(order="F"))
        vals.append(wv[h, d])
    heads, tails, vals = np.concatenate(heads), np.concatenate(tails), np.concatenate(vals)
    mat = sp.coo_matrix((np.concatenate([vals, vals]), (np.concatenate([heads, tails]),
                                                        np.concatenate([tails, heads]))), shape=(n, n)).tocsr()
    mat.sort_indices()
    return mat


def _normalized_laplacian(weights):
    """laplacian_from_weights, NORMALIZED branch (graphs.py:143-159)."""
    import scipy.sparse as sp
    weights = weights.tocsr()
    deg = np.asarray(weights.sum(axis=1)).ravel()
    if np.any(deg <= 0):
        raise DegenerateGraph("aggregate graph has an isolated super-vertex")
    d_sqrt = np.sqrt(deg)
    inv = sp.diags(1.0 / d_sqrt)
    mat = (inv @ (sp.diags(deg) - weights) @ inv).tocsr()
    mat = ((mat + mat.T) * 0.5).tocsr()
    mat.sort_indices()
    return mat, d_sqrt


def _edge_weights_device(pack, image=None, beta=None):
    torch = require_cuda()
    from .api import image_device
    dims = tuple(pack.dims)
    lattice = LatticeSpec.make(dims)     # build_graph defaults: 4 / 6-connectivity, |dI| weights
    img = image_device(image) if image is not None else pack.image_dev
    if img is None:
        raise InvalidParam("coarsen_basis needs the pack's image (pass image=)")
    b = float(pack.beta if beta is None else beta)
    w = torch.empty(lattice.n * lattice.ndir, dtype=torch.float64, device="cuda")
    _lib.call("swb_edge_weights", C.byref(lattice.c_struct()), ptr(img), b, None, ptr(w), stream_handle())
    return w.cpu().numpy(), lattice


def coarsen_basis(pack, agg: Aggregation, graph=None, variant: CoarsenVariant = CoarsenVariant.DELTA,
                  m_use: int | None = None, *, image=None):
    """aggregation.py:154-204 -> (CoarseBasis, coarse DevicePack).

    ``graph``: a reference WeightedLatticeGraph (its host weights are used),
    or None (raw edge weights recomputed on the GPU from the pack's image at
    the pack's beta, as build_graph(image, beta=pack.beta) would)."""
    import scipy.sparse as sp
    torch = require_cuda()
    from .api import _as_device
    if tuple(agg.dims) != tuple(pack.dims):
        raise DimsMismatch("aggregation and pack dims differ")
    dp = _as_device(pack)
    m = dp.m if m_use is None else int(m_use)
    if not 1 <= m <= dp.m:
        raise InvalidParam(f"m_use must be in 1..{dp.m}")
    V = dp.V
    if dp.col_map is not None:   # pack column order (RefreshedPack / UpdatedPack)
        Vc = torch.empty((V.shape[0], round_up(m, 2)), dtype=torch.float64, device="cuda")
        _lib.call("swb_gather_columns", ptr(V), dp.ldv, V.shape[0], ptr(dp.col_map), m, ptr(Vc), Vc.shape[1],
                  stream_handle())
        V = Vc
    delta = delta_weights(agg) if variant is CoarsenVariant.DELTA else None
    raw = _cluster_rows(agg, V, m, delta)
    if agg.n_super == 1:
        q = torch.ones((1, 2), dtype=torch.float64, device="cuda")
        lam = np.zeros(1)
        basis = CoarseBasis(q, lam, delta, variant)
        coarse = DevicePack(q, 1, torch.zeros(1, dtype=torch.float64, device="cuda"),
                            torch.ones(1, dtype=torch.float64, device="cuda"), 1.0, (1,), (), dp.beta,
                            PackProvenance(image_hash=b""), None)
        coarse.laplacian = None
        return basis, coarse
    Q, mk = _gram_schmidt(raw, m)
    if mk == 0:
        raise EmptyBasis("all coarsened columns collapsed to zero")
    # aggregate graph: crossing-edge weight sums (aggregation.py:142-151)
    if graph is not None and hasattr(graph, "weights"):
        wmat = graph.weights.tocoo()
    else:
        w, lattice = _edge_weights_device(dp, image)
        wmat = _symmetric_lattice_weights(w, lattice).tocoo()
    cid = agg.cluster_ids
    ci, cj = cid[wmat.row], cid[wmat.col]
    crossing = ci != cj
    w_bar = sp.coo_matrix((wmat.data[crossing], (ci[crossing], cj[crossing])),
                          shape=(agg.n_super, agg.n_super)).tocsr()
    w_bar.sum_duplicates()
    w_bar.sort_indices()
    lap, d_sqrt = _normalized_laplacian(w_bar)
    # aggregate Rayleigh quotients of the unit-norm columns, on the GPU
    ip = torch.from_numpy(lap.indptr.astype(np.int64)).to("cuda")
    ix = torch.from_numpy(lap.indices.astype(np.int64)).to("cuda")
    dv = torch.from_numpy(lap.data.astype(np.float64)).to("cuda")
    LQ = torch.empty_like(Q)
    st = stream_handle()
    _lib.call("swb_csr_spmm", ptr(ip), ptr(ix), ptr(dv), agg.n_super, ptr(Q), Q.shape[1], mk, ptr(LQ), LQ.shape[1], st)
    quad = torch.empty(mk, dtype=torch.float64, device="cuda")
    cws = WORKSPACE.get("columns", _lib.size("swb_column_workspace_bytes", mk))
    _lib.call("swb_column_products", ptr(Q), Q.shape[1], ptr(LQ), LQ.shape[1], agg.n_super, mk, ptr(quad), ptr(cws),
              cws.numel(), st)
    lam = np.maximum(quad.cpu().numpy(), 0.0)
    order = np.argsort(lam, kind="stable")
    lam = lam[order]
    Qs = torch.zeros((agg.n_super, round_up(mk, 8)), dtype=torch.float64, device="cuda")
    cmap = torch.from_numpy(order.astype(np.int32)).to("cuda")
    _lib.call("swb_gather_columns", ptr(Q), Q.shape[1], agg.n_super, ptr(cmap), mk, ptr(Qs), Qs.shape[1], st)
    d_dev = torch.from_numpy(d_sqrt.copy()).to("cuda")
    basis = CoarseBasis(Qs, lam, delta, variant)
    coarse = DevicePack(Qs, mk, torch.from_numpy(lam.copy()).to("cuda"), d_dev, float(np.linalg.norm(d_sqrt)),
                        (agg.n_super,), (), dp.beta, PackProvenance(image_hash=b""), None)
    coarse.laplacian = CoarseLaplacian(lap, d_sqrt)
    return basis, coarse


def aggregate_priors(priors, agg: Aggregation):
    """aggregation.py:207-209: mean prior row per super-vertex (device N-bar x L)."""
    torch = require_cuda()
    if hasattr(priors, "values_dev"):
        P = priors.values_dev
    elif hasattr(priors, "is_cuda"):
        P = priors
    else:
        P = torch.from_numpy(np.array(getattr(priors, "values", priors), dtype=np.float64)).to("cuda")
    k = P.shape[1]
    return _cluster_rows(agg, P.contiguous(), k)[:, :k]


def propagate(u_bar, agg: Aggregation) -> PropagatedField:
    """aggregation.py:212-219: copy each super-vertex row to its voxels."""
    torch = require_cuda()
    if hasattr(u_bar, "_u"):
        U = u_bar._u()
        k = u_bar.K
    elif hasattr(u_bar, "is_cuda"):
        U, k = u_bar, u_bar.shape[1]
    else:
        arr = np.asarray(u_bar, dtype=np.float64)
        U, k = torch.from_numpy(arr).to("cuda"), arr.shape[1]
    if U.shape[0] != agg.n_super:
        raise DimsMismatch("row count does not match the super-vertex count")
    sums = U[:, :k].sum(dim=1)
    if not bool(torch.all(torch.abs(sums - 1.0) <= 1e-6)):
        raise InvalidParam("aggregate rows must sum to 1 within 1e-6")
    cid, _, _ = agg.device()
    n = cid.numel()
    out = torch.empty((n, round_up(k, 2)), dtype=torch.float64, device="cuda")
    Uc = U if U.stride(1) == 1 else U.contiguous()
    _lib.call("swb_gather_rows", ptr(Uc), Uc.stride(0), ptr(cid), n, k, ptr(out), out.shape[1], stream_handle())
    return PropagatedField(agg.dims, out, k)
