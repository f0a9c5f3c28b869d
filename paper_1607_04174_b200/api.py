"""Public hot-path API — the drop-in for the reference's online path.

Same names, argument meaning and error behaviour as the reference:

  refresh(pack, image, new_beta)            refresh.py:63-82
  refresh_from_set(packs, image, new_beta)  refresh.py:85-88
  nearest_pack(packs, new_beta)             refresh.py:91-96
  solve_fast(pack, lap, prob, m_use=None)   fastrw.py:352-467
  hard_labels(field)                        images.py:128-130
  update_basis(pack, image, new_beta, cut_edges, method, gap_guard)
                                            north-star "update-basis" (new)

Every numeric step runs in libspecwalk_b200.so on the current CUDA stream;
results stay on the device and are materialised on the host only when a
caller reads a host attribute (``.values``, ``.labels``, ``.eigen`` ...).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import weakref

import numpy as np

from . import _lib
from .device import (CAPTURE, WORKSPACE, DeviceGraph, DevicePack, LatticeSpec, gather_vector, oz_full_workspace, ptr,
                     rotate_rows,
                     require_cuda, round_up, stream_handle, to_device, torch_mod)
from .errors import (ImageMismatch, InsufficientBasis, InvalidParam, SingularSmallSystem)
from .types import MAX_SEEDS, LabelMap, LaplacianMode, ProbabilityField, content_hash

# ---------------------------------------------------------------------------
# optional phase timing (CUDA events on the launching stream; bench.py)
# ---------------------------------------------------------------------------

class PhaseTimer:
    """Records a CUDA event at each named phase boundary on the current
    stream.  ``durations()`` (after a synchronize) gives per-phase ms."""

    def __init__(self):
        self.marks = []

    def mark(self, name: str):
        torch = torch_mod()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.marks.append((name, ev))

    def durations(self) -> dict:
        out: dict = {}
        for (name, ev), (_, nxt) in zip(self.marks, self.marks[1:]):
            out.setdefault(name, []).append(ev.elapsed_time(nxt))
        return out


TIMER: PhaseTimer | None = None


def _mark(name: str):
    if TIMER is not None:
        TIMER.mark(name)


# ---------------------------------------------------------------------------
# image plumbing (hash check of refresh.py:71-72, device copy cache)
# ---------------------------------------------------------------------------

_image_cache: dict = {}


def _image_entry(image):
    key = id(image)
    ent = _image_cache.get(key)
    if ent is not None and ent[0]() is image:
        return ent
    try:
        ref = weakref.ref(image, lambda _r, k=key: _image_cache.pop(k, None))
    except TypeError:
        ref = lambda: image  # noqa: E731 - non-weakrefable image object
    ent = [ref, None, None]
    _image_cache[key] = ent
    return ent


_seed_cache: dict = {}


def seed_tensors(seeds):
    """Device copies (int64 indices, int32 labels) of a SeedPartition, uploaded
    once per object (weakly cached like the image): a solve with fresh seed
    arrays uploads them; a session replaying the same seeds does not."""
    torch = torch_mod()
    key = id(seeds)
    ent = _seed_cache.get(key)
    if ent is not None and ent[0]() is seeds:
        return ent[1], ent[2]
    sidx = torch.from_numpy(np.ascontiguousarray(seeds.seed_indices, dtype=np.int64)).to("cuda")
    slab = torch.from_numpy(np.ascontiguousarray(seeds.seed_labels, dtype=np.int32)).to("cuda")
    try:
        ref = weakref.ref(seeds, lambda _r, k=key: _seed_cache.pop(k, None))
        _seed_cache[key] = (ref, sidx, slab)
    except TypeError:
        pass
    return sidx, slab


def image_hash(image) -> bytes:
    ent = _image_entry(image)
    if ent[1] is None:
        ent[1] = content_hash(image)
    return ent[1]


def image_device(image):
    ent = _image_entry(image)
    if ent[2] is None:
        torch = require_cuda()
        ent[2] = torch.from_numpy(np.array(image.intensities, dtype=np.float64)).to("cuda")
    return ent[2]


def _check_image(pack, image):
    want = getattr(getattr(pack, "provenance", None), "image_hash", None)
    if want and image_hash(image) != want:
        raise ImageMismatch("pack was precomputed from a different image")


# host pack -> its device copy, one upload per host pack object.  The
# reference treats packs as immutable and shared, so a host
# SpectralPack passed to repeated solve_fast / select_m / refresh calls (the
# CLI and the service session do exactly that, cli.py:143-156,
# service/sessions.py:123-157) is uploaded once and its device copy (and its
# stencil graph) lives as long as the host object.  evict_device_pack() drops
# it early.
_pack_cache: dict = {}
UPLOADS = [0]      # host -> device pack uploads (tests assert one per host pack)


def evict_device_pack(pack=None) -> None:
    """Drop the cached device copy of ``pack`` (every cached pack if None)."""
    if pack is None:
        _pack_cache.clear()
    else:
        _pack_cache.pop(id(pack), None)


def _as_device(pack, image=None, connectivity=None, weight_mode=None) -> DevicePack:
    if isinstance(pack, DevicePack):
        if image is not None and pack.image_dev is None:
            pack.image_dev = image_device(image)
        return pack
    key = (connectivity, weight_mode or "abs")
    ent = _pack_cache.get(id(pack))
    if ent is not None and ent[0]() is pack and ent[1] == key:
        dp = ent[2]
    else:
        dp = to_device(pack, image=None, connectivity=connectivity, weight_mode=weight_mode or "abs")
        UPLOADS[0] += 1
        try:
            ref = weakref.ref(pack, lambda _r, k=id(pack): _pack_cache.pop(k, None))
            _pack_cache[id(pack)] = (ref, key, dp)
        except TypeError:
            pass   # not weak-referenceable: no safe identity key, upload per call
    if image is not None and dp.image_dev is None:
        dp.image_dev = image_device(image)
    return dp


def _cut_mask_device(lattice: LatticeSpec, cut_edges):
    if cut_edges is None:
        return None
    torch = require_cuda()
    if hasattr(cut_edges, "is_cuda"):
        return cut_edges.to(torch.uint8).contiguous()
    arr = np.asarray(cut_edges)
    if arr.ndim == 2 and arr.shape == (lattice.n, lattice.ndir):
        vm = arr.astype(np.uint8)
    else:
        vm = lattice.edge_mask_to_voxel_mask(arr)
    return torch.from_numpy(np.ascontiguousarray(vm)).to("cuda")


# ---------------------------------------------------------------------------
# beta / topology update
# ---------------------------------------------------------------------------

class RefreshedPack(DevicePack):
    """Base eigenvectors with Rayleigh-quotient values on the new graph
    (refresh.py:25-51).  The column permutation is folded into the solve
    kernels (col_map) instead of re-gathering V on every ``.eigen`` access."""

    base = None
    new_beta = None
    order_dev = None

    @property
    def lambda_hat(self) -> np.ndarray:
        return self.values

    @property
    def order(self) -> np.ndarray:
        return self.order_dev.cpu().numpy().astype(np.int64)

    @property
    def laplacian(self) -> DeviceGraph:
        return self.graph


class UpdatedPack(RefreshedPack):
    """First-order eigenpair update: V' = V C Pi diag(s), lam' = refresh lam^.
    ``C`` (M x M, device) and ``P`` = V^T dL V are kept for inspection."""

    C = None
    P = None


_SIDE = {}


def _side_stream():
    """Per-device side stream + event for work that overlaps the main stream."""
    torch = torch_mod()
    dev = torch.cuda.current_device()
    if dev not in _SIDE:
        _SIDE[dev] = (torch.cuda.Stream(), torch.cuda.Event())
    return _SIDE[dev]


def _stencil_ws(lattice, m):
    lat = lattice.c_struct()
    return WORKSPACE.get("stencil", _lib.size("swb_stencil_workspace_bytes", C.byref(lat), m))


def refresh(pack, image, new_beta: float, *, connectivity=None, weight_mode=None) -> RefreshedPack:
    """refresh.py:63-82 on the device: lam^ = max(diag(V^T L'V)/diag(V^T V), 0),
    stable sort; one HBM pass over V (stencil) + an M-sized sort."""
    if new_beta < 0:
        raise InvalidParam("beta must be >= 0")
    _check_image(pack, image)
    torch = require_cuda()
    dp = _as_device(pack, image, connectivity, weight_mode)
    if dp.col_map is not None:
        raise InvalidParam("refresh a base pack, not a refreshed one (reference semantics)")
    _mark("graph")
    graph = DeviceGraph.build(dp.image_dev, dp.lattice, new_beta)
    m = dp.m
    quad = torch.empty(m, dtype=torch.float64, device="cuda")
    norm2 = torch.empty_like(quad)
    vtd = torch.empty_like(quad)
    ws = _stencil_ws(dp.lattice, m)
    lat = dp.lattice.c_struct()
    st = stream_handle()
    n = dp.n_vertices
    _mark("stencil_rayleigh")
    _lib.call("swb_stencil_rayleigh", C.byref(lat), ptr(dp.V), dp.ldv, 0, 0, n, m, ptr(graph.what),
              ptr(graph.diag), ptr(graph.d_sqrt_dev), ptr(quad), ptr(norm2), ptr(vtd), ptr(ws), ws.numel(), st)
    lam = torch.empty(m, dtype=torch.float64, device="cuda")
    order = torch.empty(m, dtype=torch.int64, device="cuda")
    _mark("coeffs")
    _lib.call("swb_update_coeffs", 0, None, 0, None, ptr(quad), ptr(norm2), m, 0.0, None, 0, ptr(lam),
              ptr(order), st)
    col_map = order.to(torch.int32)
    vtg = gather_vector(vtd, col_map) / graph.dnorm
    _mark("update_end")
    out = RefreshedPack(dp.V, m, lam, graph.d_sqrt_dev, graph.dnorm, dp.dims, dp.spacing, float(new_beta),
                        dp.provenance, dp.lattice, image_dev=dp.image_dev, graph=graph, vtg=vtg,
                        col_map=col_map, mr=dp.mr)
    out.base = pack
    out.new_beta = float(new_beta)
    out.order_dev = order
    return out


def nearest_pack(packs, new_beta: float):
    """refresh.py:91-96: nearest base pack on a log-beta scale."""
    def distance(beta: float) -> float:
        if beta <= 0 or new_beta <= 0:
            return abs(beta - new_beta)
        return abs(math.log(new_beta) - math.log(beta))
    return min(packs.packs, key=lambda p: distance(p.beta))


def refresh_from_set(packs, image, new_beta: float, **kw) -> RefreshedPack:
    return refresh(nearest_pack(packs, new_beta), image, new_beta, **kw)


def update_basis(pack, image, new_beta: float | None = None, cut_edges=None, method: str = "first_order",
                 gap_guard: float = 0.5, *, connectivity=None, weight_mode=None, keep_P: bool = False, out=None,
                 _pre_rotate=None, _m2=None):
    """Update the eigenbasis for a new beta and/or cut edges (north-star (a)).

    method="rayleigh": exactly the reference refresh (no rotation).
    method="first_order": P = V^T (L^' - L^) V (difference stencil + DMMA
    symmetric projection), gap-guarded divided differences C, rotation
    V' = V C (DMMA GEMM), eigenvalues = refresh Rayleigh quotients, columns
    stably sorted.  The old pack stays valid unless ``out``
    (an N x ldv float64 device buffer, e.g. a retired pack's V) is given to
    receive V' — the ping-pong mode of chained interactive updates.
    """
    if method not in ("first_order", "rayleigh"):
        raise InvalidParam(f"unknown method {method!r}")
    dp0 = _as_device(pack, image, connectivity, weight_mode)
    beta = dp0.beta if new_beta is None else float(new_beta)
    if method == "rayleigh" and cut_edges is None:
        return refresh(dp0 if isinstance(pack, DevicePack) else pack, image, beta)
    if beta < 0:
        raise InvalidParam("beta must be >= 0")
    _check_image(pack, image)
    torch = require_cuda()
    dp = dp0
    if dp.col_map is not None:  # materialise a refreshed pack's column order first
        V2 = torch.zeros_like(dp.V)
        _lib.call("swb_gather_columns", ptr(dp.V), dp.ldv, dp.n_vertices, ptr(dp.col_map), dp.m, ptr(V2),
                  dp.ldv, stream_handle())
        dp = DevicePack(V2, dp.m, dp.values_dev, dp.d_sqrt_dev, dp.dnorm, dp.dims, dp.spacing, dp.beta,
                        dp.provenance, dp.lattice, image_dev=dp.image_dev, graph=dp.graph, vtg=dp.vtg)
    _mark("graph")
    g_old = dp.ensure_graph()
    cut = _cut_mask_device(dp.lattice, cut_edges)
    g_new = DeviceGraph.build(dp.image_dev, dp.lattice, beta, cut)
    _mark("alloc")
    m, n, ldv = dp.m, dp.n_vertices, dp.ldv
    st = stream_handle()
    lat = dp.lattice.c_struct()
    quad = torch.empty(m, dtype=torch.float64, device="cuda")
    norm2 = torch.empty_like(quad)
    vtd = torch.empty_like(quad)
    lam = torch.empty(m, dtype=torch.float64, device="cuda")
    order = torch.empty(m, dtype=torch.int64, device="cuda")
    if method == "rayleigh":  # cut edges, no rotation
        ws = _stencil_ws(dp.lattice, m)
        _lib.call("swb_stencil_rayleigh", C.byref(lat), ptr(dp.V), ldv, 0, 0, n, m, ptr(g_new.what),
                  ptr(g_new.diag), ptr(g_new.d_sqrt_dev), ptr(quad), ptr(norm2), ptr(vtd), ptr(ws),
                  ws.numel(), st)
        _lib.call("swb_update_coeffs", 0, None, 0, None, ptr(quad), ptr(norm2), m, 0.0, None, 0, ptr(lam),
                  ptr(order), st)
        col_map = order.to(torch.int32)
        out = RefreshedPack(dp.V, m, lam, g_new.d_sqrt_dev, g_new.dnorm, dp.dims, dp.spacing, beta,
                            dp.provenance, dp.lattice, image_dev=dp.image_dev, graph=g_new,
                            vtg=gather_vector(vtd, col_map) / g_new.dnorm, col_map=col_map, mr=dp.mr)
    else:
        if out is not None:
            if tuple(out.shape) != (n, ldv) or out.dtype != torch.float64 or out.data_ptr() == dp.V.data_ptr():
                raise InvalidParam("out must be a distinct N x ldv float64 device buffer")
            W = out
        else:
            W = torch.empty((n, ldv), dtype=torch.float64, device="cuda")   # becomes V' below
        ws = _stencil_ws(dp.lattice, m)
        _mark("stencil")
        _lib.call("swb_stencil_delta", C.byref(lat), ptr(dp.V), ldv, 0, 0, n, m, ptr(g_old.what),
                  ptr(g_old.diag), ptr(g_new.what), ptr(g_new.diag), ptr(g_new.d_sqrt_dev), ptr(W), ldv,
                  ptr(quad), ptr(norm2), ptr(vtd), ptr(ws), ws.numel(), st)
        ldp = round_up(m, 2)
        P = torch.empty((m, ldp), dtype=torch.float64, device="cuda")
        tws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", n, m, m))
        # SWB_EMIT=1: the rotation's digit planes of V come out of the
        # projection's diagonal tiles when V's row maxima are known (V came
        # out of an INT8 rotation that recorded them) instead of a split pass
        # over V; measured at c4 as a wash (the projection grows by what the
        # split cost: 114.5 + 62.5 vs 93 + 82 ms, the step ~1% faster) for
        # 46 GB more resident HBM, so the split stays the default
        m2 = m if _m2 is None else int(_m2)
        int8_rot = m <= 512 and not os.environ.get("SWB_ROTATION", "").startswith("d")
        amax_in = getattr(dp, "row_amax_dev", None)
        planes = None
        _mark("project")
        emit = int8_rot and os.environ.get("SWB_EMIT", "0") == "1"
        if emit and amax_in is not None:
            planes = oz_full_workspace(n, m, m2)
        if planes is not None:
            _lib.call("swb_gemm_tn_sym_emit", ptr(dp.V), ldv, ptr(W), ldv, n, m, ptr(P), ldp, ptr(tws), tws.numel(),
                      ptr(amax_in), m2, ptr(planes), planes.numel(), st)
        else:
            _lib.call("swb_gemm_tn", ptr(dp.V), ldv, ptr(W), ldv, n, m, m, 1, ptr(P), ldp, ptr(tws), tws.numel(), st)
        Cm = torch.empty((m, ldp), dtype=torch.float64, device="cuda")
        _mark("coeffs")
        _lib.call("swb_update_coeffs", 1, ptr(P), ldp, ptr(dp.values_dev), ptr(quad), ptr(norm2), m,
                  float(gap_guard), ptr(Cm), ldp, ptr(lam), ptr(order), st)
        Vn = W  # W is dead after the projection: the rotation writes V' into its buffer
        if ldv > m:
            Vn[:, m:].zero_()
        # V'^T d = C^T (V^T d): a 1-row NN product
        vtd_row = torch.zeros((1, ldp), dtype=torch.float64, device="cuda")
        vtd_row[0, :m].copy_(vtd)
        vtg_row = torch.empty((1, ldp), dtype=torch.float64, device="cuda")
        _lib.call("swb_gemm_nn", ptr(vtd_row), ldp, ptr(Cm), ldp, 1, m, m, ptr(vtg_row), ldp, 0, st)
        out = UpdatedPack(Vn, m, lam, g_new.d_sqrt_dev, g_new.dnorm, dp.dims, dp.spacing, beta, dp.provenance,
                          dp.lattice, image_dev=dp.image_dev, graph=g_new, vtg=vtg_row[0, :m] / g_new.dnorm)
        out.C = Cm
        if keep_P:
            out.P = P
        # update_and_solve: the solve's seed system runs here, on V' rows
        # formed from V and C, and returns extra B columns for the rotation
        extra = _pre_rotate(out, dp, Cm, ldp) if _pre_rotate is not None else None
        amax_out = torch.empty(n, dtype=torch.int64, device="cuda") if emit else None
        _mark("rotate")
        if extra is None:
            rotate_rows(dp.V, ldv, Cm, ldp, n, m, Vn, ldv, st, mark=_mark, m2=m2 if planes is not None else None,
                        planes=planes, row_amax=amax_out)
        else:
            m2x, c_aug, ldca, out2, ldo2 = extra
            if planes is not None and m2x != m2:
                raise InvalidParam("update_and_solve: extra column count changed")
            rotate_rows(dp.V, ldv, c_aug, ldca, n, m, Vn, ldv, st, mark=_mark, m2=m2x, out2=out2, ldo2=ldo2,
                        planes=planes, row_amax=amax_out)
        out.row_amax_dev = amax_out
        _mark("update_tail")
    out.base = pack if method == "rayleigh" else None   # an updated pack owns new memory: no strong ref
    out.new_beta = beta
    out.order_dev = order
    _mark("update_end")
    return out


# ---------------------------------------------------------------------------
# reduced-basis random walker solve
# ---------------------------------------------------------------------------

class DeviceField:
    """Solve result on the device: labels, top-2 gap, and (lazily) U.

    Host views mirror ProbabilityField (``values``, ``K``, ``dims``) and the
    hard-label map; ``labels_dev`` / ``top2_dev`` stay on the GPU."""

    def __init__(self, dims, k, labels_dev, top2_dev, U_dev=None, recompute=None):
        self.dims = tuple(dims)
        self._k = int(k)
        self.labels_dev = labels_dev
        self.top2_dev = top2_dev
        self.U_dev = U_dev
        self._recompute = recompute
        self._field = None

    @property
    def K(self) -> int:
        return self._k

    def _u(self):
        if self.U_dev is None:
            self.U_dev = self._recompute()
        return self.U_dev

    @property
    def values(self) -> np.ndarray:
        return self.field().values

    def field(self) -> ProbabilityField:
        if self._field is None:
            self._field = ProbabilityField(self.dims, self._u()[:, :self._k].cpu().numpy())
        return self._field

    def clamped(self) -> np.ndarray:
        return np.clip(self.values, 0.0, 1.0)


def _ell_from_lap(lap, seed_idx: np.ndarray):
    """Seed rows of a host Laplacian (reference ``Laplacian`` / CSR) in ELL form."""
    torch = torch_mod()
    mat = lap.matrix if hasattr(lap, "matrix") else lap
    rows = mat[seed_idx].tocsr()
    rows.sort_indices()
    s = seed_idx.size
    r = int(np.diff(rows.indptr).max()) if s else 1
    r = max(r, 1)
    idx = np.full((s, r), -1, dtype=np.int64)
    val = np.zeros((s, r), dtype=np.float64)
    for i in range(s):
        a, b = rows.indptr[i], rows.indptr[i + 1]
        idx[i, : b - a] = rows.indices[a:b]
        val[i, : b - a] = rows.data[a:b]
    return torch.from_numpy(idx).to("cuda"), torch.from_numpy(val).to("cuda"), r


def solve_fast(pack, lap, prob, m_use: int | None = None, streaming_block: int | None = None,
               *, want_field: bool = False, check: bool = True, _defer: bool = False,
               _tp_basis=None) -> DeviceField:
    """fastrw.py:352-467 on the device.

    ``pack``: DevicePack / RefreshedPack / UpdatedPack, or a host pack
    (uploaded).  ``lap``: a DeviceGraph (device stencil), None (the pack's
    own graph), or a reference-style Laplacian (its seed rows are read on
    the host, exactly like the reference reads ``lap.matrix[s_idx]``).
    ``streaming_block`` is accepted for signature parity (V is resident).
    """
    torch = require_cuda()
    dp = _as_device(pack)
    n = dp.n_vertices
    k = prob.K
    M = dp.m
    if m_use is None:
        m_use = M
    if not 1 <= m_use <= M:
        raise InvalidParam(f"m_use must be in 1..{M}")
    if m_use < k:
        raise InsufficientBasis(f"m_use={m_use} cannot represent {k} labels")
    if getattr(prob.laplacian_mode, "value", "normalized") != LaplacianMode.NORMALIZED.value:
        raise InvalidParam("the fast path requires the normalized mode")
    if lap is not None and (lap.n_vertices if hasattr(lap, "n_vertices") else lap.shape[0]) != n:
        raise InvalidParam("Laplacian size does not match the pack")
    seeds = prob.seeds
    s = int(seeds.n_seeds)
    if s > MAX_SEEDS:
        raise InvalidParam(f"at most {MAX_SEEDS} seeds supported, got {s}")
    gamma = float(prob.gamma)
    st = stream_handle()
    _mark("solve_seeds")
    sidx, slab = seed_tensors(seeds)
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    top2 = torch.empty(n, dtype=torch.float64, device="cuda")
    ldu = round_up(k, 2)
    if s == n:  # every voxel seeded: the one-hot field, no solve (fastrw.py:389-390)
        U = torch.zeros((n, ldu), dtype=torch.float64, device="cuda")
        _lib.call("swb_apply_seeds", ptr(sidx), ptr(slab), s, 0, n, k, ptr(U), ldu, ptr(labels), ptr(top2), st)
        return DeviceField(dp.dims, k, labels, top2, U)

    # seed rows of L^ (ELL)
    if lap is None or isinstance(lap, DeviceGraph):
        graph = lap if lap is not None else dp.ensure_graph()
        R = 2 * graph.lattice.ndir + 1
        ell_idx = torch.empty((max(s, 1), R), dtype=torch.int64, device="cuda")
        ell_val = torch.empty((max(s, 1), R), dtype=torch.float64, device="cuda")
        lat = graph.lattice.c_struct()
        _lib.call("swb_seed_rows", C.byref(lat), ptr(graph.what), ptr(graph.diag), ptr(sidx), s, ptr(ell_idx),
                  ptr(ell_val), st)
    else:
        ell_idx, ell_val, R = _ell_from_lap(lap, np.asarray(seeds.seed_indices, dtype=np.int64))

    ldq = round_up(m_use, 2)
    sa = max(s, 1)
    q_s = torch.empty((sa, ldq), dtype=torch.float64, device="cuda")
    b_qn = torch.empty((sa, ldq), dtype=torch.float64, device="cuda")
    bg = torch.empty(sa, dtype=torch.float64, device="cuda")
    lsu = torch.empty((sa, k), dtype=torch.float64, device="cuda")
    dsq_s = torch.empty(sa, dtype=torch.float64, device="cuda")
    col_map = dp.col_map
    if s:
        _lib.call("swb_seed_project", ptr(dp.V), dp.ldv, 0, 0, n, m_use, ptr(col_map), ptr(sidx), ptr(slab), s,
                  ptr(ell_idx), ptr(ell_val), R, ptr(dp.d_sqrt_dev), dp.dnorm, k, ptr(q_s), ldq, ptr(b_qn),
                  ptr(bg), ptr(lsu), ptr(dsq_s), st)
    values = dp.values_dev[:m_use]
    vtg = None
    t_p = None
    ldt = round_up(k, 2)
    if gamma == 0:
        vtg = dp.ensure_vtg()[:m_use].contiguous()
    else:
        priors = prob.priors
        if not hasattr(priors, "is_cuda"):
            priors = torch.from_numpy(np.ascontiguousarray(priors, dtype=np.float64)).to("cuda")
        ph = torch.empty((n, ldt), dtype=torch.float64, device="cuda")
        _lib.call("swb_prior_hat", ptr(priors), priors.stride(0), 0, n, k, ptr(dp.d_sqrt_dev), ptr(sidx), s,
                  ptr(ph), ldt, st)
        mr = dp.mr if col_map is not None else m_use
        tp_full = torch.empty((mr, ldt), dtype=torch.float64, device="cuda")
        if _tp_basis is not None:
            # update_and_solve: V'^T P^ = C^T (V^T P^) from the basis before the rotation
            Vb, ldvb, Cm, ldc = _tp_basis
            mb = Cm.shape[0]
            tb = torch.empty((mb, ldt), dtype=torch.float64, device="cuda")
            tws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", n, mb, k))
            _lib.call("swb_gemm_tn", ptr(Vb), ldvb, ptr(ph), ldt, n, mb, k, 0, ptr(tb), ldt, ptr(tws), tws.numel(),
                      st)
            tws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", mb, mr, k))
            _lib.call("swb_gemm_tn", ptr(Cm), ldc, ptr(tb), ldt, mb, mr, k, 0, ptr(tp_full), ldt, ptr(tws),
                      tws.numel(), st)
        else:
            tws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", n, mr, k))
            _lib.call("swb_gemm_tn", ptr(dp.V), dp.ldv, ptr(ph), ldt, n, mr, k, 0, ptr(tp_full), ldt, ptr(tws),
                      tws.numel(), st)
        if col_map is not None:
            t_p = torch.empty((m_use, ldt), dtype=torch.float64, device="cuda")
            _lib.call("swb_gather_rows", ptr(tp_full), ldt, ptr(col_map), m_use, k, ptr(t_p), ldt, st)
        else:
            t_p = tp_full
    coeff = torch.empty((m_use, k), dtype=torch.float64, device="cuda")
    extra = torch.empty(k, dtype=torch.float64, device="cuda") if gamma == 0 else None
    rcond = torch.empty(1, dtype=torch.float64, device="cuda")
    _mark("solve_system")
    sws = WORKSPACE.get("small_solve", _lib.size("swb_small_solve_workspace_bytes", s, m_use, k))
    # the 1-norm condition estimate runs on a side stream, overlapping the
    # reconstruction; the current stream joins it before returning
    side, ev = _side_stream()
    ev.record()
    _lib.call("swb_small_solve_ex", gamma, s, m_use, k, ptr(q_s), ptr(b_qn), ldq, ptr(bg), ptr(lsu), ptr(dsq_s),
              dp.dnorm, ptr(slab), ptr(values), ptr(vtg), ptr(t_p), ldt, ptr(coeff), ptr(extra), ptr(rcond),
              ptr(sws), sws.numel(), st, C.c_void_p(side.cuda_stream), C.c_void_p(ev.cuda_event))
    if col_map is not None:
        mr = dp.mr
        cf = torch.empty((mr, k), dtype=torch.float64, device="cuda")
        _lib.call("swb_scatter_rows", ptr(coeff), m_use, k, ptr(col_map), ptr(cf), mr, st)
    else:
        mr, cf = m_use, coeff

    def reconstruct(with_u: bool):
        U = torch.empty((n, ldu), dtype=torch.float64, device="cuda") if with_u else None
        _lib.call("swb_reconstruct_label", ptr(dp.V), dp.ldv, 0, 0, n, mr, ptr(cf), ptr(extra), dp.dnorm,
                  ptr(dp.d_sqrt_dev), k, ptr(U), ldu, ptr(labels), ptr(top2), stream_handle())
        _lib.call("swb_apply_seeds", ptr(sidx), ptr(slab), s, 0, n, k, ptr(U), ldu, ptr(labels), ptr(top2),
                  stream_handle())
        return U

    if _defer:   # update_and_solve: the reconstruction comes out of the rotation
        return dict(dp=dp, n=n, k=k, s=s, mr=mr, cf=cf, extra=extra, rcond=rcond, side=side, labels=labels,
                    top2=top2, sidx=sidx, slab=slab, ldu=ldu, reconstruct=reconstruct, check=check)
    _mark("solve_reconstruct")
    U = reconstruct(want_field or k > 8)
    torch.cuda.current_stream().wait_stream(side)
    _mark("solve_end")
    if check and not CAPTURE["on"]:   # a captured step checks rcond after each replay
        rc = float(rcond.item())
        if _lib.load().swb_check_rcond(rc) != 0:
            raise SingularSmallSystem(
                f"seed system numerically singular (cond ~ {1.0 / max(rc, 1e-300):.3e})",
                condition=1.0 / max(rc, 1e-300))
    field = DeviceField(dp.dims, k, labels, top2, U, recompute=lambda: reconstruct(True))
    field.rcond_dev = rcond
    return field


def update_and_solve(pack, image, prob, new_beta: float | None = None, cut_edges=None, *, gap_guard: float = 0.5,
                     m_use: int | None = None, want_field: bool = False, check: bool = True, out=None,
                     connectivity=None, weight_mode=None, policy=None):
    """``update_basis(pack, image, new_beta, cut_edges)`` followed by
    ``solve_fast(updated, None, prob, m_use)`` with one pass less over the
    basis: returns ``(updated_pack, field)``, the same objects the two calls
    return (V' in full; labels / top-2 / U of the solve on V').

    The seed system only needs V' at the seeds and their stencil neighbours,
    so it is solved BEFORE the rotation on those rows formed as V[rows] C
    (a small DMMA product scattered into the V' buffer, which the rotation
    then overwrites); its coefficients enter the rotation as extra columns
    of C -- V' coeff = V (C coeff) -- which ride in the padding of the INT8
    GEMM's last 64-column tile (K = 400: 48 free columns), so the
    reconstruction (fastrw.py:456-466) costs no pass over V' and no tensor
    work; a row-wise finalize + argmax (solver.py:55-66, images.py:128-130)
    reads the N x L products.  gamma > 0 (priors): the prior projection
    V'^T P^ is C^T (V^T P^), from the basis before the rotation.  The
    all-seeded case, gamma = 0 without seeds and a policy at gamma > 0 take
    the two separate calls.  ``policy`` (an AdaptivePolicy): m_use =
    select_m(updated, prob, policy) first (adaptive.py:133-185; at gamma = 0
    it reads only the seed rows, which are formed before the rotation); the
    chosen m is ``field.m_use``."""
    torch = require_cuda()
    seeds = prob.seeds
    s = int(seeds.n_seeds)
    gamma = float(prob.gamma)
    dp0 = _as_device(pack, image, connectivity, weight_mode)
    if s >= dp0.n_vertices or (gamma == 0 and s == 0) or (policy is not None and gamma != 0):
        up = update_basis(pack, image, new_beta, cut_edges, gap_guard=gap_guard, out=out,
                          connectivity=connectivity, weight_mode=weight_mode)
        if policy is not None:
            m_use, _ = select_m(up, prob, policy)
        f = solve_fast(up, None, prob, m_use, want_field=want_field, check=check)
        f.m_use = m_use
        return up, f
    state = {}

    def pre_rotate(up, dp, Cm, ldp):
        m, ldv, st = up.m, up.ldv, stream_handle()
        g_new = up.graph
        # V' rows at the seeds and their stencil neighbours: V[rows] C
        _mark("solve_prefill")
        if s:
            sidx, _ = seed_tensors(seeds)
            R = 2 * g_new.lattice.ndir + 1
            ell_idx = torch.empty((s, R), dtype=torch.int64, device="cuda")
            ell_val = torch.empty((s, R), dtype=torch.float64, device="cuda")
            lat = g_new.lattice.c_struct()
            _lib.call("swb_seed_rows", C.byref(lat), ptr(g_new.what), ptr(g_new.diag), ptr(sidx), s, ptr(ell_idx),
                      ptr(ell_val), st)
            vg = torch.empty((s * R, ldv), dtype=torch.float64, device="cuda")
            vp = torch.empty_like(vg)
            nv = up.n_vertices
            _lib.call("swb_ell_rows_gather", ptr(dp.V), ldv, 0, nv, ptr(ell_idx), ptr(sidx), s, R, m, ptr(vg), st)
            _lib.call("swb_gemm_nn", ptr(vg), ldv, ptr(Cm), ldp, s * R, m, m, ptr(vp), ldv, 0, st)
            _lib.call("swb_ell_rows_scatter", ptr(vp), ldv, 0, nv, ptr(ell_idx), ptr(sidx), s, R, m, ptr(up.V), st)
        mu = m_use
        if policy is not None:
            mu, _ = select_m(up, prob, policy)
        state["m_use"] = mu
        d = solve_fast(up, None, prob, mu, want_field=want_field, check=check, _defer=True,
                       _tp_basis=(dp.V, ldv, Cm, ldp) if gamma != 0 else None)
        k, mr, cf = d["k"], d["mr"], d["cf"]
        # C_aug = [C | C[:, :mr] coeff]; V C_aug[:, m:] = V' coeff
        m2 = m + k
        ldca = round_up(m2, 2)
        c_aug = torch.empty((m, ldca), dtype=torch.float64, device="cuda")
        ccf = torch.empty((m, round_up(k, 2)), dtype=torch.float64, device="cuda")
        _lib.call("swb_gemm_nn", ptr(Cm), ldp, ptr(cf), k, m, mr, k, ptr(ccf), ccf.shape[1], 0, st)
        _lib.call("swb_build_caug", ptr(Cm), ldp, ptr(ccf), ccf.shape[1], m, k, ptr(c_aug), ldca, st)
        # many labels: the products go straight into the field U (finalized
        # in place); else a compact N x L block
        ldr = d["ldu"] if k > 8 else k
        uraw = torch.empty((up.n_vertices, ldr), dtype=torch.float64, device="cuda")
        state.update(d=d, uraw=uraw)
        return m2, c_aug, ldca, uraw, ldr

    up = update_basis(pack, image, new_beta, cut_edges, gap_guard=gap_guard, out=out, connectivity=connectivity,
                      weight_mode=weight_mode, _pre_rotate=pre_rotate, _m2=dp0.m + prob.K)
    d, uraw = state["d"], state["uraw"]
    n, k, dev = d["n"], d["k"], d["dp"]
    labels, top2, ldu = d["labels"], d["top2"], d["ldu"]
    _mark("solve_finalize")
    if k > 8:   # the many-label finalize works in place, in U
        U = uraw
        _lib.call("swb_finalize_label", 0, n, k, ptr(U), ldu, ptr(d["extra"]), dev.dnorm, ptr(dev.d_sqrt_dev),
                  ptr(U), ldu, ptr(labels), ptr(top2), stream_handle())
    else:
        U = torch.empty((n, ldu), dtype=torch.float64, device="cuda") if want_field else None
        _lib.call("swb_finalize_label", 0, n, k, ptr(uraw), k, ptr(d["extra"]), dev.dnorm, ptr(dev.d_sqrt_dev),
                  ptr(U), ldu, ptr(labels), ptr(top2), stream_handle())
    _lib.call("swb_apply_seeds", ptr(d["sidx"]), ptr(d["slab"]), d["s"], 0, n, k, ptr(U), ldu, ptr(labels),
              ptr(top2), stream_handle())
    torch.cuda.current_stream().wait_stream(d["side"])
    _mark("solve_end")
    if check and not CAPTURE["on"]:
        rc = float(d["rcond"].item())
        if _lib.load().swb_check_rcond(rc) != 0:
            raise SingularSmallSystem(
                f"seed system numerically singular (cond ~ {1.0 / max(rc, 1e-300):.3e})",
                condition=1.0 / max(rc, 1e-300))
    field = DeviceField(dev.dims, k, labels, top2, U, recompute=lambda: d["reconstruct"](True))
    field.rcond_dev = d["rcond"]
    field.m_use = state["m_use"]
    return up, field


def hard_labels(field) -> LabelMap:
    """images.py:128-130: argmax per voxel, ties to the lowest label."""
    if isinstance(field, DeviceField):
        return LabelMap(field.dims, field.labels_dev.cpu().numpy())
    torch = require_cuda()
    vals = np.array(field.values, dtype=np.float64)
    n, k = vals.shape
    U = torch.from_numpy(vals).to("cuda")
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.call("swb_argmax_rows", ptr(U), k, n, k, ptr(labels), None, stream_handle())
    return LabelMap(field.dims, labels.cpu().numpy())


# ---------------------------------------------------------------------------
# dynamic basis size (adaptive.py:133-185)
# ---------------------------------------------------------------------------

def select_m(pack, prob, policy=None):
    """Smallest scheduled m whose seed-fit and prior-residual criteria all
    pass, else (pack.m, saturated) — adaptive.py:133-185 on the device.

    Seed criterion: swb_seed_fit_schedule evaluates seed_fit for every
    scheduled m at once (one QR, per-step Jacobi SVDs in parallel).  Prior
    criterion: the incremental residual r <- r - V_new (V_new^T r) on the
    DMMA GEMMs (adaptive.py:113-130).  Returns (m_use, info) with the same
    info layout as the reference (steps up to the decision only).
    """
    from .types import AdaptivePolicy
    torch = require_cuda()
    policy = policy or AdaptivePolicy()
    dp = _as_device(pack)
    k = prob.K
    n = dp.n_vertices
    M = dp.m
    bound = dp.dnorm  # norm_bound(NORMALIZED, d_sqrt**2) = sqrt(sum d_sqrt^2) (adaptive.py:65-69)
    seeds = prob.seeds
    s = int(seeds.n_seeds)
    sched = policy.schedule(M, k)
    st = stream_handle()
    f_tab = None
    if s:
        sidx = torch.from_numpy(np.ascontiguousarray(seeds.seed_indices, dtype=np.int64)).to("cuda")
        slab = torch.from_numpy(np.ascontiguousarray(seeds.seed_labels, dtype=np.int32)).to("cuda")
        steps = torch.tensor(sched, dtype=torch.int32, device="cuda")
        f_dev = torch.empty((len(sched), k), dtype=torch.float64, device="cuda")
        ws = WORKSPACE.get("seed_fit", _lib.size("swb_seed_fit_workspace_bytes", s, M, k, len(sched)))
        _lib.call("swb_seed_fit_schedule", ptr(dp.V), dp.ldv, ptr(dp.col_map), ptr(sidx), ptr(slab), s,
                  ptr(dp.d_sqrt_dev), M, k, ptr(steps), len(sched), int(max(sched)), float(bound), ptr(f_dev),
                  ptr(ws), ws.numel(), st)
        f_tab = f_dev.cpu().numpy()
    g_tab = None
    if prob.priors is not None:
        tl = policy.label_subset(k)
        T = int(tl.size)
        ldt = round_up(T, 2)
        pri = prob.priors
        if hasattr(pri, "is_cuda"):
            pri = pri[:, torch.as_tensor(tl, device=pri.device)].contiguous()
        else:
            pri = torch.from_numpy(np.ascontiguousarray(np.asarray(pri, dtype=np.float64)[:, tl])).to("cuda")
        R = torch.empty((n, ldt), dtype=torch.float64, device="cuda")
        _lib.call("swb_prior_hat", ptr(pri), pri.stride(0), 0, n, T, ptr(dp.d_sqrt_dev), None, 0, ptr(R), ldt, st)
        cmap = dp.col_map if dp.col_map is not None else torch.arange(M, dtype=torch.int32, device="cuda")
        g_rows = []
        prev = 0
        G = torch.empty((T, ldt), dtype=torch.float64, device="cuda")
        for m in sched:
            dm = m - prev
            if dm > 0:
                ldn = round_up(dm, 2)
                Vn = torch.zeros((n, ldn), dtype=torch.float64, device="cuda")
                _lib.call("swb_gather_columns", ptr(dp.V), dp.ldv, n, ptr(cmap[prev:m]), dm, ptr(Vn), ldn, st)
                coef = torch.empty((dm, ldt), dtype=torch.float64, device="cuda")
                tws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", n, max(dm, T), T))
                _lib.call("swb_gemm_tn", ptr(Vn), ldn, ptr(R), ldt, n, dm, T, 0, ptr(coef), ldt, ptr(tws),
                          tws.numel(), st)
                # r -= V_new coef
                _lib.call("swb_gemm_nn_ex", ptr(Vn), ldn, ptr(coef), ldt, n, dm, T, ptr(R), ldt, 1, -1.0, st)
            tws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", n, T, T))
            _lib.call("swb_gemm_tn", ptr(R), ldt, ptr(R), ldt, n, T, T, 1, ptr(G), ldt, ptr(tws), tws.numel(), st)
            g_rows.append(torch.diagonal(G[:, :T]).clone())
            prev = m
        g_tab = torch.stack(g_rows).cpu().numpy()
    f_max = policy.seed_threshold(s) if s else None
    g_max = policy.prior_threshold(n) if prob.priors is not None else None
    info = {"steps": [], "saturated": False}
    for t, m in enumerate(sched):
        step = {"m": m, "f": [], "g": []}
        ok = True
        if f_tab is not None:
            for col in range(k):
                f = float(f_tab[t, col])
                step["f"].append(f)
                ok = ok and f <= f_max
        if g_tab is not None:
            for j in range(g_tab.shape[1]):
                g = float(g_tab[t, j])
                step["g"].append(g)
                ok = ok and g <= g_max
        info["steps"].append(step)
        if ok:
            return m, info
    info["saturated"] = True
    return M, info


# ---------------------------------------------------------------------------
# segment: the CLI "segment" flow as one library call (cli.py:126-163)
# ---------------------------------------------------------------------------

def segment(image, packs, seeds, gamma: float = 0.0, beta_online: float | None = None, adaptive: bool = False,
            m_use: int | None = None, epsilon: float = 0.1, method: str = "rayleigh", want_field: bool = False):
    """Library form of ``specwalk segment`` (cli.py:126-163).

    ``packs``: a PackSet / sequence of host or device packs of ``image``;
    ``seeds``: a SeedPartition.  With ``beta_online`` the nearest pack (log
    beta) is refreshed (``method="rayleigh"``, the reference) or updated to
    first order (``method="first_order"``).  gamma > 0 uses uniform priors
    like the CLI.  Returns (LabelMap, field, report dict)."""
    from .types import AdaptivePolicy, LabelProblem, PackSet
    if not isinstance(packs, PackSet):
        packs = PackSet(tuple(sorted(packs, key=lambda p: p.beta)))
    h = image_hash(image)
    for p in packs.packs:
        if p.provenance.image_hash != h:
            raise ImageMismatch("pack was not built from this image")
    k = seeds.num_labels
    n = image.n_voxels
    priors = None if gamma == 0 else np.full((n, k), 1.0 / k)
    prob = LabelProblem(num_labels=k, seeds=seeds, gamma=gamma, priors=priors)
    refreshed = False
    if beta_online is not None:
        base = nearest_pack(packs, beta_online)
        if method == "rayleigh":
            pack = refresh(base, image, beta_online)
        else:
            pack = update_basis(base, image, beta_online, method=method)
        lap = pack.laplacian
        refreshed = True
        base_beta = base.beta
    else:
        pack = _as_device(packs.packs[0], image)
        lap = pack.ensure_graph()
        base_beta = pack.beta
    if adaptive:
        m_use, _ = select_m(pack, prob, AdaptivePolicy(epsilon=epsilon))
    elif m_use is None:
        m_use = pack.m
    field = solve_fast(pack, lap, prob, m_use=m_use, want_field=want_field)
    labels = hard_labels(field)
    report = {"m_use": int(m_use), "refreshed": refreshed, "base_beta": float(base_beta), "num_labels": k}
    return labels, field, report
