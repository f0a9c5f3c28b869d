"""GPU-resident state of the hot path: lattice, graph stencil, spectral pack.

PyTorch is used only to own device memory and to pick the current CUDA
stream; every computation is a call into libspecwalk_b200.so.

Device layout:
  * V            row-major N x ldv float64 (ldv = round_up(m, 8), zero pad)
  * what         N x ndir float64: normalised forward-edge weights of L^
  * diag, d_sqrt N float64
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BackendUnavailable, DegenerateGraph, InvalidParam
from .types import PackProvenance, num_voxels

WEIGHT_MODES = {"abs": 0, "sq": 1}


def torch_mod():
    import torch
    return torch


def require_cuda():
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device: the B200 path has no CPU fallback")
    _lib.load()
    return torch


def stream_handle():
    torch = torch_mod()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def round_up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


class Workspace:
    """Grow-only scratch buffers keyed by purpose (one set per process)."""

    def __init__(self):
        self._bufs = {}

    def get(self, key: str, nbytes: int):
        torch = torch_mod()
        nbytes = max(int(nbytes), 256)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(round_up(nbytes, 1 << 20), dtype=torch.uint8, device="cuda")
            self._bufs[key] = buf
        return buf

    def clear(self):
        self._bufs.clear()


WORKSPACE = Workspace()


_OZ_FULL = {}


def oz_full_workspace(rows: int, m: int, m2: int):
    """The INT8 rotation workspace with one A-plane buffer per row chunk (all
    of V's digit planes resident: the projection emits them, the rotation
    skips its split).  Zero-filled once per shape: plane entries no producer
    writes (columns past m in the last K chunk, rows past the end) stay 0.
    None when it does not fit in device memory."""
    from . import _lib
    torch = torch_mod()
    key = (torch.cuda.current_device(), rows, m, m2)
    ws = _OZ_FULL.get(key)
    if ws is False:
        return None
    if ws is None:
        _OZ_FULL.clear()
        nb = _lib.size("swb_oz_gemm_nn_workspace_bytes_full", rows, m, m2)
        for attempt in range(2):
            try:
                ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
                break
            except torch.OutOfMemoryError:
                if attempt:
                    # does not fit next to the bases: the rotation splits V itself
                    _OZ_FULL[key] = False
                    import warnings
                    warnings.warn(f"oz_full_workspace: {nb / 2**30:.1f} GiB do not fit "
                                  f"(allocated {torch.cuda.memory_allocated() / 2**30:.1f} GiB); "
                                  "the rotation splits V instead", RuntimeWarning)
                    return None
                torch.cuda.empty_cache()
        _OZ_FULL[key] = ws
    return ws


def rotate_rows(V, ldv: int, Cm, ldc: int, rows: int, m: int, out, ldo: int, stream=None, mark=None,
                m2: int | None = None, out2=None, ldo2: int = 0, planes=None, row_amax=None) -> None:
    """out[rows x m] = V[rows x m] Cm[m x m] (the first-order rotation,
    reference update.py V' = V C): on the INT8 tensor cores (csrc/ozaki.cu,
    FP64-accurate digit scheme) for m <= 512, else the FP64 DMMA GEMM.
    ``mark(name)`` (the phase timer) brackets the digit split and the GEMM
    of every row chunk.  SWB_ROTATION=dmma forces the DMMA GEMM
    (measurement knob).

    ``m2 > m``: Cm is m x m2 and its columns [m, m2) are extra products
    V Cm[:, m:m2] written to ``out2`` (ld ``ldo2``); on the INT8 path they
    ride in the last column tile's padding (update_and_solve).
    ``planes``: an oz_full_workspace whose A planes of V were emitted by the
    projection (swb_gemm_tn_sym_emit): no digit split.  ``row_amax`` (int64
    N, zeroed here): receives max_c |out[r, c]| bits for the next update's
    emission."""
    import os
    from . import _lib
    st = stream if stream is not None else stream_handle()
    if rows <= 0:
        return
    m2 = m if m2 is None else int(m2)
    if m > 512 or os.environ.get("SWB_ROTATION", "").startswith("d"):
        _lib.call("swb_gemm_nn", ptr(V), ldv, ptr(Cm), ldc, rows, m, m, ptr(out), ldo, 0, st)
        if m2 > m:
            cx = Cm[:m, m:m2].contiguous()
            _lib.call("swb_gemm_nn", ptr(V), ldv, ptr(cx), m2 - m, rows, m, m2 - m, ptr(out2), ldo2, 0, st)
        return
    mark = mark or (lambda name: None)
    torch = torch_mod()
    if planes is not None:
        ws = planes
    else:
        nb = _lib.size("swb_oz_gemm_nn_workspace_bytes", rows, m, m2)
        ws = WORKSPACE.get("oz_gemm", nb)
    chunk = _lib.size("swb_oz_chunk_rows", rows, m, m2)
    nch = (rows + chunk - 1) // chunk
    if row_amax is not None:
        row_amax.zero_()
    mark("rotate_split")
    _lib.call("swb_oz_split_cols", ptr(Cm), ldc, rows, m, m2, ptr(ws), ws.numel(), st)
    if planes is not None:   # V's planes are already in buffers 0 .. nch-1
        for i in range(nch):
            r0 = i * chunk
            mark("rotate_gemm")
            _lib.call("swb_oz_gemm_planes_ex", min(chunk, rows - r0), rows, m, m2, i,
                      C.c_void_p(out.data_ptr() + 8 * r0 * ldo), ldo, m,
                      C.c_void_p(out2.data_ptr() + 8 * r0 * ldo2) if m2 > m else None, ldo2,
                      C.c_void_p(row_amax.data_ptr() + 8 * r0) if row_amax is not None else None,
                      ptr(ws), ws.numel(), st)
            mark("rotate_join")
        return
    main = torch.cuda.current_stream()
    # SWB_OZ_SERIAL=1 (measurement knob): split and GEMM in turn on one stream
    aux = _aux_stream() if nch > 1 and os.environ.get("SWB_OZ_SERIAL") != "1" else main
    ev_split = [torch.cuda.Event(), torch.cuda.Event()]
    ev_gemm = [torch.cuda.Event(), torch.cuda.Event()]
    if aux is not main:
        aux.wait_stream(main)                     # V and C's planes ready

    def split(i):
        # chunk i's A planes into buffer i % 2 on the side stream; the split
        # of chunk i+1 runs beside the GEMM of chunk i (csrc/ozaki.cu)
        r0 = i * chunk
        if i >= 2:
            aux.wait_event(ev_gemm[i & 1])        # the buffer's previous GEMM is done
        _lib.call("swb_oz_split_rows", C.c_void_p(V.data_ptr() + 8 * r0 * ldv), ldv, min(chunk, rows - r0), rows,
                  m, m2, i & 1, ptr(ws), ws.numel(), C.c_void_p(aux.cuda_stream))
        ev_split[i & 1].record(aux)

    split_first = os.environ.get("SWB_OZ_SPLIT_FIRST") == "1"   # measurement knob: the other enqueue order
    split(0)
    for i in range(nch):
        if split_first and i + 1 < nch:
            split(i + 1)
        r0 = i * chunk
        main.wait_event(ev_split[i & 1])
        mark("rotate_gemm")
        _lib.call("swb_oz_gemm_planes_ex", min(chunk, rows - r0), rows, m, m2, i & 1,
                  C.c_void_p(out.data_ptr() + 8 * r0 * ldo), ldo, m,
                  C.c_void_p(out2.data_ptr() + 8 * r0 * ldo2) if m2 > m else None, ldo2,
                  C.c_void_p(row_amax.data_ptr() + 8 * r0) if row_amax is not None else None,
                  ptr(ws), ws.numel(), st)
        ev_gemm[i & 1].record(main)
        # GEMM i is enqueued before split i+1: both become runnable together
        # (when GEMM i-1 and split i end) and cannot share an SM, so the
        # order decides which runs first -- the GEMM, with the split in the
        # SMs it frees; the other order charged the split's time to the
        # GEMM's events on some runs (same total either way)
        if not split_first and i + 1 < nch:
            split(i + 1)
        mark("rotate_join")


_AUX = {}

# CUDA-graph capture state (capture.CapturedStep): "record" while its eager
# warm-up runs (host scalars of the graphs it builds are kept), "on" while
# the step is being captured (no host reads; checks deferred to replays).
CAPTURE = {"on": False, "record": False, "dnorm": {}}


def _aux_stream():
    """The side stream of the rotation's digit split (one per device)."""
    torch = torch_mod()
    dev = torch.cuda.current_device()
    if dev not in _AUX:
        _AUX[dev] = torch.cuda.Stream(device=dev)
    return _AUX[dev]


# ---------------------------------------------------------------------------
# lattice
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class LatticeSpec:
    """Grid + neighbourhood + weight formula (see include/specwalk_b200.h)."""

    dims: tuple
    connectivity: int
    weight_mode: str = "abs"

    @staticmethod
    def make(dims, connectivity=None, weight_mode="abs") -> "LatticeSpec":
        dims = tuple(int(d) for d in dims)
        if connectivity is None:
            connectivity = 4 if len(dims) == 2 else 6
        if len(dims) == 2 and connectivity not in (4, 8):
            raise InvalidParam("2-D lattices support 4- or 8-connectivity")
        if len(dims) == 3 and connectivity != 6:
            raise InvalidParam("3-D lattices support 6-connectivity")
        if weight_mode not in WEIGHT_MODES:
            raise InvalidParam(f"unknown weight mode {weight_mode!r}")
        return LatticeSpec(dims, int(connectivity), weight_mode)

    @property
    def n(self) -> int:
        return num_voxels(self.dims)

    @property
    def nx(self) -> int:
        return self.dims[0]

    @property
    def ndir(self) -> int:
        return {4: 2, 8: 4, 6: 3}[self.connectivity]

    def c_struct(self) -> _lib.Lattice:
        nz = self.dims[2] if len(self.dims) == 3 else 1
        return _lib.Lattice(self.dims[0], self.dims[1], nz, self.connectivity, WEIGHT_MODES[self.weight_mode])

    def forward_offsets(self):
        if self.connectivity == 4:
            return [(1, 0), (0, 1)]
        if self.connectivity == 8:
            return [(1, 0), (0, 1), (1, 1), (-1, 1)]
        return [(1, 0, 0), (0, 1, 0), (0, 0, 1)]

    def edge_mask_to_voxel_mask(self, edge_mask) -> np.ndarray:
        """Edge-list mask (order of oracle.lattice_edges / reference
        lattice_edges: direction-major, heads in Fortran order) -> N x ndir."""
        edge_mask = np.asarray(edge_mask, dtype=bool).ravel()
        dims = self.dims
        nd = len(dims)
        grid = np.arange(self.n, dtype=np.int64).reshape(dims, order="F")
        out = np.zeros((self.n, self.ndir), dtype=np.uint8)
        pos = 0
        for d, off in enumerate(self.forward_offsets()):
            src = [slice(None)] * nd
            for ax, o in enumerate(off):
                if o > 0:
                    src[ax] = slice(None, -o)
                elif o < 0:
                    src[ax] = slice(-o, None)
            heads = grid[tuple(src)].ravel(order="F")
            out[heads, d] = edge_mask[pos:pos + heads.size]
            pos += heads.size
        if pos != edge_mask.size:
            raise InvalidParam(f"cut mask has {edge_mask.size} edges, lattice has {pos}")
        return out


# ---------------------------------------------------------------------------
# graph (normalised Laplacian stencil)
# ---------------------------------------------------------------------------

class DeviceGraph:
    """Normalised Laplacian L^ at one beta, as a device stencil.

    Replaces build_graph + laplacian(NORMALIZED) (graphs.py:127-159).  The
    reference ``Laplacian`` surface used by callers (``mode``, ``n_vertices``,
    ``d_sqrt``, ``matrix``) is provided lazily on the host for compatibility;
    the device path never materialises the CSR.
    """

    def __init__(self, lattice: LatticeSpec, beta: float, what, diag, d_sqrt, dnorm: float, cut_mask=None):
        self.lattice = lattice
        self.beta = float(beta)
        self.what = what
        self.diag = diag
        self.d_sqrt_dev = d_sqrt
        self.dnorm = float(dnorm)
        self.cut_mask = cut_mask
        self._host_d_sqrt = None
        self._csr = None

    @classmethod
    def build(cls, intensities_dev, lattice: LatticeSpec, beta: float, cut_mask_dev=None) -> "DeviceGraph":
        """Graph coefficients on the device plus two host scalars (||d_sqrt||
        and the degenerate flag: one small D2H).  While a CapturedStep records
        its CUDA graph (CAPTURE["on"]) the kernels are captured as usual but
        the host scalars come from its eager warm-up runs of the same graph
        (same image buffer, lattice, beta, cut), which already validated it."""
        torch = require_cuda()
        if beta < 0:
            raise InvalidParam(f"beta must be >= 0, got {beta}")
        key = (intensities_dev.data_ptr(), lattice.dims, lattice.connectivity, lattice.weight_mode, float(beta),
               cut_mask_dev.data_ptr() if cut_mask_dev is not None else 0)
        n = lattice.n
        what = torch.empty(n * lattice.ndir, dtype=torch.float64, device="cuda")
        diag = torch.empty(n, dtype=torch.float64, device="cuda")
        d_sqrt = torch.empty(n, dtype=torch.float64, device="cuda")
        flag = torch.zeros(2, dtype=torch.int32, device="cuda")
        lat = lattice.c_struct()
        st = stream_handle()
        _lib.call("swb_graph_build", C.byref(lat), ptr(intensities_dev), float(beta), ptr(cut_mask_dev),
                  ptr(what), ptr(diag), ptr(d_sqrt), ptr(flag), st)
        ss = torch.empty(1, dtype=torch.float64, device="cuda")
        ws = WORKSPACE.get("sumsq", 256 * 8)
        _lib.call("swb_sumsq", ptr(d_sqrt), n, ptr(ss), ptr(ws), ws.numel(), st)
        if CAPTURE["on"]:
            if key not in CAPTURE["dnorm"]:
                raise InvalidParam("graph capture: this graph was not built in the eager warm-up")
            return cls(lattice, beta, what, diag, d_sqrt, CAPTURE["dnorm"][key], cut_mask_dev)
        # one small D2H for the degenerate flag and ||d_sqrt|| (host scalars)
        host = torch.cat([ss, flag[:1].to(torch.float64)]).cpu().numpy()
        if host[1] != 0:
            raise DegenerateGraph("graph has an isolated vertex (zero degree)")
        dnorm = float(np.sqrt(host[0]))
        if CAPTURE["record"]:
            CAPTURE["dnorm"][key] = dnorm
        return cls(lattice, beta, what, diag, d_sqrt, dnorm, cut_mask_dev)

    @classmethod
    def build_region(cls, intensities_dev, lattice: LatticeSpec, beta: float, u_lo: int, u_hi: int,
                     cut_mask_dev=None) -> "DeviceGraph":
        """Coefficients for the units (planes / lines) [u_lo, u_hi) only, in
        full-size (globally indexed) arrays, zero elsewhere: the slab graph of
        a z-slab shard.  Degrees of the region's outermost units miss their
        outside neighbours, so callers build one unit beyond what they read.
        ``dnorm`` is left NaN (a global reduction; set by the caller)."""
        torch = require_cuda()
        if beta < 0:
            raise InvalidParam(f"beta must be >= 0, got {beta}")
        dims = lattice.dims
        unit = dims[0] * dims[1] if len(dims) == 3 else dims[0]
        sub_dims = tuple(dims[:-1]) + (u_hi - u_lo,)
        sub = LatticeSpec(sub_dims, lattice.connectivity, lattice.weight_mode)
        n, nd = lattice.n, lattice.ndir
        what = torch.zeros(n * nd, dtype=torch.float64, device="cuda")
        diag = torch.zeros(n, dtype=torch.float64, device="cuda")
        d_sqrt = torch.zeros(n, dtype=torch.float64, device="cuda")
        flag = torch.zeros(2, dtype=torch.int32, device="cuda")
        r0 = u_lo * unit
        lat = sub.c_struct()
        cut = C.c_void_p(cut_mask_dev.data_ptr() + r0 * nd) if cut_mask_dev is not None else None
        _lib.call("swb_graph_build", C.byref(lat), C.c_void_p(intensities_dev.data_ptr() + 8 * r0), float(beta), cut,
                  C.c_void_p(what.data_ptr() + 8 * r0 * nd), C.c_void_p(diag.data_ptr() + 8 * r0),
                  C.c_void_p(d_sqrt.data_ptr() + 8 * r0), ptr(flag), stream_handle())
        if int(flag[0].item()) != 0:
            raise DegenerateGraph("graph has an isolated vertex (zero degree)")
        return cls(lattice, beta, what, diag, d_sqrt, float("nan"), cut_mask_dev)

    # --- reference Laplacian surface (host, lazy) --------------------------
    @property
    def mode(self):
        from .types import LaplacianMode
        return LaplacianMode.NORMALIZED

    @property
    def n_vertices(self) -> int:
        return self.lattice.n

    @property
    def d_sqrt(self) -> np.ndarray:
        if self._host_d_sqrt is None:
            self._host_d_sqrt = self.d_sqrt_dev.cpu().numpy()
        return self._host_d_sqrt

    @property
    def matrix(self):
        """Host CSR of L^ (compatibility only; assembled from the stencil)."""
        if self._csr is None:
            import scipy.sparse as sp
            lat = self.lattice
            what = self.what.cpu().numpy().reshape(lat.n, lat.ndir)
            diag = self.diag.cpu().numpy()
            dims = lat.dims
            nd = len(dims)
            grid = np.arange(lat.n, dtype=np.int64).reshape(dims, order="F")
            rows, cols, vals = [np.arange(lat.n)], [np.arange(lat.n)], [diag]
            for d, off in enumerate(lat.forward_offsets()):
                src = [slice(None)] * nd
                dst = [slice(None)] * nd
                for ax, o in enumerate(off):
                    if o > 0:
                        src[ax], dst[ax] = slice(None, -o), slice(o, None)
                    elif o < 0:
                        src[ax], dst[ax] = slice(-o, None), slice(None, o)
                h = grid[tuple(src)].ravel(order="F")
                t = grid[tuple(dst)].ravel(order="F")
                v = -what[h, d]
                rows += [h, t]
                cols += [t, h]
                vals += [v, v]
            mat = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                shape=(lat.n, lat.n)).tocsr()
            mat.sort_indices()
            self._csr = mat
        return self._csr


# ---------------------------------------------------------------------------
# spectral pack on the device
# ---------------------------------------------------------------------------

class DevicePack:
    """GPU-resident spectral pack (the reference pack protocol, on device).

    Exposes the duck-typed surface the reference solve uses (``eigen``,
    ``d_sqrt``, ``dims``, ``m``; fastrw.py:352-360) — the host views are
    materialised lazily and only for compatibility.
    """

    def __init__(self, V, m: int, values, d_sqrt_dev, dnorm: float, dims, spacing, beta: float,
                 provenance, lattice: LatticeSpec, image_dev=None, graph: DeviceGraph | None = None,
                 vtg=None, col_map=None, mr: int | None = None):
        self.V = V
        self.ldv = V.shape[1]
        self._m = int(m)
        self.values_dev = values
        self.d_sqrt_dev = d_sqrt_dev
        self.dnorm = float(dnorm)
        self.dims = tuple(dims)
        self.spacing = tuple(spacing) if spacing else (1.0,) * len(self.dims)
        self.beta = float(beta)
        self.provenance = provenance
        self.lattice = lattice
        self.image_dev = image_dev
        self.graph = graph
        self.vtg = vtg
        self.col_map = col_map
        self.mr = int(mr) if mr is not None else int(m)
        self._host_values = None
        self._host_d_sqrt = None

    # --- reference pack surface -----------------------------------------
    @property
    def m(self) -> int:
        return self._m

    @property
    def n_vertices(self) -> int:
        return self.V.shape[0]

    @property
    def values(self) -> np.ndarray:
        if self._host_values is None:
            self._host_values = self.values_dev.cpu().numpy()
        return self._host_values

    @property
    def d_sqrt(self) -> np.ndarray:
        if self._host_d_sqrt is None:
            self._host_d_sqrt = self.d_sqrt_dev.cpu().numpy()
        return self._host_d_sqrt

    @property
    def eigen(self):
        """Host EigenBasis (N x m, column order of this pack).  Compatibility
        only — a full D2H copy of V."""
        from .types import EigenBasis
        torch = torch_mod()
        if self.col_map is not None:
            v = self.V.index_select(1, self.col_map.long())
        else:
            v = self.V[:, :self.m]
        return EigenBasis(vectors=np.asfortranarray(v.cpu().numpy()), values=self.values)

    @property
    def laplacian_mode(self):
        from .types import LaplacianMode
        return LaplacianMode.NORMALIZED

    def ensure_graph(self) -> DeviceGraph:
        if self.graph is None:
            if self.image_dev is None:
                raise InvalidParam("this pack has no image attached; pass image= to to_device()")
            self.graph = DeviceGraph.build(self.image_dev, self.lattice, self.beta)
        return self.graph

    def ensure_vtg(self):
        """V^T g for g = d_sqrt/||d_sqrt|| in this pack's column order
        (the per-basis part of fastrw.py:426, reused by every gamma=0 solve)."""
        if self.vtg is None:
            torch = torch_mod()
            vt = column_dot(self.V, self.mr, self.d_sqrt_dev) / self.dnorm
            if self.col_map is not None:
                vt = gather_vector(vt, self.col_map)
            self.vtg = vt
        return self.vtg


def column_dot(V, mr: int, x):
    """out[j] = sum_r V[r, j] x[r] for j < mr (one HBM pass over V)."""
    torch = torch_mod()
    n = V.shape[0]
    line = 64 if n % 64 == 0 else 1
    lat = _lib.Lattice(line, n // line, 1, 4, 0)
    # an empty stencil: the swb_stencil_rayleigh pass with zero coefficients
    # reduces to the column sums norm2 = sum v^2 and vtd = sum v x
    zeros = WORKSPACE.get("zero_coeffs", n * 2 * 8 + n * 8)
    z = zeros[: n * 3 * 8].view(torch.float64)
    z.zero_()
    quad = torch.empty(mr, dtype=torch.float64, device="cuda")
    norm2 = torch.empty_like(quad)
    out = torch.empty_like(quad)
    ws = WORKSPACE.get("stencil", _lib.size("swb_stencil_workspace_bytes", C.byref(lat), mr))
    _lib.call("swb_stencil_rayleigh", C.byref(lat), ptr(V), V.shape[1], 0, 0, n, mr,
              ptr(z[: 2 * n]), ptr(z[2 * n:]), ptr(x), ptr(quad), ptr(norm2), ptr(out),
              ptr(ws), ws.numel(), stream_handle())
    return out


def device_norm(x) -> float:
    """||x||_2 with the deterministic device reduction (one host scalar)."""
    torch = torch_mod()
    ss = torch.empty(1, dtype=torch.float64, device="cuda")
    ws = WORKSPACE.get("sumsq", 256 * 8)
    _lib.call("swb_sumsq", ptr(x), x.numel(), ptr(ss), ptr(ws), ws.numel(), stream_handle())
    return float(np.sqrt(ss.item()))


def gather_vector(v, idx):
    """out[j] = v[idx[j]] via the row-gather kernel (1 column)."""
    torch = torch_mod()
    m = idx.numel()
    out = torch.empty(m, dtype=torch.float64, device="cuda")
    _lib.call("swb_gather_rows", ptr(v), 1, ptr(idx), m, 1, ptr(out), 1, stream_handle())
    return out


def upload_basis(vectors, m: int | None = None):
    """Host N x m basis (any order, f32/f64) -> device row-major f64, ld = round_up(m, 8)."""
    torch = require_cuda()
    vec = np.asarray(vectors)
    n, mm = vec.shape
    if m is None:
        m = mm
    ldv = round_up(max(m, 1), 8)
    V = torch.zeros((n, ldv), dtype=torch.float64, device="cuda")
    if vec.flags.f_contiguous and vec.dtype in (np.float32, np.float64):
        # column-major on the host (the reference layout, f32 memmap or f64):
        # streamed in column blocks through pinned memory, transposed on the
        # device (staging.py) -- no second host copy of the basis
        from .staging import upload_columns
        cm = vec.T          # (mm, n) C-contiguous view: row j = column j

        def fetch(c0, c1, out):
            np.copyto(out.reshape(c1 - c0, n), cm[c0:c1])

        upload_columns(V, ldv, n, m, vec.dtype, fetch)
    elif vec.flags.f_contiguous:
        dev = torch.from_numpy(np.ascontiguousarray(vec[:, :m].T)).to("cuda")
        V[:, :m].copy_(dev.t().to(torch.float64))
    else:
        V[:, :m].copy_(torch.from_numpy(np.ascontiguousarray(vec[:, :m])).to("cuda").to(torch.float64))
    return V


def to_device(pack, image=None, connectivity=None, weight_mode="abs") -> DevicePack:
    """Host pack (reference SpectralPack or ours, or any duck-typed pack) ->
    DevicePack.  ``image`` (optional) is kept on the device for beta updates."""
    if isinstance(pack, DevicePack):
        return pack
    torch = require_cuda()
    eigen = pack.eigen
    values = np.asarray(eigen.values, dtype=np.float64)
    m = values.size
    V = upload_basis(eigen.vectors, m)
    d_sqrt = np.asarray(pack.d_sqrt, dtype=np.float64)
    d_dev = torch.from_numpy(d_sqrt.copy()).to("cuda")
    dims = tuple(int(d) for d in pack.dims)
    lattice = LatticeSpec.make(dims, connectivity, weight_mode)
    img_dev = None
    if image is not None:
        img_dev = torch.from_numpy(np.asarray(image.intensities, dtype=np.float64).copy()).to("cuda")
    prov = getattr(pack, "provenance", None) or PackProvenance(image_hash=b"")
    return DevicePack(V, m, torch.from_numpy(values.copy()).to("cuda"), d_dev,
                      device_norm(d_dev), dims, getattr(pack, "spacing", ()),
                      float(getattr(pack, "beta", 0.0)), prov, lattice, image_dev=img_dev)
