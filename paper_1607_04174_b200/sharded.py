"""z-slab sharding of the hot path across GPUs.

The eigenbasis V is split by rows along the slowest grid axis (z in 3-D, y in
2-D): rank r owns planes [z0, z1) and keeps one halo plane on each interior
side.  The image is replicated; each rank builds the graph (stencil
coefficients) of its slab only (owned units, halos and one unit beyond).

  update   halo exchange of V (one plane per neighbour) -> local difference
           stencil + local symmetric projection P_r = V_r^T W_r -> ONE
           all-reduce of [P | quad | norm2 | V^T d] -> coefficients C computed
           redundantly on every rank -> local rotation V'_r = V_r C.
  solve    owners fill their seed rows of q_s / b_qn / bg / L_s u_s (zero
           elsewhere) [+ the local t_p = V_r^T P^_r for gamma > 0] -> ONE
           all-reduce -> the small seed system solved redundantly -> local
           reconstruction + labels of the owned rows.

Communication goes through a ``Comm``: ``DistComm`` wraps torch.distributed
(NCCL on GPUs, gloo on CPU), ``LocalComm`` runs several shards in one process
(emulation for single-GPU tests).  Local numerics go through a ``Backend``:
``CudaBackend`` calls libspecwalk_b200.so; the CPU test suite supplies a
numpy backend with the same interface so the orchestration is exercised with
world_size 2 over gloo.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .device import WORKSPACE, DeviceGraph, LatticeSpec, ptr, rotate_rows, round_up, stream_handle
from .errors import InvalidParam


# ---------------------------------------------------------------------------
# slab plan
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class SlabPlan:
    """Rows owned by one rank.  A *unit* is one plane (3-D) or line (2-D)."""

    dims: tuple
    world: int
    rank: int
    u0: int          # first owned unit
    u1: int          # one past the last owned unit
    halo_lo: bool
    halo_hi: bool
    unit: int        # rows per unit

    @staticmethod
    def make(dims, world: int, rank: int) -> "SlabPlan":
        dims = tuple(int(d) for d in dims)
        n_units = dims[-1]
        unit = int(np.prod(dims[:-1]))
        if world > n_units:
            raise ValueError(f"cannot split {n_units} units over {world} ranks")
        base, extra = divmod(n_units, world)
        u0 = rank * base + min(rank, extra)
        u1 = u0 + base + (1 if rank < extra else 0)
        return SlabPlan(dims, world, rank, u0, u1, u0 > 0, u1 < n_units, unit)

    @property
    def own_begin(self) -> int:
        return self.u0 * self.unit

    @property
    def own_end(self) -> int:
        return self.u1 * self.unit

    @property
    def row_base(self) -> int:
        return (self.u0 - (1 if self.halo_lo else 0)) * self.unit

    @property
    def local_rows(self) -> int:
        return (self.u1 - self.u0 + int(self.halo_lo) + int(self.halo_hi)) * self.unit

    def own_slice(self) -> slice:
        """Owned rows inside the local buffer."""
        lo = self.unit if self.halo_lo else 0
        return slice(lo, lo + self.own_end - self.own_begin)


# ---------------------------------------------------------------------------
# communication
# ---------------------------------------------------------------------------

class LocalComm:
    """All shards in one process: collectives are plain device copies/sums."""

    def allreduce_sum(self, tensors: list) -> None:
        total = tensors[0].clone()
        for t in tensors[1:]:
            total += t
        for t in tensors:
            t.copy_(total)

    def halo_start(self, shards: list):
        self.halo_exchange(shards)   # in-process copies: nothing to overlap
        return None

    def halo_finish(self, handle) -> None:
        return None

    def halo_exchange(self, shards: list) -> None:
        for a, b in zip(shards, shards[1:]):  # a below b
            u = a.plan.unit
            own_a = a.V[a.plan.own_slice()]
            own_b = b.V[b.plan.own_slice()]
            b.V[:u].copy_(own_a[-u:])        # b's lower halo = a's last owned unit
            a.V[-u:].copy_(own_b[:u])        # a's upper halo = b's first owned unit


class DistComm:
    """torch.distributed collectives (one local shard per process)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def allreduce_sum(self, tensors: list) -> None:
        for t in tensors:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def halo_exchange(self, shards: list) -> None:
        (s,) = shards
        p = s.plan
        u = p.unit
        dist = self.dist
        ops = []
        own = s.V[p.own_slice()]
        if p.halo_lo:
            ops.append(dist.P2POp(dist.isend, own[:u].contiguous(), p.rank - 1, self.group))
            recv_lo = s.V[:u]
            ops.append(dist.P2POp(dist.irecv, recv_lo, p.rank - 1, self.group))
        if p.halo_hi:
            ops.append(dist.P2POp(dist.isend, own[-u:].contiguous(), p.rank + 1, self.group))
            recv_hi = s.V[-u:]
            ops.append(dist.P2POp(dist.irecv, recv_hi, p.rank + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def halo_start(self, shards: list):
        """Post the halo Send/Recv and return without waiting (the transfer
        overlaps the graph build and the interior stencil)."""
        (s,) = shards
        p = s.plan
        u = p.unit
        dist = self.dist
        ops = []
        own = s.V[p.own_slice()]
        if p.halo_lo:
            ops.append(dist.P2POp(dist.isend, own[:u], p.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, s.V[:u], p.rank - 1, self.group))
        if p.halo_hi:
            ops.append(dist.P2POp(dist.isend, own[-u:], p.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, s.V[-u:], p.rank + 1, self.group))
        return dist.batch_isend_irecv(ops) if ops else []

    def halo_finish(self, handle) -> None:
        for req in handle or []:
            req.wait()


class CComm:
    """The same collectives through this library's own NCCL entry points
    (swb_comm_*, csrc/comm.cu) -- the path a C host takes.  One shard per
    process; the communicator's unique id is made by rank 0 and shipped to
    the other ranks over ``bootstrap`` (a torch.distributed group of any
    backend, e.g. gloo), or passed in as ``unique_id`` (128 bytes)."""

    def __init__(self, rank: int, world: int, unique_id: bytes | None = None, bootstrap=None):
        import torch
        self.torch = torch
        lib = _lib.load()
        if unique_id is None:
            buf = (C.c_uint8 * 128)()
            if rank == 0:
                _lib.check(lib.swb_comm_unique_id(buf), "swb_comm_unique_id")
            if world > 1:
                import torch.distributed as dist
                obj = [bytes(buf)]
                dist.broadcast_object_list(obj, src=0, group=bootstrap)
                buf = (C.c_uint8 * 128).from_buffer_copy(obj[0])
            unique_id = bytes(buf)
        self._id = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self.handle = C.c_void_p()
        _lib.check(lib.swb_comm_init(self._id, world, rank, C.byref(self.handle)), "swb_comm_init")
        self.rank, self.world = rank, world
        self.stream = torch.cuda.Stream()

    def close(self) -> None:
        if self.handle:
            _lib.load().swb_comm_destroy(self.handle)
            self.handle = C.c_void_p()

    def allreduce_sum(self, tensors: list) -> None:
        st = stream_handle()
        for t in tensors:
            _lib.call("swb_comm_allreduce_f64", self.handle, ptr(t), ptr(t), t.numel(), st)

    def _halo(self, s, st) -> None:
        p = s.plan
        own_rows = p.own_end - p.own_begin
        _lib.call("swb_comm_halo_exchange", self.handle, ptr(s.V), s.V.stride(0), p.unit, own_rows,
                  int(bool(p.halo_lo)), int(bool(p.halo_hi)), st)

    def halo_exchange(self, shards: list) -> None:
        (s,) = shards
        self._halo(s, stream_handle())

    def halo_start(self, shards: list):
        """Post the Send/Recv on the comm stream (after the current stream's
        work on V); the interior stencil runs meanwhile."""
        (s,) = shards
        cur = self.torch.cuda.current_stream()
        self.stream.wait_stream(cur)
        self._halo(s, C.c_void_p(self.stream.cuda_stream))
        ev = self.torch.cuda.Event()
        ev.record(self.stream)
        return ev

    def halo_finish(self, handle) -> None:
        if handle is not None:
            self.torch.cuda.current_stream().wait_event(handle)


# ---------------------------------------------------------------------------
# local numerics on the GPU
# ---------------------------------------------------------------------------

class CudaBackend:
    """Per-shard local operations through the C ABI (device tensors)."""

    def __init__(self):
        import torch
        self.torch = torch

    # graph: the whole lattice, or (plan given) the shard's slab -- its owned
    # units, the halo units and one more unit each side for their degrees
    def graph(self, image_dev, lattice: LatticeSpec, beta: float, cut_mask=None, plan=None) -> DeviceGraph:
        if plan is None:
            return DeviceGraph.build(image_dev, lattice, beta, cut_mask)
        n_units = lattice.dims[-1]
        return DeviceGraph.build_region(image_dev, lattice, beta, max(0, plan.u0 - 2), min(n_units, plan.u1 + 2),
                                        cut_mask)

    def dnorm_partial(self, graph, plan):
        """sum of d_sqrt^2 over the owned rows (its all-reduce is ||d_sqrt||^2)."""
        t = self.torch
        out = t.empty(1, dtype=t.float64, device="cuda")
        d = graph.d_sqrt_dev[plan.own_begin: plan.own_end]
        ws = WORKSPACE.get("sumsq", 256 * 8)
        _lib.call("swb_sumsq", ptr(d), d.numel(), ptr(out), ptr(ws), ws.numel(), stream_handle())
        return out

    def empty(self, shape, dtype="f64"):
        t = self.torch
        return t.empty(shape, dtype=t.float64 if dtype == "f64" else t.int32, device="cuda")

    def zeros(self, shape):
        return self.torch.zeros(shape, dtype=self.torch.float64, device="cuda")

    def stencil_delta(self, lattice, V, plan, m, g_old, g_new, W, rows=None):
        """Difference pass over owned rows [r0, r1) (default: all owned rows);
        W holds the owned rows (row own_begin at W[0])."""
        t = self.torch
        r0, r1 = rows if rows is not None else (plan.own_begin, plan.own_end)
        quad = t.empty(m, dtype=t.float64, device="cuda")
        norm2 = t.empty_like(quad)
        vtd = t.empty_like(quad)
        lat = lattice.c_struct()
        ws = WORKSPACE.get("stencil", _lib.size("swb_stencil_workspace_bytes", C.byref(lat), m))
        Wr = W[r0 - plan.own_begin:]
        _lib.call("swb_stencil_delta", C.byref(lat), ptr(V), V.shape[1], plan.row_base, r0, r1, m,
                  ptr(g_old.what), ptr(g_old.diag), ptr(g_new.what), ptr(g_new.diag), ptr(g_new.d_sqrt_dev),
                  ptr(Wr), W.shape[1], ptr(quad), ptr(norm2), ptr(vtd), ptr(ws), ws.numel(), stream_handle())
        return quad, norm2, vtd

    def gram_sym(self, X, Y, rows, m):
        t = self.torch
        ldp = round_up(m, 2)
        P = t.empty((m, ldp), dtype=t.float64, device="cuda")
        ws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", rows, m, m))
        _lib.call("swb_gemm_tn", ptr(X), X.shape[1], ptr(Y), Y.shape[1], rows, m, m, 1, ptr(P), ldp, ptr(ws),
                  ws.numel(), stream_handle())
        return P[:, :m]

    def update_coeffs(self, P, lam_old, quad, norm2, m, gap_guard):
        t = self.torch
        ldp = round_up(m, 2)
        Pf = t.zeros((m, ldp), dtype=t.float64, device="cuda")
        Pf[:, :m] = P
        Cm = t.empty((m, ldp), dtype=t.float64, device="cuda")
        lam = t.empty(m, dtype=t.float64, device="cuda")
        order = t.empty(m, dtype=t.int64, device="cuda")
        _lib.call("swb_update_coeffs", 1, ptr(Pf), ldp, ptr(lam_old), ptr(quad), ptr(norm2), m, float(gap_guard),
                  ptr(Cm), ldp, ptr(lam), ptr(order), stream_handle())
        return Cm, lam, order

    def rotate(self, V_own, Cm, m, out_own):
        rotate_rows(V_own, V_own.shape[1], Cm, Cm.shape[1], V_own.shape[0], m, out_own, out_own.shape[1])

    def prefill_rows(self, V, plan, ell, sidx, Cm, m, V_new):
        """V_new[y] = V[y] C for the local rows y the seed kernels read (the
        seed stencil rows, clamped into the local range: every write is the
        correct V' row of a local row, halos included)."""
        t = self.torch
        ell_idx, _, R = ell
        s = int(sidx.numel())
        ldv, st = V.shape[1], stream_handle()
        vg = t.empty((s * R, ldv), dtype=t.float64, device="cuda")
        vp = t.empty_like(vg)
        _lib.call("swb_ell_rows_gather", ptr(V), ldv, plan.row_base, V.shape[0], ptr(ell_idx), ptr(sidx), s, R, m,
                  ptr(vg), st)
        _lib.call("swb_gemm_nn", ptr(vg), ldv, ptr(Cm), Cm.shape[1], s * R, m, m, ptr(vp), ldv, 0, st)
        _lib.call("swb_ell_rows_scatter", ptr(vp), ldv, plan.row_base, V.shape[0], ptr(ell_idx), ptr(sidx), s, R, m,
                  ptr(V_new), st)

    def rotate_extra(self, V_own, Cm, m, out_own, coeff, uraw):
        """out_own = V_own C and uraw = V_own (C coeff) in one rotation (the
        extra columns ride in the INT8 GEMM's padding)."""
        t = self.torch
        k = coeff.shape[1]
        ccf = t.empty((m, round_up(k, 2)), dtype=t.float64, device="cuda")
        _lib.call("swb_gemm_nn", ptr(Cm), Cm.shape[1], ptr(coeff), k, m, coeff.shape[0], k, ptr(ccf), ccf.shape[1], 0,
                  stream_handle())
        c_aug = t.empty((m, round_up(m + k, 2)), dtype=t.float64, device="cuda")
        _lib.call("swb_build_caug", ptr(Cm), Cm.shape[1], ptr(ccf), ccf.shape[1], m, k, ptr(c_aug), c_aug.shape[1],
                  stream_handle())
        rotate_rows(V_own, V_own.shape[1], c_aug, c_aug.shape[1], V_own.shape[0], m, out_own, out_own.shape[1],
                    m2=m + k, out2=uraw, ldo2=k)

    def finalize(self, uraw, plan, k, extra, dnorm, d_sqrt, sidx, slab, s, want_u=False):
        t = self.torch
        rows = plan.own_end - plan.own_begin
        ldu = round_up(k, 2)
        labels = t.empty(rows, dtype=t.int32, device="cuda")
        top2 = t.empty(rows, dtype=t.float64, device="cuda")
        U = t.empty((rows, ldu), dtype=t.float64, device="cuda") if (want_u or k > 8) else None
        src, lds = uraw, k
        if k > 8:
            U[:, :k].copy_(uraw)
            src, lds = U, ldu
        _lib.call("swb_finalize_label", plan.own_begin, plan.own_end, k, ptr(src), lds, ptr(extra), float(dnorm),
                  ptr(d_sqrt), ptr(U), ldu, ptr(labels), ptr(top2), stream_handle())
        _lib.call("swb_apply_seeds", ptr(sidx), ptr(slab), s, plan.own_begin, plan.own_end, k, ptr(U), ldu,
                  ptr(labels), ptr(top2), stream_handle())
        return labels, top2, (U[:, :k] if U is not None else None)

    def rotate_vector(self, vtd, Cm, m):
        t = self.torch
        ldp = Cm.shape[1]
        row = t.zeros((1, ldp), dtype=t.float64, device="cuda")
        row[0, :m] = vtd
        out = t.empty((1, ldp), dtype=t.float64, device="cuda")
        _lib.call("swb_gemm_nn", ptr(row), ldp, ptr(Cm), ldp, 1, m, m, ptr(out), ldp, 0, stream_handle())
        return out[0, :m].clone()

    def seed_rows(self, graph: DeviceGraph, sidx, s):
        t = self.torch
        R = 2 * graph.lattice.ndir + 1
        ell_idx = t.empty((max(s, 1), R), dtype=t.int64, device="cuda")
        ell_val = t.empty((max(s, 1), R), dtype=t.float64, device="cuda")
        lat = graph.lattice.c_struct()
        _lib.call("swb_seed_rows", C.byref(lat), ptr(graph.what), ptr(graph.diag), ptr(sidx), s, ptr(ell_idx),
                  ptr(ell_val), stream_handle())
        return ell_idx, ell_val, R

    def seed_project(self, V, plan, m, sidx, slab, s, ell, d_sqrt, dnorm, k):
        t = self.torch
        ell_idx, ell_val, R = ell
        ldq = round_up(m, 2)
        q_s = t.zeros((s, ldq), dtype=t.float64, device="cuda")
        b_qn = t.zeros((s, ldq), dtype=t.float64, device="cuda")
        bg = t.empty(s, dtype=t.float64, device="cuda")
        lsu = t.empty((s, k), dtype=t.float64, device="cuda")
        dsq = t.empty(s, dtype=t.float64, device="cuda")
        _lib.call("swb_seed_project", ptr(V), V.shape[1], plan.row_base, plan.own_begin, plan.own_end, m, None,
                  ptr(sidx), ptr(slab), s, ptr(ell_idx), ptr(ell_val), R, ptr(d_sqrt), float(dnorm), k, ptr(q_s),
                  ldq, ptr(b_qn), ptr(bg), ptr(lsu), ptr(dsq), stream_handle())
        return q_s, b_qn, bg, lsu, dsq

    def prior_projection(self, V_own, plan, m, priors_own, d_sqrt, sidx, s, k):
        t = self.torch
        rows = plan.own_end - plan.own_begin
        ldt = round_up(k, 2)
        ph = t.empty((rows, ldt), dtype=t.float64, device="cuda")
        _lib.call("swb_prior_hat", ptr(priors_own), priors_own.stride(0), plan.own_begin, plan.own_end, k,
                  ptr(d_sqrt), ptr(sidx), s, ptr(ph), ldt, stream_handle())
        tp = t.empty((m, ldt), dtype=t.float64, device="cuda")
        ws = WORKSPACE.get("gemm_tn", _lib.size("swb_gemm_tn_workspace_bytes", rows, m, k))
        _lib.call("swb_gemm_tn", ptr(V_own), V_own.shape[1], ptr(ph), ldt, rows, m, k, 0, ptr(tp), ldt, ptr(ws),
                  ws.numel(), stream_handle())
        return tp

    def small_solve(self, gamma, s, m, k, q_s, b_qn, bg, lsu, dsq, dnorm, slab, values, vtg, t_p):
        t = self.torch
        coeff = t.empty((m, k), dtype=t.float64, device="cuda")
        extra = t.empty(k, dtype=t.float64, device="cuda") if gamma == 0 else None
        rcond = t.empty(1, dtype=t.float64, device="cuda")
        ws = WORKSPACE.get("small_solve", _lib.size("swb_small_solve_workspace_bytes", s, m, k))
        ldq = q_s.shape[1] if s else round_up(m, 2)
        ldt = t_p.shape[1] if t_p is not None else round_up(k, 2)
        # as api.solve_fast: the condition estimate runs on the side stream,
        # overlapping the reconstruction; join_side() joins it
        from .api import _side_stream
        side, ev = _side_stream()
        t.cuda.current_stream().wait_stream(side)   # a previous shard's estimate still reads the workspace
        ev.record()
        _lib.call("swb_small_solve_ex", float(gamma), s, m, k, ptr(q_s), ptr(b_qn), ldq, ptr(bg), ptr(lsu), ptr(dsq),
                  float(dnorm), ptr(slab), ptr(values), ptr(vtg), ptr(t_p), ldt, ptr(coeff), ptr(extra), ptr(rcond),
                  ptr(ws), ws.numel(), stream_handle(), C.c_void_p(side.cuda_stream), C.c_void_p(ev.cuda_event))
        return coeff, extra, rcond

    def join_side(self):
        from .api import _side_stream
        self.torch.cuda.current_stream().wait_stream(_side_stream()[0])

    def reconstruct(self, V, plan, m, coeff, extra, dnorm, d_sqrt, k, sidx, slab, s, want_u=False):
        t = self.torch
        rows = plan.own_end - plan.own_begin
        ldu = round_up(k, 2)
        labels = t.empty(rows, dtype=t.int32, device="cuda")
        top2 = t.empty(rows, dtype=t.float64, device="cuda")
        U = t.empty((rows, ldu), dtype=t.float64, device="cuda") if (want_u or k > 8) else None
        _lib.call("swb_reconstruct_label", ptr(V), V.shape[1], plan.row_base, plan.own_begin, plan.own_end, m,
                  ptr(coeff), ptr(extra), float(dnorm), ptr(d_sqrt), k, ptr(U), ldu, ptr(labels), ptr(top2),
                  stream_handle())
        _lib.call("swb_apply_seeds", ptr(sidx), ptr(slab), s, plan.own_begin, plan.own_end, k, ptr(U), ldu,
                  ptr(labels), ptr(top2), stream_handle())
        return labels, top2, (U[:, :k] if U is not None else None)

    def to_host(self, x):
        return x.cpu().numpy()

    def seeds(self, seed_idx, seed_lab):
        t = self.torch
        return (t.from_numpy(np.ascontiguousarray(seed_idx, dtype=np.int64)).to("cuda"),
                t.from_numpy(np.ascontiguousarray(seed_lab, dtype=np.int32)).to("cuda"))

    def column_dot(self, V_own, x_own, m):
        from .device import column_dot
        return column_dot(V_own, m, x_own)


# ---------------------------------------------------------------------------
# shard state + the sharded update / solve
# ---------------------------------------------------------------------------

@dataclass
class Shard:
    plan: SlabPlan
    V: object                  # local rows (halo + owned) x ldv
    m: int
    values: object             # replicated eigenvalues (m)
    lattice: LatticeSpec
    image: object              # replicated intensities (backend array)
    graph: object              # replicated graph at the current beta
    beta: float
    vtg: object = None         # replicated V^T g (current column order)
    extra: dict = field(default_factory=dict)

    def own(self):
        return self.V[self.plan.own_slice()]


def _mark(name):
    from . import api
    if api.TIMER is not None:
        api.TIMER.mark(name)


def sum_in_order(xs):
    """x0 + x1 + ... left to right (a fixed summation order)."""
    total = xs[0]
    for x in xs[1:]:
        total = total + x
    return total


def sharded_update(shards: list, comm, backend, new_beta: float, gap_guard: float = 0.5, cut_mask=None):
    """First-order basis update of every local shard (one all-reduce)."""
    staged = _update_to_coeffs(shards, comm, backend, new_beta, gap_guard, cut_mask)
    for st in staged:
        _update_finish(backend, new_beta, st)
    return shards


def _update_finish(backend, new_beta, st, extra_cols=None):
    """Rotation of the owned rows and the shard's new state; ``extra_cols``
    (update_and_solve): (C coeff, out2) -- the extra products V (C coeff)."""
    sh, g_new, buf, Cm, lam, order, vtd = st
    m = sh.m
    V_new = buf
    _mark("rotate")
    if extra_cols is None:
        backend.rotate(sh.own(), Cm, m, V_new[sh.plan.own_slice()])
    else:
        backend.rotate_extra(sh.own(), Cm, m, V_new[sh.plan.own_slice()], *extra_cols)
    _mark("update_tail")
    if V_new.shape[1] > m:
        V_new[:, m:] = 0.0
    sh.vtg = backend.rotate_vector(vtd, Cm, m) / g_new.dnorm
    sh.extra["spare"] = sh.V
    sh.V = V_new
    sh.values = lam
    sh.graph = g_new
    sh.beta = float(new_beta)
    sh.extra["order"] = order
    sh.extra["C"] = Cm


def _update_to_coeffs(shards: list, comm, backend, new_beta: float, gap_guard: float, cut_mask):
    """The update through the coefficients C (halo exchange, stencil,
    projection, the one all-reduce): per shard (sh, g_new, buf, C, lam,
    order, V^T d)."""
    # the halo transfer overlaps the graph build and the interior stencil;
    # only the first / last owned unit needs the received planes
    _mark("halo")
    handle = comm.halo_start(shards)
    staged = []
    for sh in shards:
        _mark("graph")
        g_new = backend.graph(sh.image, sh.lattice, new_beta, cut_mask, plan=sh.plan)
        # ping-pong: the spare local buffer holds W = dL V in its owned rows,
        # then V' (W is dead after P); the old V becomes the next spare
        buf = sh.extra.pop("spare", None)
        if buf is None or tuple(buf.shape) != tuple(sh.V.shape):
            buf = backend.empty(tuple(sh.V.shape))
        W = buf[sh.plan.own_slice()]
        p_ = sh.plan
        lo = p_.own_begin + (p_.unit if p_.halo_lo else 0)
        hi = p_.own_end - (p_.unit if p_.halo_hi else 0)
        _mark("stencil")
        inner = backend.stencil_delta(sh.lattice, sh.V, p_, sh.m, sh.graph, g_new, W, rows=(lo, hi)) \
            if hi > lo else None
        staged.append((sh, g_new, buf, W, lo, hi, inner))
    comm.halo_finish(handle)
    parts = []
    for sh, g_new, buf, W, lo, hi, inner in staged:
        p_ = sh.plan
        pieces = [inner] if inner is not None else []
        if lo > p_.own_begin:
            pieces.append(backend.stencil_delta(sh.lattice, sh.V, p_, sh.m, sh.graph, g_new, W,
                                                rows=(p_.own_begin, lo)))
        if p_.own_end > max(hi, lo):
            pieces.append(backend.stencil_delta(sh.lattice, sh.V, p_, sh.m, sh.graph, g_new, W,
                                                rows=(max(hi, lo), p_.own_end)))
        quad, norm2, vtd = (sum_in_order([pc[i] for pc in pieces]) for i in range(3))
        _mark("project")
        P = backend.gram_sym(sh.own(), W, sh.plan.own_end - sh.plan.own_begin, sh.m)
        _mark("pack")
        m = sh.m
        flat = backend.zeros((m * m + 3 * m + 1,))
        flat[: m * m] = P.reshape(-1)
        flat[m * m: m * m + m] = quad
        flat[m * m + m: m * m + 2 * m] = norm2
        flat[m * m + 2 * m: m * m + 3 * m] = vtd
        flat[m * m + 3 * m:] = backend.dnorm_partial(g_new, p_)
        parts.append((sh, g_new, buf, flat))
    _mark("allreduce")
    comm.allreduce_sum([p[3] for p in parts])
    out = []
    for sh, g_new, buf, flat in parts:
        _mark("coeffs")
        m = sh.m
        P = flat[: m * m].reshape(m, m)
        quad, norm2, vtd = flat[m * m: m * m + m], flat[m * m + m: m * m + 2 * m], flat[m * m + 2 * m: m * m + 3 * m]
        g_new.dnorm = float(flat[m * m + 3 * m:].sum().item() ** 0.5)   # global ||d_sqrt||
        Cm, lam, order = backend.update_coeffs(P, sh.values, quad, norm2, m, gap_guard)
        out.append((sh, g_new, buf, Cm, lam, order, vtd))
    return out


def sharded_update_and_solve(shards: list, comm, backend, new_beta: float, seed_idx, seed_lab, k: int,
                             gap_guard: float = 0.5, cut_mask=None, want_u: bool = False):
    """sharded_update + sharded_solve (gamma = 0) with one pass less over the
    basis, as api.update_and_solve: the seed system is solved before the
    rotation on the V' rows the seed kernels read (each rank forms its owned
    ones as V[rows] C), and its coefficients ride as extra columns of the
    rotation, V (C coeff) = V' coeff; a row-wise finalize gives the labels.
    Two all-reduces, as the separate calls.  Returns what sharded_solve does."""
    seed_idx, seed_lab = _sorted_seeds(seed_idx, seed_lab)
    s = int(len(seed_idx))
    if s == 0:
        raise InvalidParam("update_and_solve needs seeds (gamma = 0)")
    staged = _update_to_coeffs(shards, comm, backend, new_beta, gap_guard, cut_mask)
    _mark("solve_seeds")
    solve_in = []
    for sh, g_new, buf, Cm, lam, order, vtd in staged:
        m = sh.m
        sidx, slab = backend.seeds(seed_idx, seed_lab)
        ell = backend.seed_rows(g_new, sidx, s)
        backend.prefill_rows(sh.V, sh.plan, ell, sidx, Cm, m, buf)
        q_s, b_qn, bg, lsu, dsq = backend.seed_project(buf, sh.plan, m, sidx, slab, s, ell, g_new.d_sqrt_dev,
                                                       g_new.dnorm, k)
        parts = [q_s, b_qn, bg, lsu, dsq]
        sizes = [x.numel() for x in parts]
        flat = backend.zeros((sum(sizes),))
        o = 0
        for x, n in zip(parts, sizes):
            flat[o:o + n] = x.reshape(-1)
            o += n
        solve_in.append((sidx, slab, parts, sizes, flat))
    _mark("solve_allreduce")
    comm.allreduce_sum([si[4] for si in solve_in])
    out = []
    for st, (sidx, slab, parts, sizes, flat) in zip(staged, solve_in):
        sh, g_new, buf, Cm, lam, order, vtd = st
        _mark("solve_system")
        o = 0
        views = []
        for x, n in zip(parts, sizes):
            views.append(flat[o:o + n].reshape(x.shape))
            o += n
        q_s, b_qn, bg, lsu, dsq = views
        m = sh.m
        vtg = backend.rotate_vector(vtd, Cm, m) / g_new.dnorm
        coeff, extra, rcond = backend.small_solve(0.0, s, m, k, q_s, b_qn, bg, lsu, dsq, g_new.dnorm, slab, lam,
                                                  vtg, None)
        uraw = backend.empty((sh.plan.own_end - sh.plan.own_begin, k))
        _update_finish(backend, new_beta, st, extra_cols=(coeff, uraw))
        _mark("solve_finalize")
        labels, top2, U = backend.finalize(uraw, sh.plan, k, extra, g_new.dnorm, g_new.d_sqrt_dev, sidx, slab, s,
                                           want_u)
        out.append((labels, top2, U, rcond))
    if hasattr(backend, "join_side"):
        backend.join_side()
    _mark("solve_end")
    return out


def sharded_init_vtg(shards: list, comm, backend):
    """V^T g (g = d_sqrt / ||d_sqrt||) of the current basis: local partial
    over the owned rows + one all-reduce."""
    dn = [backend.dnorm_partial(sh.graph, sh.plan) for sh in shards]
    comm.allreduce_sum(dn)
    for sh, d in zip(shards, dn):
        sh.graph.dnorm = float(d.sum().item() ** 0.5)   # global ||d_sqrt|| (slab graphs hold their part)
    parts = [backend.column_dot(sh.own(), sh.graph.d_sqrt_dev[sh.plan.own_begin: sh.plan.own_end], sh.m)
             for sh in shards]
    comm.allreduce_sum(parts)
    for sh, v in zip(shards, parts):
        sh.vtg = v / sh.graph.dnorm
    return shards


def _sorted_seeds(seed_idx, seed_lab):
    """Seeds sorted ascending (labels permuted alike); duplicates are an error
    (SeedPartition's contract, graphs.py:51-98)."""
    idx = seed_idx.cpu().numpy() if hasattr(seed_idx, "cpu") else np.asarray(seed_idx)
    lab = seed_lab.cpu().numpy() if hasattr(seed_lab, "cpu") else np.asarray(seed_lab)
    idx = idx.astype(np.int64, copy=False).ravel()
    lab = lab.astype(np.int64, copy=False).ravel()
    if idx.size > 1 and np.any(np.diff(idx) <= 0):
        o = np.argsort(idx, kind="stable")
        idx, lab = idx[o], lab[o]
        if np.any(np.diff(idx) == 0):
            raise InvalidParam("duplicate seed index")
    return idx, lab


def sharded_solve(shards: list, comm, backend, seed_idx, seed_lab, k: int, gamma: float = 0.0, priors=None,
                  want_u: bool = False):
    """Reduced-basis RW solve of every local shard (one all-reduce).

    ``priors`` (gamma > 0): per shard, the owned rows (backend array).
    Returns per shard (labels_own, top2_own, U_own or None, rcond).
    Seeds may come in any order (the seed kernels need them sorted and
    unique: they are sorted here, duplicates raise InvalidParam)."""
    seed_idx, seed_lab = _sorted_seeds(seed_idx, seed_lab)
    s = int(len(seed_idx))
    staged = []
    _mark("solve_seeds")
    for i, sh in enumerate(shards):
        m = sh.m
        sidx, slab = backend.seeds(seed_idx, seed_lab)
        ell = backend.seed_rows(sh.graph, sidx, s)
        q_s, b_qn, bg, lsu, dsq = backend.seed_project(sh.V, sh.plan, m, sidx, slab, s, ell, sh.graph.d_sqrt_dev,
                                                       sh.graph.dnorm, k)
        parts = [q_s, b_qn, bg, lsu, dsq]
        if gamma > 0:
            parts.append(backend.prior_projection(sh.own(), sh.plan, m, priors[i], sh.graph.d_sqrt_dev, sidx, s, k))
        sizes = [x.numel() for x in parts]
        flat = backend.zeros((sum(sizes),))
        o = 0
        for x, n in zip(parts, sizes):
            flat[o:o + n] = x.reshape(-1)
            o += n
        staged.append((sh, sidx, slab, parts, sizes, flat))
    _mark("solve_allreduce")
    comm.allreduce_sum([st[5] for st in staged])
    _mark("solve_system")
    out = []
    for sh, sidx, slab, parts, sizes, flat in staged:
        o = 0
        views = []
        for x, n in zip(parts, sizes):
            views.append(flat[o:o + n].reshape(x.shape))
            o += n
        q_s, b_qn, bg, lsu, dsq = views[:5]
        tp = views[5] if gamma > 0 else None
        m = sh.m
        coeff, extra, rcond = backend.small_solve(gamma, s, m, k, q_s, b_qn, bg, lsu, dsq, sh.graph.dnorm, slab,
                                                  sh.values, sh.vtg, tp)
        _mark("solve_reconstruct")
        labels, top2, U = backend.reconstruct(sh.V, sh.plan, m, coeff, extra, sh.graph.dnorm, sh.graph.d_sqrt_dev,
                                              k, sidx, slab, s, want_u)
        out.append((labels, top2, U, rcond))
    if hasattr(backend, "join_side"):
        backend.join_side()
    _mark("solve_end")
    return out


def make_shards_from_global(V_global, values, d_sqrt_unused, lattice: LatticeSpec, image_dev, beta: float,
                            world: int, ranks=None, backend=None):
    """Split a resident global basis into slab shards (tests / emulation)."""
    backend = backend or CudaBackend()
    graph = backend.graph(image_dev, lattice, beta)
    ranks = range(world) if ranks is None else ranks
    shards = []
    for r in ranks:
        plan = SlabPlan.make(lattice.dims, world, r)
        V = V_global[plan.row_base: plan.row_base + plan.local_rows].clone()
        shards.append(Shard(plan, V, int(values.numel() if hasattr(values, "numel") else len(values)), values.clone(),
                            lattice, image_dev, graph, beta))
    return shards


def gather_rows(shard_rows: list):
    """Concatenate per-shard owned-row results (emulation / rank 0 gather)."""
    import torch
    return torch.cat(shard_rows)
