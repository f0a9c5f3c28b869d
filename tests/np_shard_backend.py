"""Numpy backend for the sharded orchestration (TEST INFRASTRUCTURE).

Implements the local-shard interface of paper_1607_04174_b200.sharded.CudaBackend
on CPU torch tensors with numpy/scipy, built from the oracle's restatement
of the reference (oracle/rw_oracle.py).  It lets the z-slab orchestration
(halo exchange, the one all-reduce per phase) run with world_size > 1 over
gloo on a machine without a GPU.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import torch

from oracle import rw_oracle as O


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))


class NumpyBackend:
    def graph(self, image, lattice, beta, cut_mask=None, plan=None):
        img = image.numpy() if hasattr(image, "numpy") else np.asarray(image)
        lap = O.build_laplacian(img, lattice.dims, beta, lattice.weight_mode, lattice.connectivity,
                                cut_edges=cut_mask)
        return SimpleNamespace(lap=lap, d_sqrt_dev=_t(lap.d_sqrt), dnorm=float(np.linalg.norm(lap.d_sqrt)),
                               lattice=lattice)

    def dnorm_partial(self, graph, plan):
        d = graph.lap.d_sqrt[plan.own_begin: plan.own_end]
        return _t(np.array([np.dot(d, d)]))

    def empty(self, shape, dtype="f64"):
        return torch.zeros(shape, dtype=torch.float64)

    def zeros(self, shape):
        return torch.zeros(shape, dtype=torch.float64)

    def _cols(self, plan, V):
        return slice(plan.row_base, plan.row_base + V.shape[0])

    def stencil_delta(self, lattice, V, plan, m, g_old, g_new, W, rows=None):
        r0, r1 = rows if rows is not None else (plan.own_begin, plan.own_end)
        rows = slice(r0, r1)
        cols = self._cols(plan, V)
        Vl = V[:, :m].numpy()
        dL = (g_new.lap.matrix - g_old.lap.matrix).tocsr()[rows][:, cols]
        Ln = g_new.lap.matrix[rows][:, cols]
        W[r0 - plan.own_begin: r1 - plan.own_begin, :m] = _t(dL @ Vl)
        Vo = Vl[r0 - plan.row_base: r1 - plan.row_base]
        quad = np.einsum("ij,ij->j", Vo, Ln @ Vl)
        norm2 = np.einsum("ij,ij->j", Vo, Vo)
        vtd = Vo.T @ g_new.lap.d_sqrt[rows]
        return _t(quad), _t(norm2), _t(vtd)

    def gram_sym(self, X, Y, rows, m):
        P = X[:, :m].numpy().T @ Y[:, :m].numpy()
        return _t(0.5 * (P + P.T))

    def update_coeffs(self, P, lam_old, quad, norm2, m, gap_guard):
        lam_hat = np.maximum(quad.numpy() / norm2.numpy(), 0.0)
        Cf, lam, order = O.update_coefficients(P.numpy(), lam_old.numpy(), lam_hat, gap_guard)
        return _t(Cf), _t(lam), torch.from_numpy(order)

    def rotate(self, V_own, Cm, m, out_own):
        out_own[:, :m] = _t(V_own[:, :m].numpy() @ Cm[:, :m].numpy())

    def prefill_rows(self, V, plan, ell, sidx, Cm, m, V_new):
        # the numpy seed projection reads owned rows only: form them all
        own = slice(plan.own_begin - plan.row_base, plan.own_end - plan.row_base)
        V_new[own, :m] = _t(V[own, :m].numpy() @ Cm[:, :m].numpy())

    def rotate_extra(self, V_own, Cm, m, out_own, coeff, uraw):
        Vo = V_own[:, :m].numpy()
        out_own[:, :m] = _t(Vo @ Cm[:, :m].numpy())
        uraw[:] = _t(Vo @ (Cm[:, :m].numpy()[:, :coeff.shape[0]] @ coeff.numpy()))

    def finalize(self, uraw, plan, k, extra, dnorm, d_sqrt, sidx, slab, s, want_u=False):
        d = d_sqrt.numpy()[plan.own_begin: plan.own_end]
        u = uraw.numpy() + np.outer(d / dnorm, extra.numpy())
        u = u / d[:, None]
        idx = sidx.numpy()
        own = (idx >= plan.own_begin) & (idx < plan.own_end)
        u = O.finalize(u, idx[own] - plan.own_begin, slab.numpy()[own], k)
        return torch.from_numpy(O.hard_labels(u)), None, _t(u)

    def rotate_vector(self, vtd, Cm, m):
        return _t(Cm[:, :m].numpy().T @ vtd.numpy())

    def column_dot(self, V_own, x_own, m):
        return _t(V_own[:, :m].numpy().T @ x_own.numpy())

    def seeds(self, seed_idx, seed_lab):
        return (torch.from_numpy(np.asarray(seed_idx, dtype=np.int64)),
                torch.from_numpy(np.asarray(seed_lab, dtype=np.int32)))

    def seed_rows(self, graph, sidx, s):
        return graph.lap.matrix

    def seed_project(self, V, plan, m, sidx, slab, s, ell, d_sqrt, dnorm, k):
        csr = ell
        d = d_sqrt.numpy()
        idx = sidx.numpy()
        lab = slab.numpy()
        pos = {int(v): i for i, v in enumerate(idx)}
        q_s = np.zeros((s, m))
        b_qn = np.zeros((s, m))
        bg = np.zeros(s)
        lsu = np.zeros((s, k))
        dsq = np.zeros(s)
        Vl = V.numpy()
        for i, si in enumerate(idx):
            owner = plan.own_begin <= si < plan.own_end
            a, b = csr.indptr[si], csr.indptr[si + 1]
            for y, val in zip(csr.indices[a:b], csr.data[a:b]):
                t = pos.get(int(y))
                if t is not None:
                    if owner:
                        lsu[i, lab[t]] += val * d[y]
                else:
                    if owner:
                        bg[i] += val * (d[y] / dnorm)
                    if plan.own_begin <= y < plan.own_end:
                        b_qn[i] += val * Vl[y - plan.row_base, :m]
            if owner:
                q_s[i] = Vl[si - plan.row_base, :m]
                dsq[i] = d[si]
        return _t(q_s), _t(b_qn), _t(bg), _t(lsu), _t(dsq)

    def prior_projection(self, V_own, plan, m, priors_own, d_sqrt, sidx, s, k):
        ph = priors_own.numpy() * d_sqrt.numpy()[plan.own_begin: plan.own_end, None]
        for si in sidx.numpy():
            if plan.own_begin <= si < plan.own_end:
                ph[si - plan.own_begin] = 0.0
        return _t(V_own[:, :m].numpy().T @ ph)

    def small_solve(self, gamma, s, m, k, q_s, b_qn, bg, lsu, dsq, dnorm, slab, values, vtg, tp):
        q_s, b_qn, bg, lsu, dsq = (x.numpy() for x in (q_s, b_qn, bg, lsu, dsq))
        lab = slab.numpy()
        w = O.spectral_weights(values.numpy()[:m], gamma)
        u_s = np.zeros((s, k))
        u_s[np.arange(s), lab] = dsq
        if gamma > 0:
            t_p = tp.numpy()
            if s:
                a = np.eye(s) - (b_qn * w) @ q_s.T
                rhs = lsu + gamma * u_s + gamma * (b_qn * w) @ t_p
                f, rc = O.dense_solve(a, rhs)
                coeff = w[:, None] * (q_s.T @ f + gamma * t_p)
            else:
                coeff, rc = w[:, None] * (gamma * t_p), 1.0
            return _t(coeff), None, rc
        g_s = dsq / dnorm
        gq = vtg.numpy()[:m] - q_s.T @ g_s
        a = np.empty((s + 1, s + 1))
        a[:s, :s] = np.eye(s) - (b_qn * w) @ q_s.T
        a[:s, s] = -bg
        a[s, :s] = -(gq * w) @ q_s.T
        a[s, s] = g_s @ g_s
        rhs = np.empty((s + 1, k))
        rhs[:s] = lsu
        rhs[s] = g_s @ u_s
        sol, rc = O.dense_solve(a, rhs)
        return _t(w[:, None] * (q_s.T @ sol[:s])), _t(sol[s]), rc

    def reconstruct(self, V, plan, m, coeff, extra, dnorm, d_sqrt, k, sidx, slab, s, want_u=False):
        Vo = V[plan.own_slice(), :m].numpy()
        d = d_sqrt.numpy()[plan.own_begin: plan.own_end]
        u = Vo @ coeff.numpy()
        if extra is not None:
            u += np.outer(d / dnorm, extra.numpy())
        u = u / d[:, None]
        idx = sidx.numpy()
        own = (idx >= plan.own_begin) & (idx < plan.own_end)
        u = O.finalize(u, idx[own] - plan.own_begin, slab.numpy()[own], k)
        return torch.from_numpy(O.hard_labels(u)), None, _t(u)
