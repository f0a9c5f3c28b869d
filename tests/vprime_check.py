"""Updated-eigenvector (V') comparison used by the GPU parity tests.

north_star: "updated eigenvectors (up to sign) must agree within 1e-9
relative in FP64".  Each column a of the GPU V' is compared with the
oracle's column b as ‖a − s·b‖₂ / ‖b‖₂ with s = sign(a·b).

Columns whose stored eigenvalues are within ``cluster_gap`` of each other are
coupled by divided differences P_ji / (λ_i − λ_j) that amplify the last-ulp
differences of P, so for such groups the invariant object is the span, not
the individual vector: the group is compared by the sine of the largest
principal angle between the two spans (‖Q_a − Q_b Q_bᵀ Q_a‖₂).

The report also carries the largest elementwise relative error over the
entries with |b| > 1e-3·max|b| of their column — the quantity the INT8
digit-product rotation bounds only row-max-relatively.
"""

from __future__ import annotations

import json
import os

import numpy as np


def _groups(lam_old: np.ndarray, order: np.ndarray, cluster_gap: float):
    """Output-column groups whose stored λ are chained by gaps < cluster_gap."""
    m = lam_old.size
    srt = np.argsort(lam_old, kind="stable")
    inv = np.empty(m, dtype=np.int64)
    inv[np.asarray(order)] = np.arange(m)       # original column -> output column
    groups, cur = [], [srt[0]]
    for a, b in zip(srt[:-1], srt[1:]):
        if abs(lam_old[b] - lam_old[a]) < cluster_gap:
            cur.append(b)
        else:
            groups.append(cur)
            cur = [b]
    groups.append(cur)
    return [sorted(int(inv[i]) for i in g) for g in groups]


def compare_vprime(Vg: np.ndarray, Vo: np.ndarray, lam_old, order, *, tol=1e-9,
                   cluster_gap=1e-6, label="", assert_ok=True):
    Vg = np.asarray(Vg, dtype=np.float64)
    Vo = np.asarray(Vo, dtype=np.float64)
    assert Vg.shape == Vo.shape
    lam_old = np.asarray(lam_old, dtype=np.float64)
    worst_col = 0.0
    worst_span = 0.0
    worst_elem = 0.0
    n_single = n_grouped = 0
    for g in _groups(lam_old, order, cluster_gap):
        if len(g) == 1:
            j = g[0]
            a, b = Vg[:, j], Vo[:, j]
            s = 1.0 if a @ b >= 0 else -1.0
            nb = np.linalg.norm(b)
            err = np.linalg.norm(a - s * b) / nb
            worst_col = max(worst_col, err)
            big = np.abs(b) > 1e-3 * np.abs(b).max()
            if big.any():
                worst_elem = max(worst_elem, float(np.max(np.abs(a[big] - s * b[big]) / np.abs(b[big]))))
            n_single += 1
        else:
            qa, _ = np.linalg.qr(Vg[:, g])
            qb, _ = np.linalg.qr(Vo[:, g])
            sin = np.linalg.norm(qa - qb @ (qb.T @ qa), 2)
            worst_span = max(worst_span, float(sin))
            n_grouped += len(g)
    rep = {"label": label, "shape": list(Vg.shape), "max_col_rel_err": float(worst_col),
           "max_group_sin_angle": float(worst_span), "max_elem_rel_err_above_1e-3max": float(worst_elem),
           "columns_compared_individually": n_single, "columns_in_clusters": n_grouped,
           "cluster_gap": cluster_gap, "tol": tol}
    path = os.environ.get("SWB_PARITY_REPORT")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(rep) + "\n")
    print("V' parity", json.dumps(rep))
    if assert_ok:
        assert worst_col <= tol, rep
        assert worst_span <= tol, rep
        assert worst_elem <= tol, rep
    return rep
