"""Seed-system solvers at small n: swb_small_dense_solve (one launch) vs the
blocked swb_lu_factor + swb_lu_solve + swb_lu_rcond, CUDA-event timed."""
import sys

import numpy as np
import torch

from paper_1607_04174_b200 import _lib
from paper_1607_04174_b200.device import ptr, round_up

for n in [int(a) for a in (sys.argv[1:] or ["41", "151"])]:
    rng = np.random.default_rng(n)
    A = np.eye(n) * 3 + rng.standard_normal((n, n)) / np.sqrt(n)
    lda = round_up(n, 8)
    A0 = torch.zeros((n, lda), dtype=torch.float64, device="cuda")
    A0[:, :n] = torch.from_numpy(A)
    Ad, Bd = A0.clone(), torch.randn(n, 4, dtype=torch.float64, device="cuda")
    piv = torch.empty(n, dtype=torch.int32, device="cuda")
    an = torch.empty(1, dtype=torch.float64, device="cuda")
    rc = torch.empty(1, dtype=torch.float64, device="cuda")
    ws = torch.empty(_lib.size("swb_lu_workspace_bytes", n), dtype=torch.uint8, device="cuda")
    rws = torch.empty(_lib.size("swb_lu_solve_workspace_bytes", n, 4), dtype=torch.uint8, device="cuda")

    def small():
        Ad.copy_(A0)
        _lib.call("swb_small_dense_solve", ptr(Ad), n, lda, ptr(piv), ptr(Bd), 4, 4, ptr(an), ptr(rc), None)

    def small_norc():
        Ad.copy_(A0)
        _lib.call("swb_small_dense_solve", ptr(Ad), n, lda, ptr(piv), ptr(Bd), 4, 4, ptr(an), None, None)

    def blocked_norc():
        Ad.copy_(A0)
        _lib.call("swb_lu_factor", ptr(Ad), n, lda, ptr(piv), ptr(an), ptr(ws), ws.numel(), None)
        _lib.call("swb_lu_solve", ptr(Ad), n, lda, ptr(piv), ptr(Bd), 4, 4, ptr(rws), rws.numel(), None)

    def blocked():
        Ad.copy_(A0)
        _lib.call("swb_lu_factor", ptr(Ad), n, lda, ptr(piv), ptr(an), ptr(ws), ws.numel(), None)
        _lib.call("swb_lu_solve", ptr(Ad), n, lda, ptr(piv), ptr(Bd), 4, 4, ptr(rws), rws.numel(), None)
        _lib.call("swb_lu_rcond", ptr(Ad), n, lda, ptr(piv), ptr(an), ptr(rc), ptr(ws), ws.numel(), None)

    for name, f in (("small", small), ("blocked", blocked), ("small_norc", small_norc),
                    ("blocked_norc", blocked_norc)):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(50):
            f()
        e1.record()
        torch.cuda.synchronize()
        print(f"n={n} {name}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us", flush=True)
