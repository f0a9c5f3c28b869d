"""Time the seed-system pieces at c4 size on the GPU (CUDA events, warm):
swb_lu_factor, swb_lu_solve (L + 1 right-hand sides), swb_lu_rcond for an
(S + 1) x (S + 1) system shaped like the bordered gamma = 0 seed system
(identity minus a rank-m product), and check the solve against numpy."""

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1607_04174_b200 import _lib  # noqa: E402
from paper_1607_04174_b200.device import ptr, stream_handle  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 801
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 400
    nrhs = 5
    rng = np.random.default_rng(0)
    U = rng.standard_normal((n, m)) * 0.02
    W = rng.standard_normal((n, m)) * 0.02
    A0 = np.eye(n) - U @ W.T
    B0 = rng.standard_normal((n, nrhs))
    lda = (n + 7) // 8 * 8
    ldb = (nrhs + 1) // 2 * 2
    Ah = np.zeros((n, lda))
    Ah[:, :n] = A0
    Bh = np.zeros((n, ldb))
    Bh[:, :nrhs] = B0
    A_dev0 = torch.from_numpy(Ah).cuda()
    B_dev0 = torch.from_numpy(Bh).cuda()
    A = torch.empty_like(A_dev0)
    B = torch.empty_like(B_dev0)
    piv = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    anorm = torch.empty(2, dtype=torch.float64, device="cuda")
    rc = torch.empty(1, dtype=torch.float64, device="cuda")
    ws = torch.empty(_lib.size("swb_lu_workspace_bytes", n), dtype=torch.uint8, device="cuda")
    sws = torch.empty(_lib.size("swb_lu_solve_workspace_bytes", n, nrhs), dtype=torch.uint8, device="cuda")
    st = stream_handle()
    res = {}

    def run(reps=20):
        t = {"factor": [], "solve": [], "rcond": []}
        for _ in range(reps):
            A.copy_(A_dev0)
            B.copy_(B_dev0)
            ev = [torch.cuda.Event(True) for _ in range(4)]
            ev[0].record()
            _lib.call("swb_lu_factor", ptr(A), n, lda, ptr(piv), ptr(anorm), ptr(ws), ws.numel(), st)
            ev[1].record()
            _lib.call("swb_lu_solve", ptr(A), n, lda, ptr(piv), ptr(B), nrhs, ldb, ptr(sws), sws.numel(), st)
            ev[2].record()
            _lib.call("swb_lu_rcond", ptr(A), n, lda, ptr(piv), ptr(anorm), ptr(rc), ptr(ws), ws.numel(), st)
            ev[3].record()
            torch.cuda.synchronize()
            t["factor"].append(ev[0].elapsed_time(ev[1]))
            t["solve"].append(ev[1].elapsed_time(ev[2]))
            t["rcond"].append(ev[2].elapsed_time(ev[3]))
        return {k: float(np.median(v)) for k, v in t.items()}

    run(3)
    res["ms"] = run()
    x = B.cpu().numpy()[:, :nrhs]
    want = np.linalg.solve(A0, B0)
    res["solve_rel_err"] = float(np.abs(x - want).max() / np.abs(want).max())
    import scipy.linalg as sla
    lu, pv = sla.lu_factor(A0)
    rc_ref = sla.lapack.dgecon(lu, np.linalg.norm(A0, 1), norm="1")[0]
    res["rcond"] = float(rc.item())
    res["rcond_ref"] = float(rc_ref)
    res["n"] = n
    print(json.dumps(res))


if __name__ == "__main__":
    main()
