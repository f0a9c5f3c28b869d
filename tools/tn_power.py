"""Is the c4 projection power-bound?  Time the symmetric TN GEMM alone, an
HBM stream (the rotation's digit split on 1M-row chunks, back to back) alone,
and both at once on two streams.  Run with SWB_TN_OCC=2 so the split's
blocks fit beside the TN CTAs."""
import sys

import torch

from paper_1607_04174_b200 import _lib

n, K = 1 << 24, 400
torch.manual_seed(0)
V = torch.randn(n, K, dtype=torch.float64, device="cuda")
W = torch.randn(n, K, dtype=torch.float64, device="cuda")
P = torch.empty(K, K, dtype=torch.float64, device="cuda")
nb = _lib.size("swb_gemm_tn_workspace_bytes", n, K, K)
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
rows = 1 << 20
onb = _lib.size("swb_oz_gemm_nn_workspace_bytes", 4 * rows, K, K)
ows = torch.empty(onb, dtype=torch.uint8, device="cuda")
n_split = int(sys.argv[1]) if len(sys.argv) > 1 else 16


def tn():
    _lib.call("swb_gemm_tn", V.data_ptr(), K, W.data_ptr(), K, n, K, K, 1, P.data_ptr(), K, ws.data_ptr(), nb, None)


def splits(stream):
    for i in range(n_split):
        _lib.call("swb_oz_split_rows", V.data_ptr() + 8 * (i % 16) * rows * K, K, rows, 4 * rows, K, K, i & 1,
                  ows.data_ptr(), onb, stream.cuda_stream)


side = torch.cuda.Stream()
tn(); splits(side); torch.cuda.synchronize()


def timed(f):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    e0.record()
    f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


t_tn = timed(tn)
t_sp = timed(lambda: (splits(torch.cuda.current_stream())))


def both():
    side.wait_stream(torch.cuda.current_stream())
    splits(side)
    tn()
    torch.cuda.current_stream().wait_stream(side)


t_both = timed(both)
print(f"TN alone {t_tn:.2f} ms | {n_split} splits alone {t_sp:.2f} ms | both {t_both:.2f} ms "
      f"(serial sum {t_tn + t_sp:.2f})", flush=True)
