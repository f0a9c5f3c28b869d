"""Time the symmetric TN projection P = V^T W (swb_gemm_tn, symmetric=1) on
N x K random operands (the c4 shape by default); SWB_TN_INTERLEAVE=0 selects
the contiguous-chunk split-K for A/B."""
import sys

import torch

from paper_1607_04174_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
K = int(sys.argv[2]) if len(sys.argv) > 2 else 400
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
torch.manual_seed(0)
V = torch.randn(n, K, dtype=torch.float64, device="cuda")
W = torch.randn(n, K, dtype=torch.float64, device="cuda")
P = torch.empty(K, K, dtype=torch.float64, device="cuda")
nb = _lib.size("swb_gemm_tn_workspace_bytes", n, K, K)
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")


def tn():
    _lib.call("swb_gemm_tn", V.data_ptr(), K, W.data_ptr(), K, n, K, K, 1, P.data_ptr(), K, ws.data_ptr(), nb, None)


tn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(reps):
    tn()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"tn_sym {n}x{K}: {ms:.2f} ms  {n * K * (K + 1) / ms / 1e9:.1f} TFLOP/s", flush=True)
if n <= 1 << 20:
    ref = (V.T @ W)
    ref = torch.triu(ref) + torch.triu(ref, 1).T
    print("max |P - torch| =", (P - ref).abs().max().item())
