"""Time the INT8-tensor-core FP64 GEMM (swb_oz_gemm_nn) against the DMMA
GEMM (swb_gemm_nn) on the rotation shape rows x K x K and compare results."""
import sys
import time

import numpy as np
import torch

from paper_1607_04174_b200 import _lib

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4 << 20
K = int(sys.argv[2]) if len(sys.argv) > 2 else 400
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
torch.manual_seed(0)
A = torch.randn(rows, K, dtype=torch.float64, device="cuda") / K ** 0.5
C = torch.eye(K, dtype=torch.float64, device="cuda") + 1e-2 * torch.randn(K, K, dtype=torch.float64, device="cuda")
o1 = torch.empty(rows, K, dtype=torch.float64, device="cuda")
o2 = torch.empty_like(o1)
nb = _lib.size("swb_oz_gemm_nn_workspace_bytes", rows, K, K)
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")


def oz():
    _lib.call("swb_oz_gemm_nn", A.data_ptr(), K, C.data_ptr(), K, rows, K, K, o1.data_ptr(), K, ws.data_ptr(), nb, None)


def dm():
    _lib.call("swb_gemm_nn", A.data_ptr(), K, C.data_ptr(), K, rows, K, K, o2.data_ptr(), K, 0, None)


for name, f in (("ozaki_int8", oz), ("dmma", dm)):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name}: {ms:.2f} ms  {2 * rows * K * K / ms / 1e9:.1f} TFLOP/s (fp64-equivalent)", flush=True)
d = (o1 - o2).abs().max().item()
print("max |oz - dmma| =", d, " max |out| =", o2.abs().max().item())
import os
if os.environ.get("SWB_OZ_PROF"):
    import ctypes as C
    buf = (C.c_ulonglong * 12)()
    _lib.load().swb_oz_prof_read(buf)
    v = list(buf)
    for i, name in enumerate(("producer(wait empty)", "mma(wait tempty | wait full)", "epilogue(wait tfull)")):
        n = max(v[4 * i + 3], 1)
        print(f"{name}: w0={v[4*i]/n:.3e} w1={v[4*i+1]/n:.3e} total={v[4*i+2]/n:.3e} cyc per warp")
