"""Time the rotation's digit split alone (swb_oz_split_rows) on 1M rows x K
and report GB/s of (read 8 B + write the planes) per entry; SWB_LIB picks a
variant build (tools/build_variant.py -DOZ_SLICE_WARPS_CFG=...)."""
import sys

import torch

from paper_1607_04174_b200 import _lib

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
K = int(sys.argv[2]) if len(sys.argv) > 2 else 400
torch.manual_seed(0)
A = torch.randn(rows, K, dtype=torch.float64, device="cuda")
nb = _lib.size("swb_oz_gemm_nn_workspace_bytes", 4 * rows, K, K)
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
chunk = _lib.size("swb_oz_chunk_rows", 4 * rows, K, K)
assert chunk >= rows


def split():
    _lib.call("swb_oz_split_rows", A.data_ptr(), K, rows, 4 * rows, K, K, 0, ws.data_ptr(), nb, None)


for _ in range(3):
    split()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
reps = 20
e0.record()
for _ in range(reps):
    split()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
kp = (K + 31) // 32 * 32
byts = rows * (8.0 * K + 7.0 * kp + 8)
print(f"split {rows}x{K}: {ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s", flush=True)
