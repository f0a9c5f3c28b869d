"""cuBLAS DGEMM calibration (measurement only): torch.matmul float64."""
import torch, time
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cuBLAS DGEMM {n}^3: {2*n**3/ms/1e9:.2f} TFLOP/s")
# tall-skinny like the rotation: (16.8M/8 x 400) @ (400 x 400)
N = 2_097_152
v = torch.randn(N, 400, dtype=torch.float64, device="cuda")
c = torch.randn(400, 400, dtype=torch.float64, device="cuda")
for _ in range(3): v @ c
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5): o = v @ c
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"cuBLAS tall NN {N}x400x400: {2*N*400*400/ms/1e9:.2f} TFLOP/s")
e0.record()
for _ in range(5): g = v.T @ v
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"cuBLAS TN gram {N}x400: {2*N*400*400/ms/1e9:.2f} TFLOP/s")
x = torch.empty(2**30 // 8 * 4, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
e0.record()
for _ in range(10): y.copy_(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"copy: {2*x.numel()*8/ms/1e6:.1f} GB/s")
