// Microbenchmark: cycles per tcgen05.mma.kind::i8 (M = 128) for SS / TS
// operand modes and several N, plus tcgen05.cp 128x256b, on every SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_probe tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return uint64_t((a >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) |
         (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc(int n) { return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (8u << 24); }

template <int MODE, int N>   // MODE 0 = SS, 1 = TS, 2 = cp only, 3 = TS + cp (7 cp per 28 mma)
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t a0 = su32(sm), b0 = a0 + 32768;
    for (int it = 0; it < iters; ++it) {
      if (MODE >= 2) {
#pragma unroll
        for (int i = 0; i < 7; ++i)
          asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tm + 448 + (i & 3) * 8),
                       "l"(sdesc(a0 + i * 4096, 2048, 128)));
      }
      if (MODE != 2) {
#pragma unroll
        for (int k = 0; k < 28; ++k) {
          const uint64_t bd = sdesc(b0 + (k % 7) * 2048, N * 16, 128);
          const uint32_t d = tm + (k % 7) * (N <= 64 ? N : 0);
          if (MODE == 0) {
            const uint64_t ad = sdesc(a0 + (k % 7) * 4096, 2048, 128);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
                         "l"(ad), "l"(bd), "r"(idesc(N)), "r"(1));
          } else {
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                         "r"(tm + 448 + (k & 3) * 8), "l"(bd), "r"(idesc(N)), "r"(1));
          }
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(su32(&bar)));
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) atomicAdd(out, t1 - t0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int MODE, int N>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  auto k = probe<MODE, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024 + 1024);
  const int iters = 2000;
  k<<<148, 128, 64 * 1024 + 1024>>>(iters, d);
  cudaMemset(d, 0, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 128, 64 * 1024 + 1024>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double per = double(h) / 148 / iters;
  const double macs = MODE == 2 ? 0 : 28.0 * 128 * N * 32 * iters * 148;
  printf("%-22s %s cyc/iter %.0f  (%.1f cyc per mma)  %.3f ms  %.0f TOPS\n", name, cudaGetErrorString(err), per,
         per / 28, ms, 2 * macs / ms / 1e9);
  cudaFree(d);
}

int main() {
  run<0, 64>("SS N=64");
  run<0, 48>("SS N=48");
  run<0, 128>("SS N=128");
  run<0, 256>("SS N=256");
  run<1, 48>("TS N=48");
  run<1, 64>("TS N=64");
  run<1, 128>("TS N=128");
  run<2, 48>("cp only (7 x 128x256b)");
  run<3, 48>("TS N=48 + 7 cp");
  run<3, 64>("TS N=64 + 7 cp");
  return 0;
}
