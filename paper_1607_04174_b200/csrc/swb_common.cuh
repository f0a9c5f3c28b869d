// Shared helpers for the specwalk-b200 kernels (sm_100a, FP64).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <algorithm>

#include "../../include/specwalk_b200.h"

#define SWB_CUDA_TRY(expr)                                   \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) { swb_set_last_cuda(_e); return SWB_CUDA_ERROR; } \
  } while (0)

#define SWB_CHECK_LAUNCH()                                   \
  do {                                                       \
    swb_count_launch();                                      \
    cudaError_t _e = cudaGetLastError();                     \
    if (_e != cudaSuccess) { swb_set_last_cuda(_e); return SWB_CUDA_ERROR; } \
  } while (0)

void swb_set_last_cuda(cudaError_t e);
void swb_count_launch();
int swb_sm_count();

static inline cudaStream_t swb_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Current device ordinal (0 when no device is current).
static inline int swb_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  return dev & 63;
}

// True the first time it is called for the current device: per-device
// one-time setup (cudaFuncSetAttribute is a per-device property, so a
// process driving several GPUs needs it once on each).
static inline bool swb_first_on_device(unsigned long long* mask) {
  const unsigned long long bit = 1ull << swb_device();
  return (__atomic_fetch_or(mask, bit, __ATOMIC_ACQ_REL) & bit) == 0;
}

static inline size_t swb_align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Forward-neighbour offsets of the lattice (see swb_lattice docs in the header).
struct LatticeDev {
  int64_t nx, ny, nz;
  int ndir;            // forward directions
  int conn;            // 4, 8, 6
  int dx[4], dy[4], dz[4];
};

static inline int swb_make_lattice(const swb_lattice* lat, LatticeDev* out) {
  if (!lat || lat->nx <= 0 || lat->ny <= 0 || lat->nz <= 0) return SWB_INVALID_PARAM;
  LatticeDev d{};
  d.nx = lat->nx; d.ny = lat->ny; d.nz = lat->nz; d.conn = lat->connectivity;
  if (lat->connectivity == 4 && lat->nz == 1) {
    d.ndir = 2;
    int xs[2] = {1, 0}, ys[2] = {0, 1};
    for (int i = 0; i < 2; ++i) { d.dx[i] = xs[i]; d.dy[i] = ys[i]; d.dz[i] = 0; }
  } else if (lat->connectivity == 8 && lat->nz == 1) {
    d.ndir = 4;
    int xs[4] = {1, 0, 1, -1}, ys[4] = {0, 1, 1, 1};
    for (int i = 0; i < 4; ++i) { d.dx[i] = xs[i]; d.dy[i] = ys[i]; d.dz[i] = 0; }
  } else if (lat->connectivity == 6) {
    d.ndir = 3;
    int xs[3] = {1, 0, 0}, ys[3] = {0, 1, 0}, zs[3] = {0, 0, 1};
    for (int i = 0; i < 3; ++i) { d.dx[i] = xs[i]; d.dy[i] = ys[i]; d.dz[i] = zs[i]; }
  } else {
    return SWB_INVALID_PARAM;
  }
  if (lat->weight_mode != 0 && lat->weight_mode != 1) return SWB_INVALID_PARAM;
  *out = d;
  return SWB_OK;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// cp.async helpers (Ampere+ LDGSTS; fine on sm_100a)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" :: "r"(s), "l"(gmem), "r"(sz));
}
// 16-byte slot, `bytes` (0, 8 or 16) copied from gmem and the rest zero-filled
__device__ __forceinline__ void cp_async16_n(void* smem, const void* gmem, int bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" :: "r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" :: "r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" :: "n"(N)); }

// FP64 tensor-core MMA (DMMA.8x8x4): D = A(8x4, row) * B(4x8, col) + C.
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
