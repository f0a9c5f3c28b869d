// Tuning harness (measurement only): times NN/TN DMMA GEMM configurations on
// the c4 rotation / projection shapes.  Not part of the library.
#include <cstdio>
#include <vector>
#include "../paper_1607_04174_b200/csrc/dmma_core.cuh"

void swb_set_last_cuda(cudaError_t) {}
void swb_count_launch() {}
int swb_sm_count() { return 148; }

using namespace swb_core;

template <int WARPS_M, int WARPS_N, int WTM, int WTN, int STAGES, int MINB>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, MINB)
nn_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B, int64_t ldb, int64_t rows,
          int64_t K, int64_t M2, double* __restrict__ out, int64_t ldo, int n_tiles_n) {
  using Cf = Cfg<WARPS_M, WARPS_N, WTM, WTN, STAGES, false>;
  extern __shared__ __align__(16) double smem[];
  const int64_t tile = blockIdx.x;
  const int64_t bm = tile / n_tiles_n;
  const int bn = static_cast<int>(tile % n_tiles_n);
  const int64_t m0 = bm * Cf::BM, n0 = int64_t(bn) * Cf::BN;
  double acc[WTM][WTN][2];
#pragma unroll
  for (int i = 0; i < WTM; ++i)
#pragma unroll
    for (int j = 0; j < WTN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  mainloop<WARPS_M, WARPS_N, WTM, WTN, STAGES, false>(acc, smem, A, lda, B, ldb, 0, K, m0, rows, n0, M2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
#pragma unroll
  for (int i = 0; i < WTM; ++i) {
    int64_t r = m0 + wm * WTM * 8 + i * 8 + (lane >> 2);
    if (r >= rows) continue;
#pragma unroll
    for (int j = 0; j < WTN; ++j) {
      int64_t c = n0 + wn * WTN * 8 + j * 8 + 2 * (lane & 3);
      if (c + 1 < M2) *reinterpret_cast<double2*>(out + r * ldo + c) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
  }
}

template <int WM, int WN, int TM, int TN_, int ST, int MINB>
void run(const char* name, const double* A, const double* B, double* O, int64_t rows, int64_t K, int64_t M2) {
  using Cf = Cfg<WM, WN, TM, TN_, ST, false>;
  auto kern = nn_kernel<WM, WN, TM, TN_, ST, MINB>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cf::THREADS, Cf::SMEM);
  const int64_t tm = (rows + Cf::BM - 1) / Cf::BM;
  const int tn = (int)((M2 + Cf::BN - 1) / Cf::BN);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) kern<<<(unsigned)(tm * tn), Cf::THREADS, Cf::SMEM>>>(A, K, B, M2, rows, K, M2, O, M2, tn);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int w = 0; w < reps; ++w) kern<<<(unsigned)(tm * tn), Cf::THREADS, Cf::SMEM>>>(A, K, B, M2, rows, K, M2, O, M2, tn);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  printf("%-28s tile %3dx%-3d thr %3d occ %d smem %6zu  %8.3f ms  %6.2f TFLOP/s  err=%s\n", name, Cf::BM, Cf::BN,
         Cf::THREADS, occ, Cf::SMEM, ms, 2.0 * rows * K * M2 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t rows = 4 << 20, K = 400, M2 = 400;
  double *A, *B, *O;
  cudaMalloc(&A, rows * K * 8); cudaMalloc(&B, K * M2 * 8); cudaMalloc(&O, rows * M2 * 8);
  cudaMemset(A, 0, rows * K * 8); cudaMemset(B, 0, K * M2 * 8);
  run<4, 2, 4, 5, 3, 2>("4x2 w4x5 s3 (current)", A, B, O, rows, K, M2);
  run<2, 2, 8, 5, 3, 2>("2x2 w8x5 s3", A, B, O, rows, K, M2);
  run<2, 2, 8, 5, 2, 3>("2x2 w8x5 s2 minb3", A, B, O, rows, K, M2);
  run<4, 1, 4, 10, 2, 3>("4x1 w4x10 s2 minb3", A, B, O, rows, K, M2);
  run<2, 2, 8, 5, 4, 2>("2x2 w8x5 s4", A, B, O, rows, K, M2);
  run<2, 2, 6, 5, 3, 3>("2x2 w6x5 s3 (96x80)", A, B, O, rows, K, M2);
  run<1, 2, 16, 5, 3, 2>("1x2 w16x5 s3 (128x80)", A, B, O, rows, K, M2);
  run<2, 1, 8, 10, 3, 2>("2x1 w8x10 s3 (128x80)", A, B, O, rows, K, M2);
  run<4, 2, 8, 5, 3, 1>("4x2 w8x5 s3 (256x80)", A, B, O, rows, K, M2);
  return 0;
}
