// FP64 DMMA GEMM core shared by the GEMM, LU-update and reconstruction
// kernels: padded shared-memory tiles (bank-conflict-free fragment loads),
// a multi-stage cp.async pipeline and the mma.sync.m8n8k4.f64 inner loop.
#pragma once
#include "swb_common.cuh"

namespace swb_core {

constexpr int BK = 16;  // reduction depth per pipeline stage

__host__ __device__ constexpr int pad4mod16(int n) { return n + ((4 - n % 16) + 16) % 16; }

template <int WARPS_M, int WARPS_N, int WTM, int WTN, int STAGES, bool TN>
struct Cfg {
  static constexpr int BM = WARPS_M * WTM * 8;
  static constexpr int BN = WARPS_N * WTN * 8;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  // A in smem: TN -> [BK][A_LD] (k-major), NN -> [BM][A_LD] (m-major)
  static constexpr int A_LD = TN ? pad4mod16(BM) : pad4mod16(BK);
  static constexpr int A_ELEMS = TN ? BK * A_LD : BM * A_LD;
  static constexpr int B_LD = pad4mod16(BN);
  static constexpr int B_ELEMS = BK * B_LD;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_ELEMS * sizeof(double);
};

// ---------------------------------------------------------------------------
// shared mainloop: acc += A_tile * B_tile over k in [k_begin, k_end)
// TN:  A(m, k) = X[k][m0+m],  B(k, n) = Y[k][n0+n]   (k = row index)
// NN:  A(m, k) = A[m0+m][k],  B(k, n) = B[k][n0+n]
// ---------------------------------------------------------------------------
// Tile t -> (tile row, tile col).  Symmetric plans (BM == BN) enumerate the
// upper-triangle tiles row by row: row i holds tiles j = i .. tn-1.
__host__ __device__ __forceinline__ int2 decode_tile(int t, int tn, int symmetric) {
  if (!symmetric) return make_int2(t / tn, t % tn);
  int i = 0;
  while (t >= tn - i) { t -= tn - i; ++i; }
  return make_int2(i, i + t);
}

template <int WARPS_M, int WARPS_N, int WTM, int WTN, int STAGES, bool TN>
__device__ __forceinline__ void load_stage(double* sA, double* sB, const double* A, int64_t lda,
                                           const double* B, int64_t ldb, int64_t k0,
                                           int64_t k_end, int64_t m0, int64_t m_lim,
                                           int64_t n0, int64_t n_lim) {
  using Cf = Cfg<WARPS_M, WARPS_N, WTM, WTN, STAGES, TN>;
  const int tid = threadIdx.x;
  if (TN) {
    // X tile: BK rows (k) x BM cols, rows k0.., cols m0..
    constexpr int CH = Cf::BM / 2;              // 16B chunks per row
    for (int c = tid; c < BK * CH; c += Cf::THREADS) {
      int kr = c / CH, cc = (c % CH) * 2;
      int64_t gk = k0 + kr, gm = m0 + cc;
      bool p = (gk < k_end) && (gm < m_lim);
      const double* src = p ? (A + gk * lda + gm) : A;
      cp_async16(sA + kr * Cf::A_LD + cc, src, p);
    }
  } else {
    // A tile: BM rows x BK cols (k), rows m0.., cols k0..
    constexpr int CH = BK / 2;
    for (int c = tid; c < Cf::BM * CH; c += Cf::THREADS) {
      int mr = c / CH, cc = (c % CH) * 2;
      int64_t gm = m0 + mr, gk = k0 + cc;
      bool p = (gm < m_lim) && (gk < k_end);
      const double* src = p ? (A + gm * lda + gk) : A;
      cp_async16(sA + mr * Cf::A_LD + cc, src, p);
    }
  }
  if (((ldb & 1) == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0)) {
    constexpr int CH = Cf::BN / 2;
    for (int c = tid; c < BK * CH; c += Cf::THREADS) {
      int kr = c / CH, cc = (c % CH) * 2;
      int64_t gk = k0 + kr, gn = n0 + cc;
      bool p = (gk < k_end) && (gn < n_lim);
      const double* src = p ? (B + gk * ldb + gn) : B;
      cp_async16(sB + kr * Cf::B_LD + cc, src, p);
    }
  } else {  // odd leading dimension (small label counts): 8-byte copies
    for (int c = tid; c < BK * Cf::BN; c += Cf::THREADS) {
      int kr = c / Cf::BN, cc = c % Cf::BN;
      int64_t gk = k0 + kr, gn = n0 + cc;
      bool p = (gk < k_end) && (gn < n_lim);
      const double* src = p ? (B + gk * ldb + gn) : B;
      cp_async8(sB + kr * Cf::B_LD + cc, src, p);
    }
  }
}

template <int WARPS_M, int WARPS_N, int WTM, int WTN, int STAGES, bool TN>
__device__ __forceinline__ void mainloop(double (&acc)[WTM][WTN][2], double* smem,
                                         const double* A, int64_t lda, const double* B,
                                         int64_t ldb, int64_t k_begin, int64_t k_end,
                                         int64_t m0, int64_t m_lim, int64_t n0, int64_t n_lim) {
  using Cf = Cfg<WARPS_M, WARPS_N, WTM, WTN, STAGES, TN>;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int64_t nk = (k_end - k_begin + BK - 1) / BK;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) {
      double* st = smem + s * Cf::STAGE_ELEMS;
      load_stage<WARPS_M, WARPS_N, WTM, WTN, STAGES, TN>(st, st + Cf::A_ELEMS, A, lda, B, ldb,
                                                         k_begin + s * BK, k_end, m0, m_lim, n0, n_lim);
    }
    cp_async_commit();
  }

  const int lr = lane >> 2, lc = lane & 3;
  for (int64_t kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      int64_t nt = kt + STAGES - 1;
      if (nt < nk) {
        double* st = smem + (nt % STAGES) * Cf::STAGE_ELEMS;
        load_stage<WARPS_M, WARPS_N, WTM, WTN, STAGES, TN>(st, st + Cf::A_ELEMS, A, lda, B, ldb,
                                                           k_begin + nt * BK, k_end, m0, m_lim, n0, n_lim);
      }
      cp_async_commit();
    }
    const double* sA = smem + (kt % STAGES) * Cf::STAGE_ELEMS;
    const double* sB = sA + Cf::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[WTM], bf[WTN];
#pragma unroll
      for (int i = 0; i < WTM; ++i) {
        int m = wm * WTM * 8 + i * 8 + lr;
        int k = kk * 4 + lc;
        af[i] = TN ? sA[k * Cf::A_LD + m] : sA[m * Cf::A_LD + k];
      }
#pragma unroll
      for (int j = 0; j < WTN; ++j) {
        int n = wn * WTN * 8 + j * 8 + lr;
        int k = kk * 4 + lc;
        bf[j] = sB[k * Cf::B_LD + n];
      }
#pragma unroll
      for (int i = 0; i < WTM; ++i)
#pragma unroll
        for (int j = 0; j < WTN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
}


}  // namespace swb_core
