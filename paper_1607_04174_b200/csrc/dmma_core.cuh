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

// One pipeline stage: copy the A tile and the B tile of one BK-deep k-slice
// into shared memory.  Tile bases are 64-bit pointers computed once per
// stage; per-chunk offsets are 32-bit (tile extents are small), and the
// chunk loops have compile-time trip counts.
//   NN: A tile = BM rows x BK cols at A_t (ld lda), B tile = BK rows x BN cols
//   TN: A tile = BK rows x BM cols at A_t (ld lda) (k-major), B tile as NN
// *_rows / *_cols: valid extent of each tile (rest zero-filled).
template <int WARPS_M, int WARPS_N, int WTM, int WTN, int STAGES, bool TN>
__device__ __forceinline__ void load_stage(double* sA, double* sB, const double* A_t, int lda, int a_rows,
                                           int a_cols, const double* B_t, int ldb, int b_rows, int b_cols,
                                           bool b_vec) {
  using Cf = Cfg<WARPS_M, WARPS_N, WTM, WTN, STAGES, TN>;
  constexpr int T = Cf::THREADS;
  const int tid = threadIdx.x;
  {
    constexpr int ROWS = TN ? BK : Cf::BM;
    constexpr int CH = (TN ? Cf::BM : BK) / 2;  // 16-byte chunks per row
    constexpr int TOTAL = ROWS * CH;
#pragma unroll
    for (int i = 0; i < (TOTAL + T - 1) / T; ++i) {
      const int c = tid + i * T;
      if (TOTAL % T != 0 && c >= TOTAL) break;
      const int r = c / CH, cc = (c % CH) * 2;
      const bool p = (r < a_rows) && (cc < a_cols);
      if (TN) {
        cp_async16(sA + r * Cf::A_LD + cc, p ? A_t + r * lda + cc : A_t, p);
      } else {
        // NN: the columns are the reduction index.  An odd K ends in half a
        // chunk: copy its 8 bytes and zero-fill the rest, so whatever sits
        // past column K - 1 (a padding column, possibly NaN) never meets
        // B's zero row (NaN * 0)
        cp_async16_n(sA + r * Cf::A_LD + cc, p ? A_t + r * lda + cc : A_t, p ? (cc + 1 < a_cols ? 16 : 8) : 0);
      }
    }
  }
  if (b_vec) {
    constexpr int CH = Cf::BN / 2;
    constexpr int TOTAL = BK * CH;
#pragma unroll
    for (int i = 0; i < (TOTAL + T - 1) / T; ++i) {
      const int c = tid + i * T;
      if (TOTAL % T != 0 && c >= TOTAL) break;
      const int r = c / CH, cc = (c % CH) * 2;
      const bool p = (r < b_rows) && (cc < b_cols);
      cp_async16(sB + r * Cf::B_LD + cc, p ? B_t + r * ldb + cc : B_t, p);
    }
  } else {  // odd leading dimension / 8-byte alignment (small label counts)
    constexpr int TOTAL = BK * Cf::BN;
#pragma unroll 4
    for (int c = tid; c < TOTAL; c += T) {
      const int r = c / Cf::BN, cc = c % Cf::BN;
      const bool p = (r < b_rows) && (cc < b_cols);
      cp_async8(sB + r * Cf::B_LD + cc, p ? B_t + r * ldb + cc : B_t, p);
    }
  }
}

__device__ __forceinline__ int clamp_int(int64_t v, int hi) { return v < 0 ? 0 : (v > hi ? hi : static_cast<int>(v)); }

// Pipelined k-loop; `compute(sA, sB)` consumes one BK-deep stage.
template <int WARPS_M, int WARPS_N, int WTM, int WTN, int STAGES, bool TN, class Compute>
__device__ __forceinline__ void pipeline(double* smem, const double* A, int64_t lda, const double* B, int64_t ldb,
                                         int64_t k_begin, int64_t k_end, int64_t m0, int64_t m_lim, int64_t n0,
                                         int64_t n_lim, Compute&& compute) {
  using Cf = Cfg<WARPS_M, WARPS_N, WTM, WTN, STAGES, TN>;
  const int nk = static_cast<int>((k_end - k_begin + BK - 1) / BK);
  const bool b_vec = ((ldb & 1) == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
  // tile-base pointers of the first k-slice and their per-stage advance
  const double* a_t = TN ? A + k_begin * lda + m0 : A + m0 * lda + k_begin;
  const int64_t a_step = TN ? BK * lda : BK;
  const double* b_t = B + k_begin * ldb + n0;
  const int64_t b_step = BK * ldb;
  const int m_rows = clamp_int(m_lim - m0, Cf::BM);
  const int n_cols = clamp_int(n_lim - n0, Cf::BN);
  const int k_left = static_cast<int>(k_end - k_begin);  // per-CTA row chunks (< 2^31)

  auto issue = [&](int slot, int kt) {
    double* st = smem + slot * Cf::STAGE_ELEMS;
    const int kl = k_left - kt * BK;
    if (TN)
      load_stage<WARPS_M, WARPS_N, WTM, WTN, STAGES, TN>(st, st + Cf::A_ELEMS, a_t + kt * a_step,
                                                         static_cast<int>(lda), kl, m_rows, b_t + kt * b_step,
                                                         static_cast<int>(ldb), kl, n_cols, b_vec);
    else
      load_stage<WARPS_M, WARPS_N, WTM, WTN, STAGES, TN>(st, st + Cf::A_ELEMS, a_t + kt * a_step,
                                                         static_cast<int>(lda), m_rows, kl, b_t + kt * b_step,
                                                         static_cast<int>(ldb), kl, n_cols, b_vec);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) issue(s, s);
    cp_async_commit();
  }
  int slot = 0;                 // stage being consumed
  int fill = STAGES - 1;        // stage being filled next
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < nk) issue(fill, kt + STAGES - 1);
    cp_async_commit();
    fill = fill + 1 == STAGES ? 0 : fill + 1;
    const double* sA = smem + slot * Cf::STAGE_ELEMS;
    slot = slot + 1 == STAGES ? 0 : slot + 1;
    compute(sA, sA + Cf::A_ELEMS);
  }
  cp_async_wait<0>();
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
  const int lr = lane >> 2, lc = lane & 3;
  pipeline<WARPS_M, WARPS_N, WTM, WTN, STAGES, TN>(
      smem, A, lda, B, ldb, k_begin, k_end, m0, m_lim, n0, n_lim, [&](const double* sA, const double* sB) {
#pragma unroll
        for (int kk = 0; kk < BK / 4; ++kk) {
          double af[WTM], bf[WTN];
#pragma unroll
          for (int i = 0; i < WTM; ++i) {
            const int m = wm * WTM * 8 + i * 8 + lr;
            const int k = kk * 4 + lc;
            af[i] = TN ? sA[k * Cf::A_LD + m] : sA[m * Cf::A_LD + k];
          }
#pragma unroll
          for (int j = 0; j < WTN; ++j) {
            const int n = wn * WTN * 8 + j * 8 + lr;
            const int k = kk * 4 + lc;
            bf[j] = sB[k * Cf::B_LD + n];
          }
#pragma unroll
          for (int i = 0; i < WTM; ++i)
#pragma unroll
            for (int j = 0; j < WTN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
      });
}

}  // namespace swb_core
