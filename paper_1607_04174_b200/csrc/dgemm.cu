// FP64 tensor-core GEMMs for the N x K x K contractions of the hot path.
//
//   NN:  out[rows x M2] = A[rows x K] * B[K x M2]      (rotation V*C,
//        reconstruction for many labels)
//   TN:  out[M1 x M2]   = X^T Y, reduction over rows    (projection
//        P = V^T (dL V), t_p = V^T P^, Gram matrices)
//
// sm_100a has no FP64 kind for tcgen05.mma, so the tensor-core path is the
// warp-level DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4), fed from shared
// memory that a multi-stage cp.async pipeline fills.  Shared tiles are padded
// so every fragment load is bank-conflict free (stride = 4 mod 16 doubles).
// Split-row TN reductions go through a workspace and are summed in a fixed
// order, so results are bitwise deterministic run to run.
#include "swb_common.cuh"
#include <cstdlib>

#include "dmma_core.cuh"
#include "oz_digits.cuh"

namespace {
using namespace swb_core;

// ---------------------------------------------------------------------------
// NN kernel
// ---------------------------------------------------------------------------
template <int WARPS_M, int WARPS_N, int WTM, int WTN, int STAGES>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, 2)
gemm_nn_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
               int64_t ldb, int64_t rows, int64_t K, int64_t M2, double* __restrict__ out,
               int64_t ldo, int accumulate, double alpha, int n_tiles_n) {
  using Cf = Cfg<WARPS_M, WARPS_N, WTM, WTN, STAGES, false>;
  extern __shared__ __align__(16) double smem[];
  const int64_t tile = blockIdx.x;
  const int64_t bm = tile / n_tiles_n;
  const int bn = static_cast<int>(tile % n_tiles_n);
  const int64_t m0 = bm * Cf::BM;
  const int64_t n0 = int64_t(bn) * Cf::BN;

  double acc[WTM][WTN][2];
#pragma unroll
  for (int i = 0; i < WTM; ++i)
#pragma unroll
    for (int j = 0; j < WTN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  mainloop<WARPS_M, WARPS_N, WTM, WTN, STAGES, false>(acc, smem, A, lda, B, ldb, 0, K, m0, rows,
                                                      n0, M2);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
#pragma unroll
  for (int i = 0; i < WTM; ++i) {
    int64_t r = m0 + wm * WTM * 8 + i * 8 + (lane >> 2);
    if (r >= rows) continue;
    double* orow = out + r * ldo;
#pragma unroll
    for (int j = 0; j < WTN; ++j) {
      int64_t c = n0 + wn * WTN * 8 + j * 8 + 2 * (lane & 3);
      double v0 = alpha * acc[i][j][0], v1 = alpha * acc[i][j][1];
      if (c + 1 < M2) {
        double2* p = reinterpret_cast<double2*>(orow + c);
        if (accumulate) { double2 o = *p; v0 += o.x; v1 += o.y; }
        *p = make_double2(v0, v1);
      } else if (c < M2) {
        if (accumulate) v0 += orow[c];
        orow[c] = v0;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// TN kernel: split-K with an integer number of CTAs per output tile.  CTA
// c = t * per_tile + q computes tile t over row chunk q; every tile uses the
// same row chunks and the whole grid is one wave, so the CTAs of all tiles
// stream the same rows of X / Y at the same time and each row is fetched
// from HBM once (L2 serves the other tiles).  Partial tiles are summed in
// chunk order (deterministic).
// ---------------------------------------------------------------------------
template <int WARPS_M, int WARPS_N, int WTM, int WTN, int STAGES>
__global__ void __launch_bounds__(WARPS_M * WARPS_N * 32, 3)
gemm_tn_kernel(const double* __restrict__ X, int64_t ldx, const double* __restrict__ Y,
               int64_t ldy, int64_t rows, int64_t M1, int64_t M2, int tn, int symmetric,
               int per_tile, int64_t chunk_rows, double* __restrict__ partial) {
  using Cf = Cfg<WARPS_M, WARPS_N, WTM, WTN, STAGES, true>;
  extern __shared__ __align__(16) double smem[];
  const int c = blockIdx.x;
  const int t = c / per_tile, q = c % per_tile;
  const int2 tt = decode_tile(t, tn, symmetric);
  const int64_t m0 = int64_t(tt.x) * Cf::BM, n0 = int64_t(tt.y) * Cf::BN;
  const int64_t k_begin = int64_t(q) * chunk_rows;
  const int64_t k_end = min(rows, k_begin + chunk_rows);
  double acc[WTM][WTN][2];
#pragma unroll
  for (int i = 0; i < WTM; ++i)
#pragma unroll
    for (int j = 0; j < WTN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (k_begin < k_end)
    mainloop<WARPS_M, WARPS_N, WTM, WTN, STAGES, true>(acc, smem, X, ldx, Y, ldy, k_begin, k_end, m0, M1, n0, M2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  double* dst = partial + int64_t(c) * (Cf::BM * Cf::BN);
#pragma unroll
  for (int i = 0; i < WTM; ++i) {
    const int r = wm * WTM * 8 + i * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < WTN; ++j) {
      const int cc = wn * WTN * 8 + j * 8 + 2 * (lane & 3);
      *reinterpret_cast<double2*>(dst + r * Cf::BN + cc) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
  }
}

template <int BM, int BN>
__global__ void tn_reduce_kernel(const double* __restrict__ partial, int tn, int symmetric, int n_tiles, int per_tile,
                                 int64_t M1, int64_t M2, double* __restrict__ out, int64_t ldo) {
  const int64_t total = int64_t(n_tiles) * BM * BN;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(e / (BM * BN));
    const int rc = static_cast<int>(e % (BM * BN));
    const int2 tt = decode_tile(t, tn, symmetric);
    const int64_t i = int64_t(tt.x) * BM + rc / BN;
    const int64_t j = int64_t(tt.y) * BN + rc % BN;
    if (i >= M1 || j >= M2) continue;
    if (symmetric && j < i) continue;  // diagonal tiles: keep the upper half
    double s = 0.0;
    for (int q = 0; q < per_tile; ++q) s += partial[(int64_t(t) * per_tile + q) * (BM * BN) + rc];
    out[i * ldo + j] = s;
    if (symmetric && j != i) out[j * ldo + i] = s;
  }
}

// ---------------------------------------------------------------------------
// Symmetric TN (P = V^T W, upper triangle only).  Off-diagonal tiles run the
// regular 4-warp (W x W cells of 8x8 per warp) tile; a diagonal tile needs
// only the G(G+1)/2 upper cells of its G x G cell grid (G = 2W), split over
// the 4 warps by pairing rows, so it costs ~60 % of a full tile and gets
// proportionally longer row chunks.  One launch, one wave: CTAs
// [0, n_full*per_full) do off-diagonal tiles, the rest diagonal tiles.
// ---------------------------------------------------------------------------
// row lists per warp (-1 = none): G = 10 -> {0,7,9} {1,6} {2,5} {3,4,8}
//                                 G =  8 -> {0,7}   {1,6} {2,5} {3,4}
__host__ __device__ constexpr int diag_row(int G, int w, int k) {
  return G == 10 ? (w == 0 ? (k == 0 ? 0 : k == 1 ? 7 : 9)
                  : w == 1 ? (k == 0 ? 1 : k == 1 ? 6 : -1)
                  : w == 2 ? (k == 0 ? 2 : k == 1 ? 5 : -1)
                           : (k == 0 ? 3 : k == 1 ? 4 : 8))
                 : (k == 2 ? -1 : w == 0 ? (k == 0 ? 0 : 7) : w == 1 ? (k == 0 ? 1 : 6)
                                : w == 2 ? (k == 0 ? 2 : 5) : (k == 0 ? 3 : 4));
}
__host__ __device__ constexpr int diag_cells(int G, int w) {
  int n = 0;
  for (int k = 0; k < 3; ++k)
    if (diag_row(G, w, k) >= 0) n += G - diag_row(G, w, k);
  return n;
}
__host__ __device__ constexpr int diag_max_cells(int G) {
  int m = 0;
  for (int w = 0; w < 4; ++w) m = diag_cells(G, w) > m ? diag_cells(G, w) : m;
  return m;
}

template <int G, int WID, int A_LD, int B_LD>
__device__ __forceinline__ void diag_compute(double (&acc)[diag_max_cells(G)][2], const double* sA, const double* sB,
                                             int lr, int lc) {
#pragma unroll
  for (int kk = 0; kk < BK / 4; ++kk) {
    const int k = kk * 4 + lc;
    double af[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      constexpr int dummy = 0;
      (void)dummy;
      const int r = diag_row(G, WID, q);
      af[q] = r >= 0 ? sA[k * A_LD + r * 8 + lr] : 0.0;
    }
    int cell = 0;
#pragma unroll
    for (int c = 0; c < G; ++c) {
      bool need = false;
#pragma unroll
      for (int q = 0; q < 3; ++q) need |= (diag_row(G, WID, q) >= 0 && diag_row(G, WID, q) <= c);
      if (!need) continue;
      const double bf = sB[k * B_LD + c * 8 + lr];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int r = diag_row(G, WID, q);
        if (r < 0 || r > c) continue;
        // cell index = position of (r, c) in the warp's row-major cell list
        int idx = 0;
#pragma unroll
        for (int q2 = 0; q2 < q; ++q2)
          if (diag_row(G, WID, q2) >= 0) idx += G - diag_row(G, WID, q2);
        idx += c - r;
        dmma_8x8x4(acc[idx][0], acc[idx][1], af[q], bf);
        (void)cell;
      }
    }
  }
}

template <int G, int WID>
__device__ __forceinline__ void diag_store(const double (&acc)[diag_max_cells(G)][2], double* dst, int BN, int lane) {
  int idx = 0;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int r = diag_row(G, WID, q);
    if (r < 0) continue;
#pragma unroll
    for (int c = 0; c < G; ++c) {
      if (c < r) continue;
      const int row = r * 8 + (lane >> 2), col = c * 8 + 2 * (lane & 3);
      *reinterpret_cast<double2*>(dst + row * BN + col) = make_double2(acc[idx][0], acc[idx][1]);
      ++idx;
    }
  }
}

// The rotation's A digit planes, emitted by the projection's diagonal tiles
// (each holds every V row block of its 80 columns in shared memory once):
// row scales from row_amax (the previous rotation's row maxima), the same
// digits and layout as oz_slice_rows_kernel (oz_digits.cuh), so the planes
// -- and the rotation -- are bit-identical to the split pass they replace.
struct EmitArgs {
  const unsigned long long* row_amax;  // nullptr: no emission
  uint8_t* planes;                     // buffer 0's planes; buffer b at + b * buf_stride
  int64_t buf_stride, a_sl;            // bytes; a buffer's row scales start at its planes + a_sl
  int64_t chunk_rows, nkc;
};

// 16 rows (from row r0, valid below r_end) x the 80 (or 64) columns of
// block I held in sA ([k][A_LD], k-major): one 16-column group per thread
template <int BM, int A_LD>
__device__ __forceinline__ void emit_digits(const EmitArgs& em, const double* sA, int I, int64_t r0, int64_t r_end) {
  constexpr int GPB = BM / 16;                      // 16-column groups per block
  if (threadIdx.x >= BK * GPB) return;
  const int k = threadIdx.x / GPB, g = threadIdx.x % GPB;
  const int64_t r = r0 + k;
  const int64_t gc = int64_t(I) * GPB + g;           // global 16-column group
  if (r >= r_end || gc >= 2 * em.nkc) return;
  const double amax = __longlong_as_double(static_cast<long long>(em.row_amax[r]));
  const int e = oz_exponent(amax);
  const double scale = ldexp(1.0, 54 - e);
  double v[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) v[t] = sA[k * A_LD + 16 * g + t];
  uint4 d[OZ_S];
  oz_digits16(v, scale, d);
  const int64_t b = r / em.chunk_rows, rl = r % em.chunk_rows;
  uint8_t* base = em.planes + b * em.buf_stride;
  uint8_t* p = base + ((rl / OZ_BM) * em.nkc + (gc >> 1)) * OZ_A_STAGE + (gc & 1) * (OZ_BM * 16) +
               (rl % OZ_BM) * 16;
#pragma unroll
  for (int s = 0; s < OZ_S; ++s) *reinterpret_cast<uint4*>(p + s * OZ_A_SLICE) = d[s];
  if (gc == 0) reinterpret_cast<double*>(base + em.a_sl)[rl] = ldexp(1.0, e - 28);
}

template <int W, int STAGES>
__global__ void __launch_bounds__(128, 3)
gemm_tn_sym_kernel(const double* __restrict__ X, int64_t ldx, const double* __restrict__ Y, int64_t ldy,
                   int64_t rows, int64_t M, int T, int per_full, int64_t chunk_full, int per_diag,
                   int64_t chunk_diag, double* __restrict__ partial, const EmitArgs em) {
  using Cf = Cfg<2, 2, W, W, STAGES, true>;
  constexpr int G = 2 * W;
  extern __shared__ __align__(16) double smem[];
  const int c = blockIdx.x;
  const int n_full = T * (T - 1) / 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* dst = partial + int64_t(c) * (Cf::BM * Cf::BN);
  if (c < n_full * per_full) {
    // off-diagonal tile f -> (i, j), i < j
    int f = c / per_full;
    const int q = c % per_full;
    int i = 0;
    while (f >= T - 1 - i) { f -= T - 1 - i; ++i; }
    const int j = i + 1 + f;
    const int64_t kb = int64_t(q) * chunk_full, ke = min(rows, kb + chunk_full);
    double acc[W][W][2];
#pragma unroll
    for (int a = 0; a < W; ++a)
#pragma unroll
      for (int b = 0; b < W; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    if (kb < ke)
      mainloop<2, 2, W, W, STAGES, true>(acc, smem, X, ldx, Y, ldy, kb, ke, int64_t(i) * Cf::BM, M,
                                         int64_t(j) * Cf::BN, M);
    const int wm = warp / 2, wn = warp % 2;
#pragma unroll
    for (int a = 0; a < W; ++a) {
      const int r = wm * W * 8 + a * 8 + (lane >> 2);
#pragma unroll
      for (int b = 0; b < W; ++b) {
        const int cc = wn * W * 8 + b * 8 + 2 * (lane & 3);
        *reinterpret_cast<double2*>(dst + r * Cf::BN + cc) = make_double2(acc[a][b][0], acc[a][b][1]);
      }
    }
    return;
  }
  const int d = c - n_full * per_full;
  const int i = d / per_diag, q = d % per_diag;
  const int64_t kb = int64_t(q) * chunk_diag, ke = min(rows, kb + chunk_diag);
  double acc[diag_max_cells(G)][2];
#pragma unroll
  for (int a = 0; a < diag_max_cells(G); ++a) acc[a][0] = acc[a][1] = 0.0;
  const int lr = lane >> 2, lc = lane & 3;
  if (kb < ke) {
    int64_t r_stage = kb;
    pipeline<2, 2, W, W, STAGES, true>(
        smem, X, ldx, Y, ldy, kb, ke, int64_t(i) * Cf::BM, M, int64_t(i) * Cf::BN, M,
        [&](const double* sA, const double* sB) {
          if (em.row_amax) emit_digits<Cf::BM, Cf::A_LD>(em, sA, i, r_stage, ke);
          r_stage += BK;
          switch (warp) {
            case 0: diag_compute<G, 0, Cf::A_LD, Cf::B_LD>(acc, sA, sB, lr, lc); break;
            case 1: diag_compute<G, 1, Cf::A_LD, Cf::B_LD>(acc, sA, sB, lr, lc); break;
            case 2: diag_compute<G, 2, Cf::A_LD, Cf::B_LD>(acc, sA, sB, lr, lc); break;
            default: diag_compute<G, 3, Cf::A_LD, Cf::B_LD>(acc, sA, sB, lr, lc); break;
          }
        });
  }
  switch (warp) {
    case 0: diag_store<G, 0>(acc, dst, Cf::BN, lane); break;
    case 1: diag_store<G, 1>(acc, dst, Cf::BN, lane); break;
    case 2: diag_store<G, 2>(acc, dst, Cf::BN, lane); break;
    default: diag_store<G, 3>(acc, dst, Cf::BN, lane); break;
  }
}

// out[i, j] (i <= j) = sum of the tile's CTA partials, mirrored.  A block
// takes 32 consecutive elements; warp w sums the partials q = w, w + 8, ...
// (four independent loads in flight), and the eight warp sums are added in
// warp order: a fixed summation order, so P is reproducible run to run.
template <int BM>
__global__ void __launch_bounds__(256)
tn_sym_reduce_kernel(const double* __restrict__ partial, int T, int per_full, int per_diag, int64_t M,
                     double* __restrict__ out, int64_t ldo) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n_tiles = T * (T + 1) / 2;
  const int n_full = T * (T - 1) / 2;
  const int64_t total = int64_t(n_tiles) * BM * BM;
  const int64_t e = int64_t(blockIdx.x) * 32 + lane;
  bool ok = e < total;
  int64_t i = 0, j = 0;
  double s = 0.0;
  if (ok) {
    const int t = static_cast<int>(e / (BM * BM));
    const int rc = static_cast<int>(e % (BM * BM));
    const int2 tt = decode_tile(t, T, 1);
    i = int64_t(tt.x) * BM + rc / BM;
    j = int64_t(tt.y) * BM + rc % BM;
    ok = i < M && j < M && j >= i;
    if (ok) {
      int c0, cnt;
      if (tt.x == tt.y) {
        c0 = n_full * per_full + tt.x * per_diag;
        cnt = per_diag;
      } else {
        int f = 0;
        for (int a = 0; a < tt.x; ++a) f += T - 1 - a;
        f += tt.y - tt.x - 1;
        c0 = f * per_full;
        cnt = per_full;
      }
      const double* p = partial + int64_t(c0) * (BM * BM) + rc;
      constexpr int64_t S = int64_t(BM) * BM;
      int q = w;
      for (; q + 24 < cnt; q += 32) {
        const double a0 = p[q * S], a1 = p[(q + 8) * S], a2 = p[(q + 16) * S], a3 = p[(q + 24) * S];
        s += a0; s += a1; s += a2; s += a3;
      }
      for (; q < cnt; q += 8) s += p[q * S];
    }
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && ok) {
    s = red[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) s += red[k][lane];
    out[i * ldo + j] = s;
    if (j != i) out[j * ldo + i] = s;
  }
}

// ---------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------
template <int WARPS_M, int WARPS_N, int WTM, int WTN, int STAGES>
int launch_nn(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int64_t K,
              int64_t M2, double* out, int64_t ldo, int accumulate, double alpha, cudaStream_t st) {
  using Cf = Cfg<WARPS_M, WARPS_N, WTM, WTN, STAGES, false>;
  auto kern = gemm_nn_kernel<WARPS_M, WARPS_N, WTM, WTN, STAGES>;
  static unsigned long long attr_done = 0;
  if (swb_first_on_device(&attr_done)) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Cf::SMEM)));
  }
  const int64_t tm = (rows + Cf::BM - 1) / Cf::BM;
  const int tn = static_cast<int>((M2 + Cf::BN - 1) / Cf::BN);
  const int64_t grid = tm * tn;
  if (grid <= 0) return SWB_OK;
  if (grid > 0x7fffffffLL) return SWB_INVALID_PARAM;
  kern<<<static_cast<unsigned>(grid), Cf::THREADS, Cf::SMEM, st>>>(A, lda, B, ldb, rows, K, M2, out,
                                                                     ldo, accumulate, alpha, tn);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

// Split-K TN launches about this many waves of CTAs: with a single wave
// the CTAs that finish first leave their SMs idle for the rest of the
// kernel; several shorter waves keep every SM busy to the end (measured at
// c4: one wave 95.4 ms, 8 waves 82.9 ms).  SWB_TN_WAVES overrides (1..16).
int tn_waves() {
  static const int waves = [] {
    const char* e = getenv("SWB_TN_WAVES");
    const int v = e ? atoi(e) : 8;
    return v >= 1 && v <= 16 ? v : 8;
  }();
  return waves;
}

// TN plan: per_tile CTAs per output tile
struct TnPlan {
  int n_tiles, tn, per_tile, n_ctas;
  int64_t chunk_rows;
};

template <int BM, int BN>
TnPlan plan_tn(int64_t rows, int64_t M1, int64_t M2, int symmetric, int slots) {
  TnPlan p{};
  const int tm = static_cast<int>((M1 + BM - 1) / BM), tn = static_cast<int>((M2 + BN - 1) / BN);
  p.n_tiles = symmetric ? tm * (tm + 1) / 2 : tm * tn;  // symmetric => BM == BN, tm == tn
  p.tn = tn;
  int per = std::max(1, slots / p.n_tiles);
  const int64_t max_per = std::max<int64_t>(1, rows / 512);  // >= 512 rows per chunk
  if (per > max_per) per = static_cast<int>(max_per);
  int64_t cr = (rows + per - 1) / per;
  cr = std::max<int64_t>(BK, (cr + BK - 1) / BK * BK);
  p.chunk_rows = cr;
  p.per_tile = static_cast<int>(std::max<int64_t>(1, (rows + cr - 1) / cr));
  p.n_ctas = p.n_tiles * p.per_tile;
  return p;
}

enum TnKind { TN_80x80 = 0, TN_64x64 = 1, TN_80x16 = 2 };

TnKind choose_tn(int64_t M1, int64_t M2) {
  if (M2 <= 16) return TN_80x16;
  auto waste = [&](int b) { return ((M1 + b - 1) / b) * b * ((M2 + b - 1) / b) * b; };
  return waste(80) <= waste(64) ? TN_80x80 : TN_64x64;
}

constexpr int TN_STAGES = 3;

template <int WARPS_M, int WARPS_N, int WTM, int WTN>
int run_tn(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t rows, int64_t M1,
           int64_t M2, int symmetric, double* out, int64_t ldo, void* ws, size_t ws_bytes,
           cudaStream_t st, bool size_only, size_t* need) {
  using Cf = Cfg<WARPS_M, WARPS_N, WTM, WTN, TN_STAGES, true>;
  auto kern = gemm_tn_kernel<WARPS_M, WARPS_N, WTM, WTN, TN_STAGES>;
  static int occ_dev[64] = {};
  int& occ = occ_dev[swb_device()];
  if (occ == 0 && !size_only) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Cf::SMEM)));
    SWB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cf::THREADS, Cf::SMEM));
    if (occ < 1) occ = 1;
  }
  // size queries may run before any device call: bound the occupancy by 8
  // (the partial workspace grows with the CTA count)
  const int occ_used = occ > 0 ? occ : 8;
  TnPlan p = plan_tn<Cf::BM, Cf::BN>(rows, M1, M2, symmetric, swb_sm_count() * occ_used * tn_waves());
  const size_t part_bytes = sizeof(double) * size_t(p.n_ctas) * Cf::BM * Cf::BN;
  *need = part_bytes;
  if (size_only) return SWB_OK;
  if (ws_bytes < *need || ws == nullptr) return SWB_WORKSPACE_TOO_SMALL;
  double* partial = reinterpret_cast<double*>(ws);
  kern<<<p.n_ctas, Cf::THREADS, Cf::SMEM, st>>>(X, ldx, Y, ldy, rows, M1, M2, p.tn, symmetric, p.per_tile,
                                                p.chunk_rows, partial);
  SWB_CHECK_LAUNCH();
  const int64_t total = int64_t(p.n_tiles) * Cf::BM * Cf::BN;
  int rb = static_cast<int>(std::min<int64_t>((total + 255) / 256, int64_t(swb_sm_count()) * 8));
  tn_reduce_kernel<Cf::BM, Cf::BN><<<rb, 256, 0, st>>>(partial, p.tn, symmetric, p.n_tiles, p.per_tile, M1, M2,
                                                       out, ldo);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

template <int W>
int run_tn_sym(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t rows, int64_t M, double* out,
               int64_t ldo, void* ws, size_t ws_bytes, cudaStream_t st, bool size_only, size_t* need,
               const EmitArgs& em = EmitArgs{}) {
  using Cf = Cfg<2, 2, W, W, TN_STAGES, true>;
  constexpr int G = 2 * W;
  auto kern = gemm_tn_sym_kernel<W, TN_STAGES>;
  static int occ_dev[64] = {};
  int& occ = occ_dev[swb_device()];
  // SWB_TN_OCC=n (measurement knob): at most n CTAs per SM, by padding the
  // dynamic shared memory, to leave room for a co-running kernel
  static const size_t smem_req = [] {
    const char* e = getenv("SWB_TN_OCC");
    const int cap = e ? atoi(e) : 0;
    return cap >= 1 && cap <= 3 ? std::max<size_t>(Cf::SMEM, size_t(228 * 1024) / size_t(cap + 1) + 1024)
                                : size_t(Cf::SMEM);
  }();
  if (occ == 0 && !size_only) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_req)));
    SWB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cf::THREADS, smem_req));
    if (occ < 1) occ = 1;
  }
  const int slots = swb_sm_count() * (occ > 0 ? occ : 8) * tn_waves();
  const int T = static_cast<int>((M + Cf::BM - 1) / Cf::BM);
  const int n_full = T * (T - 1) / 2;
  // diagonal / full tile cost; emitting diagonal tiles also convert their
  // V block to digit planes, measured at ~0.1 of a full tile's stage
  // (SWB_TN_EMIT_COST overrides; the CTA counts per tile, and so P's
  // split-K summation order, then differ from the plain projection's)
  static const double emit_cost = [] {
    const char* e = getenv("SWB_TN_EMIT_COST");
    return e ? atof(e) : 0.1;
  }();
  const double ratio = double(diag_max_cells(G)) / double(W * W) + (em.row_amax ? emit_cost : 0.0);
  int per_full = std::max(1, static_cast<int>(slots / (n_full + ratio * T)));
  // >= 512 rows per chunk; when that leaves SMs without a CTA (c1: 16 K rows, one diagonal tile -> 18
  // CTAs) down to 128 rows, so the latency-bound small problems use the whole GPU
  int64_t min_rows = 512;
  if ((n_full + ratio * T) * double(rows / 512) < double(swb_sm_count())) min_rows = 128;
  const int64_t max_per = std::max<int64_t>(1, rows / min_rows);
  if (per_full > max_per) per_full = static_cast<int>(max_per);
  int per_diag = std::max(1, static_cast<int>(ratio * per_full + 0.5));
  int64_t chunk_full = std::max<int64_t>(BK, ((rows + per_full - 1) / per_full + BK - 1) / BK * BK);
  int64_t chunk_diag = std::max<int64_t>(BK, ((rows + per_diag - 1) / per_diag + BK - 1) / BK * BK);
  per_full = static_cast<int>((rows + chunk_full - 1) / chunk_full);
  per_diag = static_cast<int>((rows + chunk_diag - 1) / chunk_diag);
  if (per_full < 1) per_full = 1;
  if (per_diag < 1) per_diag = 1;
  const int n_ctas = n_full * per_full + T * per_diag;
  *need = sizeof(double) * size_t(n_ctas) * Cf::BM * Cf::BN;
  if (size_only) return SWB_OK;
  if (ws_bytes < *need || ws == nullptr) return SWB_WORKSPACE_TOO_SMALL;
  double* partial = reinterpret_cast<double*>(ws);
  kern<<<n_ctas, Cf::THREADS, smem_req, st>>>(X, ldx, Y, ldy, rows, M, T, per_full, chunk_full, per_diag, chunk_diag,
                                              partial, em);
  SWB_CHECK_LAUNCH();
  const int64_t total = int64_t(T * (T + 1) / 2) * Cf::BM * Cf::BN;
  const unsigned rb = static_cast<unsigned>((total + 31) / 32);
  tn_sym_reduce_kernel<Cf::BM><<<rb, 256, 0, st>>>(partial, T, per_full, per_diag, M, out, ldo);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

int dispatch_tn(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t rows, int64_t M1,
                int64_t M2, int symmetric, double* out, int64_t ldo, void* ws, size_t ws_bytes,
                cudaStream_t st, bool size_only, size_t* need, const EmitArgs& em = EmitArgs{}) {
  switch (choose_tn(M1, M2)) {
    case TN_80x80:
      if (symmetric)
        return run_tn_sym<5>(X, ldx, Y, ldy, rows, M1, out, ldo, ws, ws_bytes, st, size_only, need, em);
      return run_tn<2, 2, 5, 5>(X, ldx, Y, ldy, rows, M1, M2, symmetric, out, ldo, ws, ws_bytes, st,
                                size_only, need);
    case TN_64x64:
      if (symmetric)
        return run_tn_sym<4>(X, ldx, Y, ldy, rows, M1, out, ldo, ws, ws_bytes, st, size_only, need, em);
      return run_tn<2, 2, 4, 4>(X, ldx, Y, ldy, rows, M1, M2, symmetric, out, ldo, ws, ws_bytes, st,
                                size_only, need);
    default:
      return run_tn<2, 2, 5, 1>(X, ldx, Y, ldy, rows, M1, M2, 0, out, ldo, ws, ws_bytes, st,
                                size_only, need);
  }
}

}  // namespace

extern "C" int swb_oz_layout_info(int64_t rows, int64_t K, int64_t M2, int64_t* info);

extern "C" size_t swb_gemm_tn_workspace_bytes(int64_t rows, int64_t M1, int64_t M2) {
  size_t need = 0;
  if (rows <= 0 || M1 <= 0 || M2 <= 0) return 0;
  dispatch_tn(nullptr, 0, nullptr, 0, rows, M1, M2, 1, nullptr, 0, nullptr, 0, nullptr, true, &need);
  size_t need2 = 0;
  dispatch_tn(nullptr, 0, nullptr, 0, rows, M1, M2, 0, nullptr, 0, nullptr, 0, nullptr, true, &need2);
  return need > need2 ? need : need2;
}

extern "C" int swb_gemm_tn(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t rows,
                           int64_t M1, int64_t M2, int symmetric, double* out, int64_t ldo,
                           void* workspace, size_t workspace_bytes, void* stream) {
  if (M1 <= 0 || M2 <= 0 || rows < 0 || !out) return SWB_INVALID_PARAM;
  if (ldx < M1 || ldy < M2 || ldo < M2 || (ldx & 1) || (ldy & 1)) return SWB_INVALID_PARAM;
  if (symmetric && M1 != M2) return SWB_INVALID_PARAM;
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 15) return SWB_INVALID_PARAM;
  cudaStream_t st = swb_stream(stream);
  if (rows == 0) {
    for (int64_t i = 0; i < M1; ++i)
      SWB_CUDA_TRY(cudaMemsetAsync(out + i * ldo, 0, sizeof(double) * M2, st));
    return SWB_OK;
  }
  size_t need = 0;
  return dispatch_tn(X, ldx, Y, ldy, rows, M1, M2, symmetric, out, ldo, workspace, workspace_bytes, st,
                     false, &need);
}

int swb_gemm_nn_alpha(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int64_t K,
                      int64_t M2, double* out, int64_t ldo, int accumulate, double alpha, cudaStream_t st) {
  if (rows < 0 || K <= 0 || M2 <= 0 || !A || !B || !out) return SWB_INVALID_PARAM;
  if (lda < K || ldb < M2 || ldo < M2 || (lda & 1) || (ldo & 1)) return SWB_INVALID_PARAM;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(out)) & 15) return SWB_INVALID_PARAM;
  if (reinterpret_cast<uintptr_t>(B) & 7) return SWB_INVALID_PARAM;
  if (rows == 0) return SWB_OK;
  // pick the column tile that wastes the least of M2
  auto padded = [&](int64_t b) { return (M2 + b - 1) / b * b; };
  const int64_t p80 = padded(80), p64 = padded(64), p128 = padded(128), p32 = padded(32);
  // (ties prefer the 4-warp configurations: the 8-warp 128-column tile is
  // register-capped at two CTAs per SM)
  int64_t best = p80;
  int which = 80;
  if (p64 < best) { best = p64; which = 64; }
  if (p128 < best) { best = p128; which = 128; }
  if (p32 < best) { best = p32; which = 32; }
  switch (which) {
    case 128: return launch_nn<4, 2, 4, 8, 3>(A, lda, B, ldb, rows, K, M2, out, ldo, accumulate, alpha, st);
    case 64: return launch_nn<2, 2, 8, 4, 3>(A, lda, B, ldb, rows, K, M2, out, ldo, accumulate, alpha, st);
    case 32: return launch_nn<4, 2, 4, 2, 3>(A, lda, B, ldb, rows, K, M2, out, ldo, accumulate, alpha, st);
    // 4 warps x (64 x 40) warp tiles: 40 independent DMMAs per k-step per warp
    // measured best on B200 (tools/gemm_tune.cu: 33.5 vs 32.9 TFLOP/s for 8 x (32 x 40))
    default: return launch_nn<2, 2, 8, 5, 3>(A, lda, B, ldb, rows, K, M2, out, ldo, accumulate, alpha, st);
  }
}

extern "C" int swb_gemm_nn(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows,
                           int64_t K, int64_t M2, double* out, int64_t ldo, int accumulate,
                           void* stream) {
  return swb_gemm_nn_alpha(A, lda, B, ldb, rows, K, M2, out, ldo, accumulate, 1.0, swb_stream(stream));
}

extern "C" int swb_gemm_nn_ex(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows,
                              int64_t K, int64_t M2, double* out, int64_t ldo, int accumulate, double alpha,
                              void* stream) {
  return swb_gemm_nn_alpha(A, lda, B, ldb, rows, K, M2, out, ldo, accumulate, alpha, swb_stream(stream));
}

// ---------------------------------------------------------------------------
// FP64 tensor-core peak probe (measurement only): back-to-back independent
// DMMA.8x8x4 on every SM; bench.py times it to get the live FP64 roofline.
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(256) dmma_probe_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_8x8x4(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
}  // namespace

extern "C" int swb_fp64_peak_probe(int iters, double* sink, double* flops_out, void* stream) {
  if (iters <= 0 || !sink || !flops_out) return SWB_INVALID_PARAM;
  const int blocks = swb_sm_count() * 2;
  dmma_probe_kernel<<<blocks, 256, 0, swb_stream(stream)>>>(sink, iters);
  SWB_CHECK_LAUNCH();
  *flops_out = 2.0 * 256.0 * 8.0 * double(iters) * double(blocks) * 8.0;  // 8 warps per block
  return SWB_OK;
}

// The symmetric projection P = X^T Y (swb_gemm_tn, symmetric) whose diagonal
// tiles also emit the INT8 rotation's A digit planes of X (rows x M) into an
// oz workspace sized by swb_oz_gemm_nn_workspace_bytes_full(rows, M, M2), row
// scales from row_amax (bits of max_c |X[r, c]|): the digit split of the
// rotation that follows is then not needed (swb_oz_gemm_planes_ex on buffers
// 0 .. chunks-1).  Column groups past M inside the last 32-column K chunk are
// left untouched: the caller keeps them zero.
extern "C" int swb_gemm_tn_sym_emit(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t rows,
                                    int64_t M, double* out, int64_t ldo, void* workspace, size_t workspace_bytes,
                                    const unsigned long long* row_amax, int64_t M2, void* oz_workspace,
                                    size_t oz_workspace_bytes, void* stream) {
  if (M <= 0 || rows <= 0 || !out || !row_amax || !oz_workspace || M2 < M) return SWB_INVALID_PARAM;
  if (ldx < M || ldy < M || ldo < M || (ldx & 1) || (ldy & 1)) return SWB_INVALID_PARAM;
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 15) return SWB_INVALID_PARAM;
  if (choose_tn(M, M) == TN_80x16) return SWB_INVALID_PARAM;
  int64_t info[5];
  int rc = swb_oz_layout_info(rows, M, M2, info);
  if (rc) return rc;
  const int64_t nbuf = (rows + info[0] - 1) / info[0];
  if (oz_workspace_bytes < size_t(info[2] + nbuf * info[4])) return SWB_WORKSPACE_TOO_SMALL;
  EmitArgs em{row_amax, static_cast<uint8_t*>(oz_workspace) + info[2], info[4], info[3], info[0], info[1]};
  size_t need = 0;
  return dispatch_tn(X, ldx, Y, ldy, rows, M, M, 1, out, ldo, workspace, workspace_bytes, swb_stream(stream), false,
                     &need, em);
}
