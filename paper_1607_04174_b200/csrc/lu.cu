// Dense FP64 LU with partial pivoting, 1-norm condition estimate and solve:
// the seed system of the fast random walker (reference fastrw.py:332-344,
// which calls LAPACK getrf / gecon / getrs through scipy).
//
// Row-major storage.  Right-looking blocked LU (panel width 32):
//   panel  : one CTA factors rows [k,n) x cols [k,k+32) (the panel lives in
//            shared memory when it fits, the tail rows stay in global)
//   swaps  : the panel's row interchanges applied to the other columns
//   trsm   : U12 = L11^-1 A12
//   update : A22 -= L21 U12 on the DMMA tensor-core GEMM
// rcond follows LAPACK dgecon: Higham's dlacn2 estimator of
// ||U^-1 L^-1||_1 (single CTA), rcond = 1/(anorm * est).
#include "swb_common.cuh"

namespace {

constexpr int NB = 32;           // panel width
constexpr int PANEL_THREADS = 1024;
constexpr int PANEL_LD = NB + 1;  // smem panel row stride (doubles)
constexpr int PANEL_SMEM_ROWS = 840;  // 840*33*8 = 221,760 B

struct ArgMax { double v; int i; };

__device__ __forceinline__ ArgMax argmax_merge(ArgMax a, ArgMax b) {
  // idamax semantics: larger |value|, ties -> smaller index
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__device__ ArgMax block_argmax(ArgMax a, ArgMax* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
    a = argmax_merge(a, b);
  }
  if (lane == 0) sh[warp] = a;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    a = lane < nw ? sh[lane] : ArgMax{-1.0, 0x7fffffff};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgMax b;
      b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
      b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
      a = argmax_merge(a, b);
    }
    if (lane == 0) sh[0] = a;
  }
  __syncthreads();
  ArgMax r = sh[0];
  __syncthreads();
  return r;
}

// column sums of |A| (for the 1-norm)
// cs[j] = sum_i |A[i, j]|: a (32 x 8) block per 32 columns, the 8 row
// groups (rows ty, ty + 8, ...) reduced in a fixed order -- coalesced rows
// and 8 independent load streams instead of one serial column walk
__global__ void __launch_bounds__(256) colabs_kernel(const double* __restrict__ A, int64_t n, int64_t lda,
                                                     double* __restrict__ cs) {
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j = blockIdx.x * 32 + tx;
  double s = 0.0;
  if (j < n)
    for (int64_t i = ty; i < n; i += 8) s += fabs(A[i * lda + j]);
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && j < n) {
    double t = red[0][tx];
#pragma unroll
    for (int g = 1; g < 8; ++g) t += red[g][tx];
    cs[j] = t;
  }
}

__global__ void max_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
  __shared__ double red[1024];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = v[i];
    m = (x > m || x != x) ? x : m;  // NaN propagates like np.linalg.norm
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double b = red[threadIdx.x + o];
      if (b > red[threadIdx.x] || b != b) red[threadIdx.x] = b;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// Factor the panel rows [k,n) x cols [k,k+w).  piv[k+jj] = global pivot row.
__global__ void __launch_bounds__(PANEL_THREADS)
panel_kernel(double* __restrict__ A, int64_t n, int64_t lda, int64_t k, int w, int32_t* __restrict__ piv,
             int32_t* __restrict__ zero_pivot) {
  extern __shared__ double sp[];
  __shared__ ArgMax sh[32];
  __shared__ double prow[NB];
  const int64_t rows = n - k;
  const int64_t srows = rows < PANEL_SMEM_ROWS ? rows : PANEL_SMEM_ROWS;
  auto row = [&](int64_t i) -> double* { return i < srows ? sp + i * PANEL_LD : A + (k + i) * lda + k; };
  for (int64_t e = threadIdx.x; e < srows * w; e += blockDim.x) {
    const int64_t i = e / w, c = e % w;
    sp[i * PANEL_LD + c] = A[(k + i) * lda + k + c];
  }
  __syncthreads();
  // Thread t owns rows i = t (mod blockDim): its pivot-search candidates and
  // its row updates are the same rows, so a column step needs only two
  // barriers (after the warp-level pivot partials, after the swap).
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int jj = 0; jj < w; ++jj) {
    ArgMax a{-1.0, 0x7fffffff};
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
      if (i < jj) continue;
      const double v = fabs(row(i)[jj]);
      a = argmax_merge(a, ArgMax{v != v ? __longlong_as_double(0x7ff0000000000000LL) : v, static_cast<int>(i)});
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgMax b;
      b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
      b.i = __shfl_xor_sync(0xffffffffu, a.i, o);
      a = argmax_merge(a, b);
    }
    if (lane == 0) sh[warp] = a;
    __syncthreads();
    // every warp reduces the per-warp partials itself (shuffles, no extra barrier)
    ArgMax best = lane < nwarp ? sh[lane] : ArgMax{-1.0, 0x7fffffff};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgMax b;
      b.v = __shfl_xor_sync(0xffffffffu, best.v, o);
      b.i = __shfl_xor_sync(0xffffffffu, best.i, o);
      best = argmax_merge(best, b);
    }
    const int p = best.i;
    if (threadIdx.x == 0) piv[k + jj] = static_cast<int32_t>(k + p);
    for (int c = threadIdx.x; c < w; c += blockDim.x) {
      double* rj = row(jj);
      double* rp = row(p);
      const double t = rj[c];
      if (p != jj) { rj[c] = rp[c]; rp[c] = t; }
      prow[c] = p != jj ? rj[c] : t;
    }
    __syncthreads();
    const double pv = prow[jj];
    if (pv == 0.0) {
      if (threadIdx.x == 0) atomicExch(zero_pivot, 1);
      continue;  // LAPACK: column left unscaled, info > 0
    }
    // LAPACK dgetf2 / dgetrf2: scale by the reciprocal when |pivot| >= sfmin
    const bool recip = fabs(pv) >= 2.2250738585072014e-308;
    const double rinv = 1.0 / pv;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
      if (i <= jj) continue;
      double* ri = row(i);
      const double l = recip ? ri[jj] * rinv : ri[jj] / pv;
      ri[jj] = l;
      for (int c = jj + 1; c < w; ++c) ri[c] -= l * prow[c];
    }
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < srows * w; e += blockDim.x) {
    const int64_t i = e / w, c = e % w;
    A[(k + i) * lda + k + c] = sp[i * PANEL_LD + c];
  }
}

// Register-resident panel (rows <= 1024, width <= RW): thread t owns panel
// row t in registers for the whole factorisation, so a column step is a
// warp-shuffle pivot search, one barrier for the per-warp partials, a row
// swap + pivot-row broadcast through shared memory (second barrier) and a
// rank-1 update in registers -- no shared-memory traffic for the update.
constexpr int RW = 16;

__global__ void __launch_bounds__(1024)
panel_reg_kernel(double* __restrict__ A, int64_t n, int64_t lda, int64_t k, int w, int32_t* __restrict__ piv,
                 int32_t* __restrict__ zero_pivot) {
  __shared__ ArgMax sh[32];
  __shared__ double prow[RW];
  __shared__ double swp[RW];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarp = blockDim.x >> 5;
  const int64_t rows = n - k;
  const bool mine = t < rows;
  double a[RW];
#pragma unroll
  for (int c = 0; c < RW; ++c) a[c] = (mine && c < w) ? A[(k + t) * lda + k + c] : 0.0;
#pragma unroll
  for (int jj = 0; jj < RW; ++jj) {
    if (jj >= w) break;
    ArgMax best{-1.0, 0x7fffffff};
    if (mine && t >= jj) {
      const double v = fabs(a[jj]);
      best = ArgMax{v != v ? __longlong_as_double(0x7ff0000000000000LL) : v, t};
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgMax b;
      b.v = __shfl_xor_sync(0xffffffffu, best.v, o);
      b.i = __shfl_xor_sync(0xffffffffu, best.i, o);
      best = argmax_merge(best, b);
    }
    if (lane == 0) sh[warp] = best;
    __syncthreads();
    best = lane < nwarp ? sh[lane] : ArgMax{-1.0, 0x7fffffff};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgMax b;
      b.v = __shfl_xor_sync(0xffffffffu, best.v, o);
      b.i = __shfl_xor_sync(0xffffffffu, best.i, o);
      best = argmax_merge(best, b);
    }
    const int p = best.i;
    if (t == 0) piv[k + jj] = static_cast<int32_t>(k + p);
    if (t == p) {
#pragma unroll
      for (int c = 0; c < RW; ++c) prow[c] = a[c];       // the new row jj
    }
    if (t == jj && p != jj) {
#pragma unroll
      for (int c = 0; c < RW; ++c) swp[c] = a[c];        // old row jj goes to row p
    }
    __syncthreads();
    if (p != jj) {
      if (t == jj) {
#pragma unroll
        for (int c = 0; c < RW; ++c) a[c] = prow[c];
      } else if (t == p) {
#pragma unroll
        for (int c = 0; c < RW; ++c) a[c] = swp[c];
      }
    }
    const double pv = prow[jj];
    if (pv == 0.0) {
      if (t == 0) atomicExch(zero_pivot, 1);
      continue;  // LAPACK: column left unscaled, info > 0
    }
    if (mine && t > jj) {
      // LAPACK dgetf2 / dgetrf2: scale by the reciprocal when |pivot| >= sfmin
      const double l = fabs(pv) >= 2.2250738585072014e-308 ? a[jj] * (1.0 / pv) : a[jj] / pv;
      a[jj] = l;
#pragma unroll
      for (int c = jj + 1; c < RW; ++c) a[c] -= l * prow[c];
    }
  }
  if (mine) {
#pragma unroll
    for (int c = 0; c < RW; ++c)
      if (c < w) A[(k + t) * lda + k + c] = a[c];
  }
}

// apply the panel's interchanges to columns outside [k, k+w)
__global__ void swap_kernel(double* __restrict__ A, int64_t n, int64_t lda, int64_t k, int w,
                            const int32_t* __restrict__ piv) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t ncols = n - w;
  if (t >= ncols) return;
  const int64_t c = t < k ? t : t + w;
  for (int jj = 0; jj < w; ++jj) {
    const int64_t p = piv[k + jj];
    if (p != k + jj) {
      double* a = A + (k + jj) * lda + c;
      double* b = A + p * lda + c;
      const double x = *a; *a = *b; *b = x;
    }
  }
}

// U12 = L11^-1 A12 for columns [k+w, n)
__global__ void trsm_kernel(double* __restrict__ A, int64_t n, int64_t lda, int64_t k, int w) {
  __shared__ double L[NB][NB + 1];
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) L[e / w][e % w] = A[(k + e / w) * lda + k + e % w];
  __syncthreads();
  const int64_t c = k + w + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (c >= n) return;
  double x[NB];
#pragma unroll
  for (int r = 0; r < NB; ++r)
    if (r < w) x[r] = A[(k + r) * lda + c];
#pragma unroll
  for (int r = 0; r < NB; ++r) {
    if (r >= w) break;
    double s = x[r];
#pragma unroll
    for (int q = 0; q < NB; ++q)
      if (q < r) s -= L[r][q] * x[q];
    x[r] = s;
    A[(k + r) * lda + c] = s;
  }
}

// ---- triangular solves on the LU factors (single CTA, blocked by 32) ----
// op: 0 = L (unit lower), 1 = U (upper), 2 = U^T (lower), 3 = L^T (unit upper)
// B is n x nrhs (ldb) in global memory.
__device__ void tri_solve(const double* __restrict__ LU, int64_t n, int64_t lda, double* B, int64_t nrhs,
                          int64_t ldb, int op) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool forward = (op == 0 || op == 2);
  const bool unit = (op == 0 || op == 3);
  // element (i, j) of the triangular operator T
  auto T = [&](int64_t i, int64_t j) -> double { return (op == 2 || op == 3) ? LU[j * lda + i] : LU[i * lda + j]; };
  const int64_t nblk = (n + 31) / 32;
  // the diagonal block, staged so that the serial chain below waits on
  // shared-memory loads rather than global ones
  __shared__ double sblk[32 * 33];
  for (int64_t bb = 0; bb < nblk; ++bb) {
    const int64_t blk = forward ? bb : nblk - 1 - bb;
    const int64_t b0 = blk * 32, b1 = min(n, b0 + 32);
    const int bs = static_cast<int>(b1 - b0);
    for (int e = threadIdx.x; e < bs * bs; e += blockDim.x) sblk[(e / bs) * 33 + e % bs] = T(b0 + e / bs, b0 + e % bs);
    __syncthreads();
    // diagonal block: warp per rhs column, lane per row
    for (int64_t c = warp; c < nrhs; c += nw) {
      double x = lane < bs ? B[(b0 + lane) * ldb + c] : 0.0;
      for (int s = 0; s < bs; ++s) {
        const int r = forward ? s : bs - 1 - s;
        double xr = __shfl_sync(0xffffffffu, x, r);
        if (!unit) xr = xr / sblk[r * 33 + r];
        if (lane == r) x = xr;
        const bool below = forward ? (lane > r) : (lane < r);
        if (below && lane < bs) x -= sblk[lane * 33 + r] * xr;
      }
      if (lane < bs) B[(b0 + lane) * ldb + c] = x;
    }
    __syncthreads();
    // trailing update of the remaining rows
    const int64_t r_lo = forward ? b1 : 0, r_hi = forward ? n : b0;
    const int64_t cnt = (r_hi - r_lo) * nrhs;
    for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) {
      const int64_t i = r_lo + e / nrhs, c = e % nrhs;
      double s = B[i * ldb + c];
      for (int64_t q = b0; q < b1; ++q) s -= T(i, q) * B[q * ldb + c];
      B[i * ldb + c] = s;
    }
    __syncthreads();
  }
}

constexpr int64_t GETRS_SMEM_N = 12288;   // 2 * 4 * n bytes of shared memory

__global__ void __launch_bounds__(1024)
getrs_kernel(const double* __restrict__ LU, int64_t n, int64_t lda, const int32_t* __restrict__ piv,
             double* B, int64_t nrhs, int64_t ldb, int32_t* __restrict__ perm, double* __restrict__ tmp) {
  // B <- P^T B (LAPACK dlaswp forward): compose the interchanges into one
  // permutation (thread 0, O(n) dependent swaps -- in shared memory when it
  // fits, which keeps the serial chain at shared-memory latency), then
  // gather the rows in parallel
  extern __shared__ int32_t sperm[];
  const bool in_smem = n <= GETRS_SMEM_N;
  int32_t* pm = in_smem ? sperm : perm;
  int32_t* pv = in_smem ? sperm + n : nullptr;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    pm[j] = static_cast<int32_t>(j);
    if (in_smem) pv[j] = piv[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t j = 0; j < n; ++j) {
      const int64_t p = in_smem ? pv[j] : piv[j];
      if (p != j) { const int32_t t = pm[j]; pm[j] = pm[p]; pm[p] = t; }
    }
  }
  __syncthreads();
  if (in_smem)
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) perm[j] = pm[j];
  __syncthreads();
  for (int64_t e = threadIdx.x; e < n * nrhs; e += blockDim.x) {
    const int64_t i = e / nrhs, c = e % nrhs;
    tmp[e] = B[int64_t(perm[i]) * ldb + c];
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < n * nrhs; e += blockDim.x) {
    const int64_t i = e / nrhs, c = e % nrhs;
    B[i * ldb + c] = tmp[e];
  }
  __syncthreads();
  tri_solve(LU, n, lda, B, nrhs, ldb, 0);
  tri_solve(LU, n, lda, B, nrhs, ldb, 1);
}

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

__device__ int block_idamax(const double* x, int64_t n, ArgMax* sh) {
  ArgMax a{-1.0, 0x7fffffff};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a = argmax_merge(a, ArgMax{fabs(x[i]), static_cast<int>(i)});
  return block_argmax(a, sh).i;
}

// LAPACK dlacn2 (Higham's 1-norm estimator of ||A^-1||_1, the heart of
// dgecon), kase loop unrolled into straight-line code.  inv() / inv_t()
// overwrite x (n) with A^-1 x / A^-T x; the whole CTA calls them.
template <class Inv, class InvT>
__device__ double dlacn2_est(int64_t n, double* __restrict__ x, int32_t* __restrict__ isgn, Inv inv, InvT inv_t,
                             double* red, ArgMax* sh, int* flag) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = 1.0 / double(n);
  __syncthreads();
  inv();
  double est;
  if (n == 1) return fabs(x[0]);
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += fabs(x[i]);
  est = block_sum(s, red);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const bool pos = x[i] >= 0.0;
    x[i] = pos ? 1.0 : -1.0;
    isgn[i] = pos ? 1 : -1;
  }
  __syncthreads();
  inv_t();
  int j = block_idamax(x, n, sh);
  int iter = 2;
  while (true) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = (i == j) ? 1.0 : 0.0;
    __syncthreads();
    inv();
    const double estold = est;
    s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += fabs(x[i]);
    est = block_sum(s, red);
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      if ((x[i] >= 0.0 ? 1 : -1) != isgn[i]) *flag = 1;
    __syncthreads();
    const bool changed = *flag != 0;
    __syncthreads();
    if (!changed || est <= estold) break;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const bool pos = x[i] >= 0.0;
      x[i] = pos ? 1.0 : -1.0;
      isgn[i] = pos ? 1 : -1;
    }
    __syncthreads();
    inv_t();
    const int jlast = j;
    j = block_idamax(x, n, sh);
    if (x[jlast] != fabs(x[j]) && iter < 5) { ++iter; continue; }
    break;
  }
  // the alternative estimate (dlacn2's final step)
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double sgn = (i & 1) ? -1.0 : 1.0;
    x[i] = sgn * (1.0 + double(i) / double(n - 1));
  }
  __syncthreads();
  inv();
  s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += fabs(x[i]);
  const double temp = 2.0 * (block_sum(s, red) / double(3 * n));
  return temp > est ? temp : est;
}

// dgecon (norm '1'): rcond = 1 / (anorm * est) on the LU factors of A.
__global__ void __launch_bounds__(1024)
gecon_kernel(const double* __restrict__ LU, int64_t n, int64_t lda, const double* __restrict__ anorm_p,
             double* __restrict__ x, int32_t* __restrict__ isgn, double* __restrict__ rcond_out) {
  __shared__ double red[32];
  __shared__ ArgMax sh[32];
  __shared__ int flag;
  const double anorm = *anorm_p;
  if (n == 0) { if (threadIdx.x == 0) *rcond_out = 1.0; return; }
  if (!(anorm > 0.0)) { if (threadIdx.x == 0) *rcond_out = (anorm == 0.0) ? 0.0 : anorm; return; }
  // exactly singular U -> rcond 0 (dlatrs would return scale 0)
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    if (LU[i * lda + i] == 0.0) flag = 1;
  __syncthreads();
  if (flag) { if (threadIdx.x == 0) *rcond_out = 0.0; return; }
  // ||A^-1||_1 == ||U^-1 L^-1||_1: the row permutation does not change column sums
  auto inv = [&]() { tri_solve(LU, n, lda, x, 1, 1, 0); tri_solve(LU, n, lda, x, 1, 1, 1); };
  auto inv_t = [&]() { tri_solve(LU, n, lda, x, 1, 1, 2); tri_solve(LU, n, lda, x, 1, 1, 3); };
  const double est = dlacn2_est(n, x, isgn, inv, inv_t, red, sh, &flag);
  if (threadIdx.x == 0) *rcond_out = est != 0.0 ? (1.0 / est) / anorm : 0.0;
}

// dgecon of A = I - Ut Vt^T (n x n, Ut / Vt n x r row-major, ld ldr) through
// the Woodbury identity, with K = I_r - Vt^T Ut factored (LU, pivots pk):
//   A^-1 x  = x + Ut K^-1 (Vt^T x),   A^-T x = x + Vt K^-T (Ut^T x).
// The estimator sees the same A^-1 / A^-T products as dgecon on A itself.
__global__ void __launch_bounds__(1024)
gecon_wb_kernel(int64_t n, int64_t r, const double* __restrict__ Ut, const double* __restrict__ Vt, int64_t ldr,
                const double* __restrict__ K, int64_t ldk, const int32_t* __restrict__ pk,
                const double* __restrict__ anorm_p, double* __restrict__ x, double* __restrict__ t,
                int32_t* __restrict__ isgn, double* __restrict__ rcond_out) {
  __shared__ double red[32];
  __shared__ ArgMax sh[32];
  __shared__ int flag;
  const double anorm = *anorm_p;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (n == 0) { if (threadIdx.x == 0) *rcond_out = 1.0; return; }
  if (!(anorm > 0.0)) { if (threadIdx.x == 0) *rcond_out = (anorm == 0.0) ? 0.0 : anorm; return; }
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < r; i += blockDim.x)
    if (K[i * ldk + i] == 0.0) flag = 1;           // K singular <=> A singular
  __syncthreads();
  if (flag) { if (threadIdx.x == 0) *rcond_out = 0.0; return; }
  // t = X^T x (X n x r), column by thread
  auto proj = [&](const double* X) {
    for (int64_t j = threadIdx.x; j < r; j += blockDim.x) {
      double a = 0.0;
      for (int64_t i = 0; i < n; ++i) a = fma(X[i * ldr + j], x[i], a);
      t[j] = a;
    }
    __syncthreads();
  };
  // x += X t, row by warp
  auto add = [&](const double* X) {
    for (int64_t i = warp; i < n; i += nw) {
      double a = 0.0;
      for (int64_t j = lane; j < r; j += 32) a = fma(X[i * ldr + j], t[j], a);
      a = warp_sum(a);
      if (lane == 0) x[i] += a;
    }
    __syncthreads();
  };
  auto perm = [&](bool forward) {          // t <- P t (getrs order) or P^T t
    if (threadIdx.x == 0) {
      if (forward) {
        for (int64_t j = 0; j < r; ++j) {
          const int64_t p = pk[j];
          if (p != j) { const double v = t[j]; t[j] = t[p]; t[p] = v; }
        }
      } else {
        for (int64_t j = r - 1; j >= 0; --j) {
          const int64_t p = pk[j];
          if (p != j) { const double v = t[j]; t[j] = t[p]; t[p] = v; }
        }
      }
    }
    __syncthreads();
  };
  auto inv = [&]() {                        // x <- A^-1 x
    proj(Vt);
    perm(true);
    tri_solve(K, r, ldk, t, 1, 1, 0);
    tri_solve(K, r, ldk, t, 1, 1, 1);
    add(Ut);
  };
  auto inv_t = [&]() {                      // x <- A^-T x
    proj(Ut);
    tri_solve(K, r, ldk, t, 1, 1, 2);
    tri_solve(K, r, ldk, t, 1, 1, 3);
    perm(false);
    add(Vt);
  };
  const double est = dlacn2_est(n, x, isgn, inv, inv_t, red, sh, &flag);
  if (threadIdx.x == 0) *rcond_out = est != 0.0 ? (1.0 / est) / anorm : 0.0;
}

}  // namespace

// internal: out = alpha*A*B (+ out), see dgemm.cu
int swb_gemm_nn_alpha(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int64_t K,
                      int64_t M2, double* out, int64_t ldo, int accumulate, double alpha, cudaStream_t st);

extern "C" size_t swb_lu_workspace_bytes(int64_t n) {
  // column sums (n) + zero-pivot flag + gecon scratch (x: n, isgn: n)
  return swb_align_up(sizeof(double) * size_t(n + 1), 256) + 256 +
         swb_align_up(sizeof(double) * size_t(n + 1), 256) + swb_align_up(sizeof(int32_t) * size_t(n + 1), 256);
}

// ---- small systems in one launch -----------------------------------------
// n <= SMALL_N: the whole of A in shared memory (ld n | 1 against bank
// conflicts on the column walks): the 1-norm, LU with partial pivoting
// (dgetf2: idamax pivot with NaN as the largest, ties to the lowest row;
// reciprocal scaling when |pivot| >= sfmin; a zero pivot leaves its column
// unscaled), getrs on the nrhs right-hand sides in B, and dgecon's estimate
// on the factors -- replacing the panel / swap / trsm / GEMM launches per
// panel, getrs and gecon of the blocked path (the seed systems of the small
// configurations are latency-bound).  The factors and pivots are written
// back to A / piv as swb_lu_factor leaves them.
constexpr int SMALL_N = 160;
constexpr int SMALL_THREADS = 512;

__global__ void __launch_bounds__(SMALL_THREADS)
small_dense_kernel(double* __restrict__ A_g, int64_t n_, int64_t lda, int32_t* __restrict__ piv_g,
                   double* __restrict__ B, int64_t nrhs, int64_t ldb, double* __restrict__ anorm_out,
                   double* __restrict__ rcond_out, int with_rcond) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ ArgMax sh[32];
  __shared__ int flag;
  __shared__ int zero_pivot;
  const int n = static_cast<int>(n_);
  const int ld = n | 1;
  double* A = sm;
  double* x = A + size_t(n) * ld;
  int32_t* isgn = reinterpret_cast<int32_t*>(x + n);
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < n * n; e += nt) A[(e / n) * ld + e % n] = A_g[int64_t(e / n) * lda + e % n];
  if (tid == 0) zero_pivot = 0;
  __syncthreads();
  // 1-norm of A (max column sum)
  double cmax = 0.0;
  for (int j = tid; j < n; j += nt) {
    double c = 0.0;
    for (int i = 0; i < n; ++i) c += fabs(A[i * ld + j]);
    cmax = (c > cmax || c != c) ? c : cmax;
  }
  {
    ArgMax a{cmax, tid};
    const double anorm = block_argmax(a, sh).v;
    if (tid == 0) *anorm_out = anorm;
  }
  // LU with partial pivoting
  for (int j = 0; j < n; ++j) {
    ArgMax a{-1.0, 0x7fffffff};
    for (int i = j + tid; i < n; i += nt) {
      const double v = fabs(A[i * ld + j]);
      a = argmax_merge(a, ArgMax{v != v ? __longlong_as_double(0x7ff0000000000000LL) : v, i});
    }
    const int p = block_argmax(a, sh).i;
    if (tid == 0) piv_g[j] = p;
    if (p != j)
      for (int c = tid; c < n; c += nt) {
        const double t = A[j * ld + c];
        A[j * ld + c] = A[p * ld + c];
        A[p * ld + c] = t;
      }
    __syncthreads();
    const double pv = A[j * ld + j];
    if (pv == 0.0) {
      if (tid == 0) zero_pivot = 1;
      continue;
    }
    const bool recip = fabs(pv) >= 2.2250738585072014e-308;
    const double rp = 1.0 / pv;
    for (int i = j + 1 + tid; i < n; i += nt) A[i * ld + j] = recip ? A[i * ld + j] * rp : A[i * ld + j] / pv;
    __syncthreads();
    const int w = n - j - 1;
    for (int e = tid; e < w * w; e += nt) {
      const int i = j + 1 + e / w, c = j + 1 + e % w;
      A[i * ld + c] -= A[i * ld + j] * A[j * ld + c];
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += nt) A_g[int64_t(e / n) * lda + e % n] = A[(e / n) * ld + e % n];
  // B <- P B, then L and U solves (dgetrs)
  for (int64_t c = tid; c < nrhs; c += nt)
    for (int j = 0; j < n; ++j) {
      const int p = piv_g[j];
      if (p != j) {
        const double t = B[int64_t(j) * ldb + c];
        B[int64_t(j) * ldb + c] = B[int64_t(p) * ldb + c];
        B[int64_t(p) * ldb + c] = t;
      }
    }
  __syncthreads();
  tri_solve(A, n, ld, B, nrhs, ldb, 0);
  tri_solve(A, n, ld, B, nrhs, ldb, 1);
  if (!with_rcond) return;   // the caller runs gecon on the factors (e.g. on a side stream)
  // dgecon (norm '1') on the factors
  const double anorm = *anorm_out;
  if (!(anorm > 0.0)) { if (tid == 0) *rcond_out = (anorm == 0.0) ? 0.0 : anorm; return; }
  if (tid == 0) flag = 0;
  __syncthreads();
  for (int i = tid; i < n; i += nt)
    if (A[i * ld + i] == 0.0) flag = 1;
  __syncthreads();
  if (flag || zero_pivot) { if (tid == 0) *rcond_out = 0.0; return; }
  auto inv = [&]() { tri_solve(A, n, ld, x, 1, 1, 0); tri_solve(A, n, ld, x, 1, 1, 1); };
  auto inv_t = [&]() { tri_solve(A, n, ld, x, 1, 1, 2); tri_solve(A, n, ld, x, 1, 1, 3); };
  const double est = dlacn2_est(n, x, isgn, inv, inv_t, red, sh, &flag);
  if (tid == 0) *rcond_out = est != 0.0 ? (1.0 / est) / anorm : 0.0;
}

// n <= 160 without the condition estimate (the seed systems of c1 / c2-sized
// problems; gecon runs on a side stream): column-owner threads.  Thread c
// owns column c of the augmented matrix [A | B] in shared memory (ld odd:
// conflict-free) and a column step needs ONE CTA barrier.  A panel warp that
// owns no column runs one column ahead: in iteration j it applies step j to
// column j + 1 (lanes over the rows, in registers), finds that column's pivot
// (dgetf2's idamax: NaN largest, ties to the lowest row), scales it and
// publishes pivot and multipliers in a double-buffered broadcast array --
// while every column thread swaps and updates its own column for step j.
// The right-hand sides ride as columns c >= n (so L y = P b is done when
// the factorization is), then one warp per right-hand side back-substitutes
// column-wise with its column in registers.  Element for element the same
// operations as small_dense_kernel's factorization (identical factors and
// pivots).
constexpr int COL_N = 160;
constexpr int COL_COLS = 256;
constexpr size_t COL_SMEM_MAX = 220 * 1024;

// RPL: rows per lane of the pivot search / back-substitution (n <= 32 RPL)
template <int RPL>
__global__ void __launch_bounds__(COL_COLS + 32)
small_dense_col_kernel(double* __restrict__ A_g, int n, int64_t lda, int32_t* __restrict__ piv_g,
                       double* __restrict__ B, int nrhs, int64_t ldb, double* __restrict__ anorm_out) {
  extern __shared__ double sm[];
  __shared__ ArgMax sh[32];
  __shared__ double lbuf[2][COL_N + 8];
  __shared__ int pbuf[2], skipbuf[2];
  const int nc = n + nrhs;
  const int ld = nc | 1;
  double* Aug = sm;              // (n + 8) x ld: 8 pad rows so the 8-row update batches need no bounds checks
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  // [A | B] -> shared memory, four independent global loads in flight per thread
  for (int e0 = tid; e0 < n * nc; e0 += 4 * nt) {
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = e0 + k * nt, i = e / nc, c = e - i * nc;
      v[k] = e < n * nc ? (c < n ? A_g[int64_t(i) * lda + c] : B[int64_t(i) * ldb + (c - n)]) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = e0 + k * nt, i = e / nc, c = e - i * nc;
      if (e < n * nc) Aug[i * ld + c] = v[k];
    }
  }
  for (int e = tid; e < 8 * ld; e += nt) Aug[n * ld + e] = 0.0;   // pad rows
  if (tid < 2 * (COL_N + 8)) (&lbuf[0][0])[tid] = 0.0;
  __syncthreads();
  // 1-norm of A (max column sum), summed in row order as small_dense_kernel
  {
    double cmax = 0.0;
    if (tid < n) {
      double c = 0.0;
      const double* col = Aug + tid;
      for (int i0 = 0; i0 < n; i0 += 8, col += 8 * ld) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = fabs(col[k * ld]);   // pad rows are zero
#pragma unroll
        for (int k = 0; k < 8; ++k) c += v[k];
      }
      cmax = (c > cmax || c != c) ? c : cmax;
    }
    const double anorm = block_argmax(ArgMax{cmax, tid}, sh).v;
    if (tid == 0) *anorm_out = anorm;
  }
  // The last warp is the panel warp: it owns no column.  In iteration j it
  // applies step j to column j + 1 (lanes over the rows), finds that column's
  // pivot in registers and publishes step j + 1 -- while the column threads
  // apply step j to every other column, so the pivot chain hides behind the
  // trailing update.
  const bool panel = warp == nw - 1;
  auto panel_step = [&](int j) {   // j = -1: the first column, nothing to apply
    const int jn = j + 1, bn = jn & 1;
    double v[RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int i = jn + lane + 32 * k;
      v[k] = i < n ? Aug[i * ld + jn] : 0.0;
    }
    if (j >= 0) {
      const int b = j & 1;
      const int p = pbuf[b];
      const double a_j = Aug[j * ld + jn];
      double ajc = a_j;
      if (p != j) {                  // rows j / p swap: row p (>= jn, in registers) takes a_j
        ajc = Aug[p * ld + jn];
#pragma unroll
        for (int k = 0; k < RPL; ++k)
          if (jn + lane + 32 * k == p) v[k] = a_j;
        if (lane == 0) Aug[j * ld + jn] = ajc;
      }
      if (!skipbuf[b]) {
        const double* l = lbuf[b];
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
          const int i = jn + lane + 32 * k;
          if (i < n) v[k] -= l[i] * ajc;
        }
      }
    }
    ArgMax a{-1.0, 0x7fffffff};
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int i = jn + lane + 32 * k;
      if (i < n) {
        const double f = fabs(v[k]);
        a = argmax_merge(a, ArgMax{f != f ? __longlong_as_double(0x7ff0000000000000LL) : f, i});
      }
    }
    // |v| >= 0 (or +inf): its bit pattern orders like the value, so the warp
    // argmax is three integer redux ops (high word, low word, lowest row
    // among the ties); lanes without a row carry (0, INT_MAX) and lose every tie
    const unsigned long long bits = a.i == 0x7fffffff ? 0ull : static_cast<unsigned long long>(__double_as_longlong(a.v));
    const unsigned hi = static_cast<unsigned>(bits >> 32), lo = static_cast<unsigned>(bits);
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    bool cand = hi == mhi;
    const unsigned mlo = __reduce_max_sync(0xffffffffu, cand ? lo : 0u);
    cand = cand && lo == mlo;
    const int p2 = static_cast<int>(__reduce_min_sync(0xffffffffu, cand ? static_cast<unsigned>(a.i) : 0x7fffffffu));
    const int ks = (p2 - jn) >> 5;
    double vs = v[0];
#pragma unroll
    for (int k = 1; k < RPL; ++k) vs = k == ks ? v[k] : vs;
    const double pv = __shfl_sync(0xffffffffu, vs, (p2 - jn) & 31);
    const double aj = __shfl_sync(0xffffffffu, v[0], 0);
    if (lane == 0) {
      pbuf[bn] = p2;
      skipbuf[bn] = pv == 0.0;
      piv_g[jn] = p2;
    }
    const bool recip = fabs(pv) >= 2.2250738585072014e-308;
    const double rp = __drcp_rn(pv);              // == 1.0 / pv (both correctly rounded)
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int i = jn + lane + 32 * k;
      if (i < n) {
        double x = i == p2 ? aj : v[k];
        if (i == jn) {
          x = pv;
        } else if (pv != 0.0) {                   // a zero pivot leaves its column unscaled (dgetf2)
          x = recip ? x * rp : x / pv;
          lbuf[bn][i] = x;
        }
        Aug[i * ld + jn] = x;
      }
    }
  };
  if (panel) panel_step(-1);
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const int b = j & 1;
    if (panel) {
      if (j + 1 < n) panel_step(j);
    } else if (tid < nc && tid != j && tid != j + 1) {
      const int p = pbuf[b];
      double ajc = Aug[j * ld + tid];
      if (p != j) {
        const double t = Aug[p * ld + tid];
        Aug[p * ld + tid] = ajc;
        Aug[j * ld + tid] = t;
        ajc = t;
      }
      if (tid > j && !skipbuf[b]) {
        // batches of 8 rows in registers: loads, then FMAs, then stores (a
        // plain loop serialises on the shared-memory store -> load order);
        // the last batch runs into the pad rows
        const double* l = lbuf[b] + j + 1;
        double* col = Aug + (j + 1) * ld + tid;
        for (int rem = n - j - 1; rem > 0; rem -= 8, col += 8 * ld, l += 8) {
          double v[8], m[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            v[k] = col[k * ld];
            m[k] = l[k];
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] -= m[k] * ajc;
#pragma unroll
          for (int k = 0; k < 8; ++k) col[k * ld] = v[k];
        }
      }
    }
    __syncthreads();
  }
  for (int i = warp; i < n; i += nw)
    for (int c = lane; c < n; c += 32) A_g[int64_t(i) * lda + c] = Aug[i * ld + c];
  // U x = y, column-oriented: warp per right-hand side, the column in
  // registers (rows lane and lane + 32), x_j broadcast by shuffle
  for (int c = n + warp; c < nc; c += nw) {
    double y[RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) y[k] = lane + 32 * k < n ? Aug[(lane + 32 * k) * ld + c] : 0.0;
    for (int j = n - 1; j >= 0; --j) {
      double u[RPL];
#pragma unroll
      for (int k = 0; k < RPL; ++k) u[k] = lane + 32 * k < j ? Aug[(lane + 32 * k) * ld + j] : 0.0;
      const double ujj = Aug[j * ld + j];
      const int jk = j >> 5;
      double ys = y[0];
#pragma unroll
      for (int k = 1; k < RPL; ++k) ys = k == jk ? y[k] : ys;
      const double x = __shfl_sync(0xffffffffu, ys, j & 31) / ujj;
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        if (k == jk && lane == (j & 31)) y[k] = x;
        if (lane + 32 * k < j) y[k] -= u[k] * x;
      }
    }
#pragma unroll
    for (int k = 0; k < RPL; ++k)
      if (lane + 32 * k < n) B[int64_t(lane + 32 * k) * ldb + (c - n)] = y[k];
  }
}

extern "C" int swb_small_dense_solve(double* A, int64_t n, int64_t lda, int32_t* piv, double* B, int64_t nrhs,
                                     int64_t ldb, double* anorm_out, double* rcond_out, void* stream) {
  if (n <= 0 || n > SMALL_N || !A || !piv || !B || !anorm_out || lda < n || nrhs < 0 || (nrhs > 0 && ldb < nrhs))
    return SWB_INVALID_PARAM;
  // SWB_SMALL_COL=0 (measurement knob): always the row-parallel kernel
  static const bool col_env = [] { const char* e = getenv("SWB_SMALL_COL"); return !(e && e[0] == '0'); }();
  const size_t smem_c = sizeof(double) * size_t(n + 8) * size_t((n + nrhs) | 1);
  if (col_env && !rcond_out && n <= COL_N && n + nrhs <= COL_COLS && smem_c <= COL_SMEM_MAX) {
    const int nc = static_cast<int>(n + nrhs);
    static unsigned long long attr_c = 0;
    if (swb_first_on_device(&attr_c)) {
      SWB_CUDA_TRY(cudaFuncSetAttribute(small_dense_col_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(COL_SMEM_MAX)));
      SWB_CUDA_TRY(cudaFuncSetAttribute(small_dense_col_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(COL_SMEM_MAX)));
    }
    const unsigned threads = static_cast<unsigned>(std::max(128, (nc + 31) / 32 * 32)) + 32;   // column warps (>= 4 for the loads / stores) + the panel warp
    if (n <= 64)
      small_dense_col_kernel<2><<<1, threads, smem_c, swb_stream(stream)>>>(A, static_cast<int>(n), lda, piv, B,
                                                                            static_cast<int>(nrhs), ldb, anorm_out);
    else
      small_dense_col_kernel<5><<<1, threads, smem_c, swb_stream(stream)>>>(A, static_cast<int>(n), lda, piv, B,
                                                                            static_cast<int>(nrhs), ldb, anorm_out);
    SWB_CHECK_LAUNCH();
    return SWB_OK;
  }
  const size_t smem = sizeof(double) * (size_t(n) * size_t(n | 1) + n) + sizeof(int32_t) * n;
  static unsigned long long attr = 0;
  if (swb_first_on_device(&attr)) {
    const size_t most = sizeof(double) * (size_t(SMALL_N) * size_t(SMALL_N | 1) + SMALL_N) + sizeof(int32_t) * SMALL_N;
    SWB_CUDA_TRY(cudaFuncSetAttribute(small_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(most)));
  }
  // fewer warps for the smaller systems: every column step is a few CTA barriers
  const unsigned threads = n <= 64 ? 128 : (n <= 128 ? 256 : SMALL_THREADS);
  small_dense_kernel<<<1, threads, smem, swb_stream(stream)>>>(A, n, lda, piv, B, nrhs, ldb, anorm_out, rcond_out,
                                                               rcond_out ? 1 : 0);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_lu_factor(double* A, int64_t n, int64_t lda, int32_t* piv, double* anorm_out, void* ws,
                             size_t ws_bytes, void* stream) {
  if (n < 0 || (n > 0 && (!A || !piv || lda < n || (lda & 1)))) return SWB_INVALID_PARAM;
  if (n > 0x7fffffff) return SWB_INVALID_PARAM;
  if (!ws || ws_bytes < swb_lu_workspace_bytes(n)) return SWB_WORKSPACE_TOO_SMALL;
  cudaStream_t st = swb_stream(stream);
  double* cs = static_cast<double*>(ws);
  int32_t* zp = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + swb_align_up(sizeof(double) * size_t(n + 1), 256));
  SWB_CUDA_TRY(cudaMemsetAsync(zp, 0, sizeof(int32_t), st));
  if (n == 0) {
    if (anorm_out) SWB_CUDA_TRY(cudaMemsetAsync(anorm_out, 0, sizeof(double), st));
    return SWB_OK;
  }
  if (anorm_out) {
    colabs_kernel<<<static_cast<unsigned>((n + 31) / 32), 256, 0, st>>>(A, n, lda, cs);
    SWB_CHECK_LAUNCH();
    max_kernel<<<1, 1024, 0, st>>>(cs, n, anorm_out);
    SWB_CHECK_LAUNCH();
  }
  static unsigned long long attr = 0;
  const int smem = PANEL_SMEM_ROWS * PANEL_LD * sizeof(double);
  if (swb_first_on_device(&attr)) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  // systems up to 1024 rows: 16-wide panels held in registers (one row per
  // thread); larger ones: 32-wide panels in shared memory
  const bool reg_panel = n <= 1024;
  const int nb = reg_panel ? RW : NB;
  const unsigned reg_threads = static_cast<unsigned>((n + 31) / 32 * 32);
  for (int64_t k = 0; k < n; k += nb) {
    const int w = static_cast<int>(std::min<int64_t>(nb, n - k));
    if (reg_panel)
      panel_reg_kernel<<<1, reg_threads, 0, st>>>(A, n, lda, k, w, piv, zp);
    else
      panel_kernel<<<1, PANEL_THREADS, smem, st>>>(A, n, lda, k, w, piv, zp);
    SWB_CHECK_LAUNCH();
    const int64_t others = n - w;
    if (others > 0) {
      swap_kernel<<<static_cast<unsigned>((others + 255) / 256), 256, 0, st>>>(A, n, lda, k, w, piv);
      SWB_CHECK_LAUNCH();
    }
    const int64_t rest = n - k - w;
    if (rest > 0) {
      trsm_kernel<<<static_cast<unsigned>((rest + 127) / 128), 128, 0, st>>>(A, n, lda, k, w);
      SWB_CHECK_LAUNCH();
      int rc = swb_gemm_nn_alpha(A + (k + w) * lda + k, lda, A + k * lda + k + w, lda, rest, w, rest,
                                 A + (k + w) * lda + k + w, lda, 1, -1.0, st);
      if (rc) return rc;
    }
  }
  return SWB_OK;
}

extern "C" int swb_lu_rcond(const double* LU, int64_t n, int64_t lda, const int32_t* piv, const double* anorm,
                            double* rcond_out, void* ws, size_t ws_bytes, void* stream) {
  (void)piv;  // ||A^-1||_1 == ||U^-1 L^-1||_1: the row permutation does not change column sums
  if (n < 0 || !anorm || !rcond_out || (n > 0 && (!LU || lda < n))) return SWB_INVALID_PARAM;
  if (!ws || ws_bytes < swb_lu_workspace_bytes(n)) return SWB_WORKSPACE_TOO_SMALL;
  cudaStream_t st = swb_stream(stream);
  char* base = static_cast<char*>(ws) + swb_align_up(sizeof(double) * size_t(n + 1), 256) + 256;
  double* x = reinterpret_cast<double*>(base);
  int32_t* isgn = reinterpret_cast<int32_t*>(base + swb_align_up(sizeof(double) * size_t(n + 1), 256));
  gecon_kernel<<<1, 1024, 0, st>>>(LU, n, lda, anorm, x, isgn, rcond_out);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" size_t swb_lu_solve_workspace_bytes(int64_t n, int64_t nrhs) {
  return swb_align_up(sizeof(int32_t) * size_t(n + 1), 256) + sizeof(double) * size_t(n) * size_t(nrhs > 0 ? nrhs : 1);
}

extern "C" int swb_lu_solve(const double* LU, int64_t n, int64_t lda, const int32_t* piv, double* B,
                            int64_t nrhs, int64_t ldb, void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || nrhs < 0 || (n > 0 && (!LU || !piv || !B || lda < n || ldb < nrhs))) return SWB_INVALID_PARAM;
  if (n == 0 || nrhs == 0) return SWB_OK;
  if (!workspace || workspace_bytes < swb_lu_solve_workspace_bytes(n, nrhs)) return SWB_WORKSPACE_TOO_SMALL;
  int32_t* perm = static_cast<int32_t*>(workspace);
  double* tmp = reinterpret_cast<double*>(static_cast<char*>(workspace) +
                                          swb_align_up(sizeof(int32_t) * size_t(n + 1), 256));
  const size_t smem = n <= GETRS_SMEM_N ? sizeof(int32_t) * 2 * size_t(n) : 0;
  static unsigned long long attr = 0;   // set once per device to the largest size getrs can ask for
  if (smem > 48 * 1024 && swb_first_on_device(&attr)) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(getrs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(sizeof(int32_t) * 2 * size_t(GETRS_SMEM_N))));
  }
  getrs_kernel<<<1, 1024, smem, swb_stream(stream)>>>(LU, n, lda, piv, B, nrhs, ldb, perm, tmp);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_check_rcond(double rcond) {
  // fastrw.py:340: not finite or < 1e-14 -> SingularSmallSystem
  if (!(rcond == rcond) || rcond == __builtin_inf() || rcond < 1e-14) return SWB_SINGULAR_SMALL_SYSTEM;
  return SWB_OK;
}

extern "C" size_t swb_gecon_wb_workspace_bytes(int64_t n, int64_t r) {
  return swb_align_up(sizeof(double) * size_t(n + 1), 256) + swb_align_up(sizeof(double) * size_t(r + 1), 256) +
         swb_align_up(sizeof(int32_t) * size_t(n + 1), 256);
}

extern "C" int swb_gecon_wb(int64_t n, int64_t r, const double* Ut, const double* Vt, int64_t ldr, const double* K,
                            int64_t ldk, const int32_t* pk, const double* anorm, double* rcond_out, void* ws,
                            size_t ws_bytes, void* stream) {
  if (n < 0 || r <= 0 || !Ut || !Vt || !K || !pk || !anorm || !rcond_out || ldr < r || ldk < r) return SWB_INVALID_PARAM;
  if (!ws || ws_bytes < swb_gecon_wb_workspace_bytes(n, r)) return SWB_WORKSPACE_TOO_SMALL;
  char* base = static_cast<char*>(ws);
  double* x = reinterpret_cast<double*>(base);
  double* t = reinterpret_cast<double*>(base + swb_align_up(sizeof(double) * size_t(n + 1), 256));
  int32_t* isgn = reinterpret_cast<int32_t*>(base + swb_align_up(sizeof(double) * size_t(n + 1), 256) +
                                             swb_align_up(sizeof(double) * size_t(r + 1), 256));
  gecon_wb_kernel<<<1, 1024, 0, swb_stream(stream)>>>(n, r, Ut, Vt, ldr, K, ldk, pk, anorm, x, t, isgn, rcond_out);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_norm1(const double* A, int64_t n, int64_t lda, double* out, void* ws, size_t ws_bytes,
                         void* stream) {
  // ||A||_1 (max column sum of |A|, NaN-propagating like np.linalg.norm)
  if (n < 0 || !out || (n > 0 && (!A || lda < n))) return SWB_INVALID_PARAM;
  if (!ws || ws_bytes < sizeof(double) * size_t(n + 1)) return SWB_WORKSPACE_TOO_SMALL;
  cudaStream_t st = swb_stream(stream);
  if (n == 0) { SWB_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double), st)); return SWB_OK; }
  double* cs = static_cast<double*>(ws);
  colabs_kernel<<<static_cast<unsigned>((n + 31) / 32), 256, 0, st>>>(A, n, lda, cs);
  SWB_CHECK_LAUNCH();
  max_kernel<<<1, 1024, 0, st>>>(cs, n, out);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}
