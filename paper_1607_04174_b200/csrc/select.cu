// Dynamic basis size (reference adaptive.py:72-185) on the device.
//
// seed_fit(q_s[:, :m], u_k, bound) for every scheduled m and label k:
//   1. one Householder QR of the full seed block q_s = Q R (S x M), with Q^T
//      applied to the label columns U = onehot * d_sqrt[s] -> C = Q^T U.
//      For every prefix m, q_s[:, :m] = Q[:, :m] R[:m, :m], so its singular
//      values / left-projections are those of the small R_m and
//      b = U_q^T u = U_R^T c[:m]  (adaptive.py:82-83).
//   2. per scheduled m (one CTA each, all steps in parallel): one-sided
//      (Hestenes) Jacobi SVD of R_m in shared memory, sigma descending, the
//      reference's cutoff 1e-13 * sigma_0 (adaptive.py:85), perp, and the
//      ridge bisection on mu (<= 200 steps, tol 1e-6 * bound, :96-110).
#include <cooperative_groups.h>

#include <cstdlib>

#include "swb_common.cuh"

namespace cg = cooperative_groups;

namespace {

__device__ double block_reduce_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

// At: M x S (row j = column j of q_s), Ut: K x S (row k = label column).
// In place: At[j][i] = R_ij for i <= j (Householder vectors below), Ut = Q^T U.
__global__ void __launch_bounds__(1024) householder_kernel(double* __restrict__ At, int64_t S, int64_t M,
                                                           double* __restrict__ Ut, int64_t K) {
  __shared__ double red[32];
  __shared__ double sh_tau, sh_beta, sh_scale;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t r = S < M ? S : M;
  for (int64_t j = 0; j < r; ++j) {
    double* x = At + j * S;
    double s = 0.0;
    for (int64_t i = j + 1 + threadIdx.x; i < S; i += blockDim.x) s += x[i] * x[i];
    const double sigma = block_reduce_sum(s, red);
    if (threadIdx.x == 0) {
      const double alpha = x[j];
      // LAPACK dlarfg: H = I - tau v v^T, v[0] = 1, H x = beta e_1
      if (sigma == 0.0) {
        sh_tau = 0.0; sh_beta = alpha; sh_scale = 0.0;
      } else {
        const double nrm = sqrt(alpha * alpha + sigma);
        const double beta = alpha >= 0.0 ? -nrm : nrm;
        sh_tau = (beta - alpha) / beta;
        sh_scale = 1.0 / (alpha - beta);
        sh_beta = beta;
      }
    }
    __syncthreads();
    const double tau = sh_tau, scale = sh_scale;
    for (int64_t i = j + 1 + threadIdx.x; i < S; i += blockDim.x) x[i] *= scale;
    __syncthreads();
    if (threadIdx.x == 0) x[j] = sh_beta;
    if (tau != 0.0) {
      // apply H to the remaining columns of q_s and to the label columns
      const int64_t nvec = (M - j - 1) + K;
      for (int64_t t = warp; t < nvec; t += nw) {
        double* y = t < M - j - 1 ? At + (j + 1 + t) * S : Ut + (t - (M - j - 1)) * S;
        double w = lane == 0 ? y[j] : 0.0;
        for (int64_t i = j + 1 + lane; i < S; i += 32) w += x[i] * y[i];
        w = warp_sum(w) * tau;
        if (lane == 0) y[j] -= w;
        for (int64_t i = j + 1 + lane; i < S; i += 32) y[i] -= w * x[i];
      }
    }
    __syncthreads();
  }
}

// The same QR with the trailing columns spread over the whole GPU: one
// cooperative launch, every CTA owns columns c = blockIdx.x + k * gridDim.x
// of [q_s | U] (M + K columns).  Step j: each CTA forms reflector j from
// column j itself (the same fixed-order block reduction everywhere, so every
// CTA holds bit-identical tau / beta / v, staged in shared memory), applies
// it to its own columns c > j, and a grid barrier closes the step; the owner
// of column j writes v / beta back after the barrier (nobody reads column j
// again).  The single-CTA kernel above spends ~16 us a column on its 32
// warps walking ~150 columns in turn (S = 1000: 2.4 ms); here a step is two
// block reductions and one grid barrier.
constexpr int HH_THREADS = 256;

__device__ __forceinline__ double block_sum_256(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < HH_THREADS / 32; ++w) s += red[w];   // same order in every thread
  __syncthreads();
  return s;
}

__global__ void __launch_bounds__(HH_THREADS) householder_coop_kernel(double* __restrict__ At, int64_t S, int64_t M,
                                                                      double* __restrict__ Ut, int64_t K) {
  extern __shared__ double hv[];   // v = [1; x[j+1:] * scale] of the current step (S doubles)
  __shared__ double red[HH_THREADS / 32];
  cg::grid_group grid = cg::this_grid();
  const int64_t r = S < M ? S : M;
  const int64_t nc = M + K;
  auto col = [&](int64_t c) { return c < M ? At + c * S : Ut + (c - M) * S; };
  for (int64_t j = 0; j < r; ++j) {
    const double* x = At + j * S;
    double s = 0.0;
    for (int64_t i = j + 1 + threadIdx.x; i < S; i += HH_THREADS) {
      const double xi = __ldcg(x + i);
      hv[i] = xi;
      s = fma(xi, xi, s);
    }
    const double sigma = block_sum_256(s, red);
    const double alpha = __ldcg(x + j);
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (sigma != 0.0) {   // LAPACK dlarfg: H = I - tau v v^T, v[0] = 1, H x = beta e_1
      const double nrm = sqrt(alpha * alpha + sigma);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    for (int64_t i = j + 1 + threadIdx.x; i < S; i += HH_THREADS) hv[i] *= scale;   // own entries: no sync needed
    __syncthreads();
    if (tau != 0.0) {
      for (int64_t c = blockIdx.x; c < nc; c += gridDim.x) {
        if (c <= j) continue;
        double* y = col(c);
        double w = threadIdx.x == 0 ? y[j] : 0.0;
        for (int64_t i = j + 1 + threadIdx.x; i < S; i += HH_THREADS) w = fma(hv[i], y[i], w);
        w = block_sum_256(w, red) * tau;
        if (threadIdx.x == 0) y[j] -= w;
        for (int64_t i = j + 1 + threadIdx.x; i < S; i += HH_THREADS) y[i] = fma(-w, hv[i], y[i]);
      }
    }
    grid.sync();
    if (j % gridDim.x == blockIdx.x) {   // owner of column j: v and beta in place
      double* xo = At + j * S;
      for (int64_t i = j + 1 + threadIdx.x; i < S; i += HH_THREADS) xo[i] = hv[i];
      if (threadIdx.x == 0) xo[j] = beta;
    }
    __syncthreads();   // hv is rewritten by the next step
  }
}

// Round-robin tournament: round rd, slot p of n (even) players
__device__ __forceinline__ void rr_pair(int rd, int p, int n, int& a, int& b) {
  // player 0 fixed, others rotate
  auto pos = [&](int k) { return k == 0 ? 0 : 1 + ((k - 1 + rd) % (n - 1)); };
  a = pos(p);
  b = pos(n - 1 - p);
}

__device__ __forceinline__ double lds64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// One-sided (Hestenes) Jacobi sweeps over the n columns (length r) of W,
// until a sweep rotates nothing.  SMEM: W lives in shared memory (explicit
// ld/st.shared: the generic pointer would compile to generic LD/ST).
template <bool SMEM>
__device__ __forceinline__ void jacobi_sweeps(double* W, int64_t r, int n, int* rotated) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // one-sided Jacobi sweeps.  Each pair of a round-robin round goes to an
  // 8-lane group (4 pairs per warp at once, 64 pair slots per 512-thread
  // CTA): its two columns are read from shared memory once into registers
  // (r <= 8 * JR), the three dot products reduce over 3 shuffle levels and
  // the rotation is applied from registers, so a pair costs one read and one
  // write of its columns -- the sweep is bound by shared-memory bandwidth
  // (6 -> 4 column accesses per pair) and by the sqrt / div chain, which
  // four pairs per warp share.
  constexpr int JG = 8, JR = 20;
  const int grp = lane / JG, gl = lane % JG;
  const int slot = warp * (32 / JG) + grp, nslots = nw * (32 / JG);
  const int npairs = n / 2;
  const int passes = (npairs + nslots - 1) / nslots;
  const bool regs = r <= int64_t(JG) * JR;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) *rotated = 0;
    __syncthreads();
    for (int rd = 0; rd < n - 1; ++rd) {
      for (int ps = 0; ps < passes; ++ps) {
        const int p = slot + ps * nslots;
        const bool live = p < npairs;
        int a = 0, b = 1;
        if (live) {
          rr_pair(rd, p, n, a, b);
          if (a > b) { const int t = a; a = b; b = t; }
        }
        double* wa = W + int64_t(a) * r;
        double* wb = W + int64_t(b) * r;
        const uint32_t sa = SMEM ? static_cast<uint32_t>(__cvta_generic_to_shared(wa)) : 0u;
        const uint32_t sb = SMEM ? static_cast<uint32_t>(__cvta_generic_to_shared(wb)) : 0u;
        auto lda = [&](int64_t i) { return SMEM ? lds64(sa + 8u * uint32_t(i)) : wa[i]; };
        auto ldb = [&](int64_t i) { return SMEM ? lds64(sb + 8u * uint32_t(i)) : wb[i]; };
        auto sta = [&](int64_t i, double v) { if (SMEM) sts64(sa + 8u * uint32_t(i), v); else wa[i] = v; };
        auto stb = [&](int64_t i, double v) { if (SMEM) sts64(sb + 8u * uint32_t(i), v); else wb[i] = v; };
        double xa[JR], yb[JR];
        double al = 0.0, be = 0.0, ga = 0.0;
        if (live) {
          if (regs) {
#pragma unroll
            for (int q = 0; q < JR; ++q) {
              const int64_t i = gl + q * JG;
              xa[q] = i < r ? lda(i) : 0.0;
              yb[q] = i < r ? ldb(i) : 0.0;
              al = fma(xa[q], xa[q], al); be = fma(yb[q], yb[q], be); ga = fma(xa[q], yb[q], ga);
            }
          } else {
            for (int64_t i = gl; i < r; i += JG) {
              const double x = lda(i), y = ldb(i);
              al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
            }
          }
        }
#pragma unroll
        for (int o = JG / 2; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (live && ga != 0.0 && ga * ga > 1e-30 * (al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          if (regs) {
#pragma unroll
            for (int q = 0; q < JR; ++q) {
              const int64_t i = gl + q * JG;
              if (i < r) {
                sta(i, c * xa[q] - s * yb[q]);
                stb(i, s * xa[q] + c * yb[q]);
              }
            }
          } else {
            for (int64_t i = gl; i < r; i += JG) {
              const double x = lda(i), y = ldb(i);
              sta(i, c * x - s * y);
              stb(i, s * x + c * y);
            }
          }
          if (gl == 0) *rotated = 1;
        }
      }
      __syncthreads();
    }
    const int any = *rotated;
    __syncthreads();
    if (!any) break;
  }
}

// ---------------------------------------------------------------------------
// Fast path of seed_fit for a square, well-conditioned R_m (S >= m): the
// reference only needs, per label, the singular values sigma_j of q_s and
// the projections b = U^T u (adaptive.py:82-110), and every quantity it forms
// from them is orthogonally invariant:
//   perp  = |u|^2 - |b|^2 = |u|^2 - |w|^2          (w = Q^T u, first m entries)
//   a2(mu) = sum_j (sigma_j b_j / (sigma_j^2 + mu))^2 = |y(mu)|^2,
//   resid(mu) = sum_j (b_j - sigma_j z_j)^2 = |g - B y(mu)|^2,
// with R_m = U_B B V_B^T (Golub-Kahan, B upper bidiagonal), g = U_B^T w and
// y(mu) = argmin |B y - g|^2 + mu |y|^2 -- solved in O(m) per mu by Givens
// rotations of [B; sqrt(mu) I] (Elden's bidiagonal ridge), not by forming
// B^T B.  sigma_0 (the bisection's starting bracket, adaptive.py:101) and
// sigma_min come from Sturm-sequence multisection on B^T B.  The path is
// taken when sigma_min > 1e-6 sigma_0: then no singular value is below the
// reference cutoff 1e-13 sigma_0 (all kept, as in the reference) and the
// ridge solve is accurate to ~kappa * eps.  Otherwise the Jacobi SVD below
// runs.  One bidiagonalisation per scheduled m replaces ~12 Jacobi sweeps.
// ---------------------------------------------------------------------------

// number of eigenvalues of the symmetric tridiagonal T (diag t, off o) < x
__device__ int sturm_count(const double* t, const double* o2, int m, double x) {
  int cnt = 0;
  double q = t[0] - x;
  if (q < 0.0) ++cnt;
  for (int i = 1; i < m; ++i) {
    if (q == 0.0) q = -1e-300;
    q = (t[i] - x) - o2[i - 1] / q;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}

// k-th smallest eigenvalue (0-based) of T by 32-way multisection (one warp)
__device__ double tridiag_eig(const double* t, const double* o2, int m, int k, double lo, double hi) {
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < 40 && hi - lo > 1e-17 * fmax(fabs(lo), fabs(hi)); ++it) {
    const double x = lo + (hi - lo) * (lane + 1) / 33.0;
    const int c = sturm_count(t, o2, m, x);
    // eigenvalue k lies below the first point whose count exceeds k
    const unsigned above = __ballot_sync(0xffffffffu, c > k);
    const int first = above ? __ffs(above) - 1 : 32;
    const double nlo = first == 0 ? lo : lo + (hi - lo) * first / 33.0;
    const double nhi = first == 32 ? hi : lo + (hi - lo) * (first + 1) / 33.0;
    lo = nlo;
    hi = nhi;
  }
  return 0.5 * (lo + hi);
}

// y(mu) = argmin |B y - g|^2 + mu |y|^2 (B: d[0..m), e[0..m-1) upper
// bidiagonal) by Givens rotations of [B; sqrt(mu) I]; returns |y|^2 and sets
// *resid = |g - B y|^2.  sc: per-lane scratch, element i at sc[i * ST]
// (y, then the rotated diagonal and super-diagonal at +m*ST, +2m*ST).
template <int ST>
__device__ double ridge_bidiag(const double* d, const double* e, const double* g, int m, double mu, double* sc,
                               double* resid) {
  double* y = sc;
  double* rd = sc + int64_t(m) * ST;
  double* re = sc + 2 * int64_t(m) * ST;
  const double smu = sqrt(mu);
  double cv = 0.0, ch = 0.0;           // carry row: value at column i, right-hand side
  for (int i = 0; i < m; ++i) {
    double x = d[i], xe = i + 1 < m ? e[i] : 0.0, xr = g[i];
    double v1 = 0.0, h1 = 0.0;
    if (smu > 0.0) {                    // eliminate the sqrt(mu) row of column i
      const double rr = hypot(x, smu), c = x / rr, s = smu / rr;
      v1 = -s * xe; h1 = -s * xr;
      x = rr; xe *= c; xr *= c;
    }
    double v2 = 0.0, h2 = 0.0;
    if (cv != 0.0) {                    // eliminate the carried row
      const double rr = hypot(x, cv), c = x / rr, s = cv / rr;
      v2 = -s * xe; h2 = -s * xr + c * ch;
      x = rr; xe *= c; xr = c * xr + s * ch;
    } else {
      h2 = ch;
    }
    rd[i * ST] = x; re[i * ST] = xe; y[i * ST] = xr;
    // merge the two rows whose only entry is now in column i+1
    const double rr = hypot(v1, v2);
    if (rr > 0.0) {
      const double c = v1 / rr, s = v2 / rr;
      cv = rr; ch = c * h1 + s * h2;
    } else {
      cv = 0.0; ch = 0.0;
    }
  }
  double a2 = 0.0, res = 0.0, ynext = 0.0;
  for (int i = m - 1; i >= 0; --i) {
    const double yi = (y[i * ST] - (i + 1 < m ? re[i * ST] * ynext : 0.0)) / rd[i * ST];
    a2 = fma(yi, yi, a2);
    const double rr = g[i] - (d[i] * yi + (i + 1 < m ? e[i] * ynext : 0.0));
    res = fma(rr, rr, res);
    ynext = yi;
  }
  *resid = res;
  return a2;
}

// seed_fit's bound search (adaptive.py:96-110) with one warp: the doubling of
// hi and the bisection follow the reference's exact sequence of points, but
// 31 lanes evaluate the next five bisection levels (a complete binary tree of
// candidate mids) at once and lane 0 walks the path the comparisons select,
// so the serial chain is ~7 ridge solves instead of ~70.
__device__ double warp_ridge_fit(const double* d, const double* e, const double* g, int m, double sg0, double ww,
                                 double perp, double bound, double* sc) {
  const int lane = threadIdx.x & 31;
  const double b2 = bound * bound;
  double res;
  // doubling: hi0 * 2^k, k = 32 q + lane
  double hi = sg0 * sqrt(ww) / bound, a2hi = 0.0, reshi = 0.0;
  for (int q = 0; q < 64; ++q) {
    double h = hi;
    for (int t = 0; t < lane; ++t) h *= 2.0;
    const double a = ridge_bidiag<32>(d, e, g, m, h, sc, &res);
    const unsigned ok = __ballot_sync(0xffffffffu, !(a > b2));
    if (ok) {
      const int k = __ffs(ok) - 1;
      hi = __shfl_sync(0xffffffffu, h, k);
      a2hi = __shfl_sync(0xffffffffu, a, k);
      reshi = __shfl_sync(0xffffffffu, res, k);
      break;
    }
    hi = __shfl_sync(0xffffffffu, h, 31) * 2.0;
  }
  double lo = 0.0;
  int it = 0;
  bool done = false;   // the reference tests convergence only after a bisection step
  while (!done && it < 200) {
    // node h = lane + 1 (heap order): its interval from the path bits below the leading one
    const int h = lane + 1;
    const int depth = 31 - __clz(h);
    double l = lo, u = hi;
    for (int bit = depth - 1; bit >= 0; --bit) {
      const double mid = 0.5 * (l + u);
      if ((h >> bit) & 1) l = mid; else u = mid;
    }
    const double mid = 0.5 * (l + u);
    double a = 0.0, rs = 0.0;
    if (lane < 31) a = ridge_bidiag<32>(d, e, g, m, mid, sc, &rs);
    // walk five levels along the comparisons (same decisions as the sequential loop)
    int node = 1;
    for (int lvl = 0; lvl < 5 && !done && it < 200; ++lvl) {
      const double am = __shfl_sync(0xffffffffu, a, node - 1);
      const double rm = __shfl_sync(0xffffffffu, rs, node - 1);
      const double mm = __shfl_sync(0xffffffffu, mid, node - 1);
      if (am > b2) {
        lo = mm;
        node = 2 * node + 1;
      } else {
        hi = mm; a2hi = am; reshi = rm;
        node = 2 * node;
      }
      ++it;
      if (fabs(sqrt(a2hi) - bound) <= 1e-6 * bound) done = true;
    }
  }
  return fmax(perp + reshi, 0.0);
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = lane < nw ? red[lane] : 0.0;
  return warp_sum(t);
}

// A: m x m column-major in shared memory (A[i + j*ld]), G: K label vectors
// (stride m).  Golub-Kahan: A -> B (d, e); G <- U_B^T G.  Returns with d, e
// filled (shared) and A overwritten.
__device__ void bidiagonalize(double* A, int ld, int m, double* G, int K, double* d, double* e, double* red,
                              double* hv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = 0; j < m; ++j) {
    // left reflector on column j, rows j..m-1
    double ss = 0.0;
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) ss = fma(A[i + j * ld], A[i + j * ld], ss);
    const double sig = block_sum(ss, red);
    const double alpha = A[j + j * ld];
    double beta = alpha, tau = 0.0, scale = 0.0;
    if (sig != 0.0) {
      const double nrm = sqrt(alpha * alpha + sig);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    __syncthreads();
    for (int i = j + threadIdx.x; i < m; i += blockDim.x) hv[i] = i == j ? 1.0 : A[i + j * ld] * scale;
    __syncthreads();
    if (threadIdx.x == 0) d[j] = beta;
    if (tau != 0.0) {
      const int ncol = (m - j - 1) + K;
      for (int t = warp; t < ncol; t += nw) {
        double* y = t < m - j - 1 ? A + (j + 1 + t) * ld : G + (t - (m - j - 1)) * m;
        double w = 0.0;
        for (int i = j + lane; i < m; i += 32) w = fma(hv[i], y[i], w);
        w = warp_sum(w) * tau;
        for (int i = j + lane; i < m; i += 32) y[i] = fma(-w, hv[i], y[i]);
      }
    }
    __syncthreads();
    if (j + 1 >= m) break;
    if (j + 2 >= m) {                   // last super-diagonal entry, no reflector
      if (threadIdx.x == 0) e[j] = A[j + (j + 1) * ld];
      __syncthreads();
      continue;
    }
    // right reflector on row j, columns j+1..m-1
    ss = 0.0;
    for (int c = j + 2 + threadIdx.x; c < m; c += blockDim.x) ss = fma(A[j + c * ld], A[j + c * ld], ss);
    const double sig2 = block_sum(ss, red);
    const double alpha2 = A[j + (j + 1) * ld];
    double beta2 = alpha2, tau2 = 0.0, scale2 = 0.0;
    if (sig2 != 0.0) {
      const double nrm = sqrt(alpha2 * alpha2 + sig2);
      beta2 = alpha2 >= 0.0 ? -nrm : nrm;
      tau2 = (beta2 - alpha2) / beta2;
      scale2 = 1.0 / (alpha2 - beta2);
    }
    __syncthreads();
    for (int c = j + 1 + threadIdx.x; c < m; c += blockDim.x) hv[c] = c == j + 1 ? 1.0 : A[j + c * ld] * scale2;
    __syncthreads();
    if (threadIdx.x == 0) e[j] = beta2;
    if (tau2 != 0.0) {
      for (int i = j + 1 + warp; i < m; i += nw) {   // rows j+1..m-1
        double w = 0.0;
        for (int c = j + 1 + lane; c < m; c += 32) w = fma(A[i + c * ld], hv[c], w);
        w = warp_sum(w) * tau2;
        for (int c = j + 1 + lane; c < m; c += 32) A[i + c * ld] = fma(-w, hv[c], A[i + c * ld]);
      }
    }
    __syncthreads();
  }
}

// One CTA per scheduled m.  W (m_pad x r) = R_m^T in shared or global
// scratch; sigma, b, f outputs per step.
__global__ void __launch_bounds__(512) jacobi_fit_kernel(const double* __restrict__ At, int64_t S, int64_t M,
                                                         const double* __restrict__ Ut, int64_t K,
                                                         const int32_t* __restrict__ steps,
                                                         const double* __restrict__ uu, double bound,
                                                         double* __restrict__ scratch, int64_t scratch_stride,
                                                         double* __restrict__ f_out, int allow_fast) {
  extern __shared__ double sm[];
  __shared__ int rotated;
  __shared__ double red[32];
  __shared__ int fast_ok;
  __shared__ double sig_hi;
  const int st = blockIdx.x;
  const int64_t m = steps[st];
  const int64_t r = (S < m ? S : m);  // rows of R_m
  const int n = static_cast<int>((m + 1) / 2 * 2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // ---- fast path: square R_m, bidiagonal ridge (see above) ----
  {
    const int ld = static_cast<int>(m) | 1;   // odd stride: conflict-free row access
    const size_t need = sizeof(double) * (size_t(ld) * m + size_t(K) * m + 5 * size_t(m) + 64);
    const bool try_fast = allow_fast && r == m && m >= 2 && K <= 16 && bound > 0.0 && need <= 200 * 1024;
    if (try_fast) {
      double* A = sm;
      double* G = A + size_t(ld) * m;
      double* d = G + size_t(K) * m;
      double* e = d + m;
      double* t = e + m;        // B^T B diagonal
      double* o2 = t + m;       // squared off-diagonal
      double* hv = o2 + m;
      for (int64_t q = threadIdx.x; q < m * m; q += blockDim.x) {
        const int64_t j = q / m, i = q % m;
        A[i + j * ld] = i <= j ? At[j * S + i] : 0.0;
      }
      for (int64_t q = threadIdx.x; q < int64_t(K) * m; q += blockDim.x) {
        const int64_t k = q / m, i = q % m;
        G[k * m + i] = Ut[k * S + i];
      }
      __syncthreads();
      bidiagonalize(A, ld, static_cast<int>(m), G, static_cast<int>(K), d, e, red, hv);
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        t[i] = d[i] * d[i] + (i > 0 ? e[i - 1] * e[i - 1] : 0.0);
        if (i + 1 < m) { const double od = d[i] * e[i]; o2[i] = od * od; }
      }
      __syncthreads();
      if (warp < 2) {
        // Gershgorin bracket of B^T B, then lambda_max (warp 0) / lambda_min (warp 1)
        double gh = 0.0;
        for (int i = 0; i < m; ++i) {
          const double rad = (i > 0 ? sqrt(o2[i - 1]) : 0.0) + (i + 1 < m ? sqrt(o2[i]) : 0.0);
          gh = fmax(gh, t[i] + rad);
        }
        const double lam = tridiag_eig(t, o2, static_cast<int>(m), warp == 0 ? static_cast<int>(m) - 1 : 0, 0.0,
                                       gh * (1.0 + 1e-12));
        if (lane == 0) {
          if (warp == 0) sig_hi = lam; else red[31] = lam;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) fast_ok = sig_hi > 0.0 && red[31] > 1e-12 * sig_hi;
      __syncthreads();
      if (fast_ok) {
        const double sg0 = sqrt(sig_hi);
        const int mm = static_cast<int>(m);
        for (int64_t k = warp; k < K; k += nw) {
          const double* g = G + k * m;
          double* sc = scratch + st * scratch_stride + (k * 3 * m) * 32 + lane;   // lane-interleaved
          double ww = 0.0;
          for (int i = 0; i < mm; ++i) ww = fma(g[i], g[i], ww);
          const double perp = uu[k] - ww;
          double res;
          const double a20 = ridge_bidiag<32>(d, e, g, mm, 0.0, sc, &res);
          const double f = a20 <= bound * bound ? fmax(perp, 0.0)
                                                : warp_ridge_fit(d, e, g, mm, sg0, ww, perp, bound, sc);
          if (lane == 0) f_out[int64_t(st) * K + k] = f;
        }
        return;
      }
      __syncthreads();
    }
  }
  const bool in_smem = size_t(n) * r * sizeof(double) + size_t(m) * 2 * sizeof(double) <= 200 * 1024;
  double* W = in_smem ? sm : scratch + st * scratch_stride;  // n x r, row j = column j of R_m
  double* nrm = in_smem ? sm + size_t(n) * r : scratch + st * scratch_stride + size_t(n) * r;
  for (int64_t e = threadIdx.x; e < int64_t(n) * r; e += blockDim.x) {
    const int64_t j = e / r, i = e % r;
    W[e] = (j < m && i <= j) ? At[j * S + i] : 0.0;
  }
  __syncthreads();
  if (in_smem)
    jacobi_sweeps<true>(W, r, n, &rotated);
  else
    jacobi_sweeps<false>(W, r, n, &rotated);
  // column norms = singular values
  for (int64_t j = warp; j < m; j += nw) {
    double s = 0.0;
    for (int64_t i = lane; i < r; i += 32) s += W[j * r + i] * W[j * r + i];
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(s);
  }
  __syncthreads();
  // rank of each column by sigma (descending, ties by index): top r are the thin SVD
  int* rank = reinterpret_cast<int*>(nrm + m);
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    int rk = 0;
    const double v = nrm[j];
    for (int64_t i = 0; i < m; ++i) rk += (nrm[i] > v) || (nrm[i] == v && i < j);
    rank[j] = rk;
  }
  __syncthreads();
  double smax = 0.0;
  for (int64_t j = 0; j < m; ++j) smax = fmax(smax, nrm[j]);
  const double cutoff = fmax(1e-13 * smax, 1e-300);
  // per label: b_j = w_j . c_k / sigma_j (top r columns), then the fit.
  // m <= 32 * FIT_REG: the b_j and sigma_j of the label live in the warp's
  // registers (lane l holds j = l, l + 32, ...), computed once, so each of
  // the up to 200 bisection steps is a register sum over the kept columns
  // instead of m dot products of length r.
  constexpr int FIT_REG = 16;
  if (m <= 32 * FIT_REG) {
    for (int64_t k = warp; k < K; k += nw) {
      const double* ck = Ut + k * S;
      const double u2 = uu[k];
      double f;
      if (bound <= 0.0) {
        f = u2;
      } else {
        double bj[FIT_REG], sg[FIT_REG];   // sg = 0: column not kept (below cutoff or outside the top r)
        double bb = 0.0, a20 = 0.0, bk2 = 0.0, sg0 = 0.0;
        int nkeep = 0;
#pragma unroll
        for (int q = 0; q < FIT_REG; ++q) { bj[q] = 0.0; sg[q] = 0.0; }
        for (int64_t j = 0; j < m; ++j) {
          if (rank[j] >= r) continue;
          const double sgj = nrm[j];
          double d = 0.0;
          for (int64_t i = lane; i < r; i += 32) d += W[j * r + i] * ck[i];
          d = warp_sum(d);
          const double b = sgj > 0.0 ? d / sgj : 0.0;
          bb += b * b;
          if (rank[j] == 0) sg0 = sgj;
          if (sgj > cutoff) {
            ++nkeep;
            bk2 += b * b;
            const double z = sgj * b / (sgj * sgj);
            a20 += z * z;
#pragma unroll
            for (int q = 0; q < FIT_REG; ++q)
              if (j == lane + 32 * q) { bj[q] = b; sg[q] = sgj; }
          }
        }
        const double perp = u2 - bb;
        if (nkeep == 0) {
          f = u2;
        } else if (a20 <= bound * bound) {
          f = fmax(perp, 0.0);
        } else {
          auto a2 = [&](double mu) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < FIT_REG; ++q) {
              const double z = sg[q] * bj[q] / (sg[q] * sg[q] + mu);
              acc += sg[q] > 0.0 ? z * z : 0.0;
            }
            return warp_sum(acc);
          };
          double lo = 0.0, hi = sg0 * sqrt(bk2) / bound;
          while (a2(hi) > bound * bound) hi *= 2.0;
          for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (a2(mid) > bound * bound) lo = mid; else hi = mid;
            if (fabs(sqrt(a2(hi)) - bound) <= 1e-6 * bound) break;
          }
          double res = 0.0;
#pragma unroll
          for (int q = 0; q < FIT_REG; ++q) {
            const double z = sg[q] * bj[q] / (sg[q] * sg[q] + hi);
            const double rr = bj[q] - sg[q] * z;
            res += sg[q] > 0.0 ? rr * rr : 0.0;
          }
          f = fmax(perp + warp_sum(res), 0.0);
        }
      }
      if (lane == 0) f_out[int64_t(st) * K + k] = f;
    }
    return;
  }
  for (int64_t k = warp; k < K; k += nw) {
    const double* ck = Ut + k * S;
    const double u2 = uu[k];
    double f;
    if (bound <= 0.0) {
      f = u2;
    } else {
      // pass 1: perp and a2(0), ||b_kept||
      double bb = 0.0, a20 = 0.0, bk2 = 0.0;
      int nkeep = 0;
      for (int64_t j = 0; j < m; ++j) {
        if (rank[j] >= r) continue;
        const double sg = nrm[j];
        double d = 0.0;
        for (int64_t i = lane; i < r; i += 32) d += W[j * r + i] * ck[i];
        d = warp_sum(d);
        const double bj = sg > 0.0 ? d / sg : 0.0;
        bb += bj * bj;
        if (sg > cutoff) {
          ++nkeep;
          bk2 += bj * bj;
          const double z = sg * bj / (sg * sg);
          a20 += z * z;
        }
      }
      const double perp = u2 - bb;
      if (nkeep == 0) {
        f = u2;
      } else if (a20 <= bound * bound) {
        f = fmax(perp, 0.0);
      } else {
        auto a2 = [&](double mu) {
          double acc = 0.0;
          for (int64_t j = 0; j < m; ++j) {
            if (rank[j] >= r || !(nrm[j] > cutoff)) continue;
            const double sg = nrm[j];
            double d = 0.0;
            for (int64_t i = lane; i < r; i += 32) d += W[j * r + i] * ck[i];
            d = warp_sum(d);
            const double z = sg * (d / sg) / (sg * sg + mu);
            acc += z * z;
          }
          return acc;
        };
        double sg0 = 0.0;
        for (int64_t j = 0; j < m; ++j)
          if (rank[j] == 0) sg0 = nrm[j];
        double lo = 0.0, hi = sg0 * sqrt(bk2) / bound;
        while (a2(hi) > bound * bound) hi *= 2.0;
        for (int it = 0; it < 200; ++it) {
          const double mid = 0.5 * (lo + hi);
          if (a2(mid) > bound * bound) lo = mid; else hi = mid;
          if (fabs(sqrt(a2(hi)) - bound) <= 1e-6 * bound) break;
        }
        double res = 0.0;
        for (int64_t j = 0; j < m; ++j) {
          if (rank[j] >= r || !(nrm[j] > cutoff)) continue;
          const double sg = nrm[j];
          double d = 0.0;
          for (int64_t i = lane; i < r; i += 32) d += W[j * r + i] * ck[i];
          d = warp_sum(d);
          const double bj = d / sg;
          const double z = sg * bj / (sg * sg + hi);
          const double rr = bj - sg * z;
          res += rr * rr;
        }
        f = fmax(perp + res, 0.0);
      }
    }
    if (lane == 0) f_out[int64_t(st) * K + k] = f;
  }
}

__global__ void seed_block_kernel(const double* __restrict__ V, int64_t ldv, const int32_t* __restrict__ col_map,
                                  const int64_t* __restrict__ seed_idx, const int32_t* __restrict__ seed_lab,
                                  const double* __restrict__ d_sqrt, int64_t S, int64_t M, int64_t K,
                                  double* __restrict__ At, double* __restrict__ Ut, double* __restrict__ uu) {
  // At[j][i] = V[s_i, col(j)], Ut[k][i] = [lab_i == k] d_sqrt[s_i]
  const int64_t total = (M + K) * S;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / S, i = e % S;
    const int64_t s = seed_idx[i];
    if (j < M) {
      At[j * S + i] = V[s * ldv + (col_map ? col_map[j] : j)];
    } else {
      const int64_t k = j - M;
      Ut[k * S + i] = (seed_lab[i] == k) ? d_sqrt[s] : 0.0;
    }
  }
  if (blockIdx.x == 0) {
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
      double a = 0.0;
      for (int64_t i = 0; i < S; ++i) {
        const double v = (seed_lab[i] == k) ? d_sqrt[seed_idx[i]] : 0.0;
        a += v * v;
      }
      uu[k] = a;
    }
  }
}

}  // namespace

extern "C" size_t swb_seed_fit_workspace_bytes(int64_t S, int64_t M, int64_t K, int64_t n_steps) {
  const int64_t n = (M + 1) / 2 * 2;
  const int64_t r = S < M ? S : M;
  // per step: the Jacobi path's W (n x r) + norms, or the bidiagonal path's
  // lane-interleaved ridge scratch (3 M doubles per lane and label)
  const size_t per = std::max(size_t(n) * r + 2 * size_t(M) + 2, size_t(K) * 3 * size_t(M) * 32);
  return swb_align_up(sizeof(double) * size_t(M + K) * S, 256) + swb_align_up(sizeof(double) * size_t(K), 256) +
         swb_align_up(sizeof(double) * size_t(n_steps) * per, 256);
}

extern "C" int swb_seed_fit_schedule(const double* V, int64_t ldv, const int32_t* col_map, const int64_t* seed_idx,
                                     const int32_t* seed_lab, int64_t S, const double* d_sqrt, int64_t M, int64_t K,
                                     const int32_t* steps, int64_t n_steps, int32_t max_step, double bound,
                                     double* f_out, void* workspace, size_t workspace_bytes, void* stream) {
  if (S <= 0 || M <= 0 || K <= 0 || n_steps <= 0 || !V || !seed_idx || !seed_lab || !d_sqrt || !steps || !f_out)
    return SWB_INVALID_PARAM;
  if (max_step > M || max_step <= 0) return SWB_INVALID_PARAM;
  if (!workspace || workspace_bytes < swb_seed_fit_workspace_bytes(S, M, K, n_steps)) return SWB_WORKSPACE_TOO_SMALL;
  cudaStream_t st = swb_stream(stream);
  char* base = static_cast<char*>(workspace);
  double* At = reinterpret_cast<double*>(base);
  double* Ut = At + M * S;
  double* uu = reinterpret_cast<double*>(base + swb_align_up(sizeof(double) * size_t(M + K) * S, 256));
  double* scratch = reinterpret_cast<double*>(reinterpret_cast<char*>(uu) + swb_align_up(sizeof(double) * size_t(K), 256));
  const int64_t n = (M + 1) / 2 * 2;
  const int64_t r = S < M ? S : M;
  const int64_t sstride = std::max(n * r + 2 * M + 2, K * 3 * M * 32);
  // SWB_SELECT_FAST=0: every step on the Jacobi SVD (measurement / A-B knob)
  const char* fe = getenv("SWB_SELECT_FAST");
  const int allow_fast = !(fe && fe[0] == '0');
  seed_block_kernel<<<swb_sm_count() * 2, 256, 0, st>>>(V, ldv, col_map, seed_idx, seed_lab, d_sqrt, S, M, K, At, Ut, uu);
  SWB_CHECK_LAUNCH();
  // QR: the cooperative whole-GPU kernel when column j fits in shared
  // memory (S <= 16K seeds); SWB_HH_COOP=0 keeps the single-CTA kernel
  static int hh_occ[64] = {};
  int& occ = hh_occ[swb_device()];
  const char* he = getenv("SWB_HH_COOP");
  const size_t hh_smem = sizeof(double) * size_t(S);
  bool coop = !(he && he[0] == '0') && S >= 64 && S <= 16384 && M + K >= 2;
  if (coop && occ == 0) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(householder_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(16384 * sizeof(double))));
    SWB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, householder_coop_kernel, HH_THREADS,
                                                               16384 * sizeof(double)));
    if (occ < 1) occ = -1;
  }
  if (coop && occ > 0) {
    int g = static_cast<int>(std::min<int64_t>(M + K, int64_t(occ) * swb_sm_count()));
    void* args[] = {&At, const_cast<int64_t*>(&S), const_cast<int64_t*>(&M), &Ut, const_cast<int64_t*>(&K)};
    SWB_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(householder_coop_kernel), dim3(g),
                                             dim3(HH_THREADS), args, hh_smem, st));
  } else {
    householder_kernel<<<1, 1024, 0, st>>>(At, S, M, Ut, K);
  }
  SWB_CHECK_LAUNCH();
  // shared memory: W (n_max x r_max) + sigma + rank when they fit
  const int64_t nmax = (int64_t(max_step) + 1) / 2 * 2;
  const int64_t rmax = S < max_step ? S : max_step;
  size_t smem = sizeof(double) * size_t(nmax) * rmax + sizeof(double) * 2 * size_t(max_step);
  if (smem > 200 * 1024) smem = sizeof(double) * 2 * size_t(max_step) + 64;  // W lives in global scratch
  (void)smem;
  const size_t dyn = 200 * 1024 + 1024;
  static unsigned long long attr = 0;
  if (swb_first_on_device(&attr)) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(jacobi_fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
  }
  jacobi_fit_kernel<<<static_cast<unsigned>(n_steps), 512, dyn, st>>>(At, S, M, Ut, K, steps, uu, bound, scratch,
                                                                       sstride, f_out, allow_fast);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}
