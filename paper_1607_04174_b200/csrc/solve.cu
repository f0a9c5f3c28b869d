// Reduced-basis random-walker solve (reference fastrw.py:352-467):
//   pass 1   seed projections q_s, b_qn (stencil rows of L^ at the seeds)
//   system   (S+1)^2 bordered (gamma = 0) or S^2 (gamma > 0) seed system,
//            LU + rcond + solve, coefficients coeff (m x L)
//   pass 2   reconstruction V*coeff (+ g c), finalize (solver.py:55-66) and
//            hard labels (images.py:128-130) fused in one HBM-bound kernel
#include <cstdlib>

#include "swb_common.cuh"
#include "dmma_core.cuh"

namespace {

// ---------------------------------------------------------------------------
// seed rows in ELL form, built from the stencil coefficients
// ---------------------------------------------------------------------------
struct SeedGeom {
  LatticeDev lat;
  int n;                 // entries per row (2*ndir + 1), sorted by offset
  int64_t off[9];
  int dir[9], kind[9], dx[9], dy[9], dz[9];
};

int make_seed_geom(const swb_lattice* lat, SeedGeom* g) {
  int rc = swb_make_lattice(lat, &g->lat);
  if (rc) return rc;
  const LatticeDev& L = g->lat;
  struct E { int64_t off; int dir, kind, dx, dy, dz; };
  E es[9];
  int n = 0;
  for (int d = 0; d < L.ndir; ++d) {
    int64_t o = L.dx[d] + L.nx * (L.dy[d] + L.ny * int64_t(L.dz[d]));
    es[n++] = {o, d, 1, L.dx[d], L.dy[d], L.dz[d]};
    es[n++] = {-o, d, 2, -L.dx[d], -L.dy[d], -L.dz[d]};
  }
  es[n++] = {0, -1, 0, 0, 0, 0};
  for (int i = 1; i < n; ++i)
    for (int j = i; j > 0 && es[j].off < es[j - 1].off; --j) { E t = es[j]; es[j] = es[j - 1]; es[j - 1] = t; }
  g->n = n;
  for (int i = 0; i < n; ++i) {
    g->off[i] = es[i].off; g->dir[i] = es[i].dir; g->kind[i] = es[i].kind;
    g->dx[i] = es[i].dx; g->dy[i] = es[i].dy; g->dz[i] = es[i].dz;
  }
  return SWB_OK;
}

__global__ void seed_rows_kernel(const SeedGeom g, const double* __restrict__ what, const double* __restrict__ diag,
                                 const int64_t* __restrict__ seed_idx, int64_t S, int64_t* __restrict__ ell_idx,
                                 double* __restrict__ ell_val) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= S) return;
  const int64_t v = seed_idx[i];
  const int64_t x = v % g.lat.nx, y = (v / g.lat.nx) % g.lat.ny, z = v / (g.lat.nx * g.lat.ny);
  for (int e = 0; e < g.n; ++e) {
    int64_t idx = -1;
    double val = 0.0;
    if (g.kind[e] == 0) {
      idx = v; val = diag[v];
    } else {
      const int64_t x2 = x + g.dx[e], y2 = y + g.dy[e], z2 = z + g.dz[e];
      if (x2 >= 0 && x2 < g.lat.nx && y2 >= 0 && y2 < g.lat.ny && z2 >= 0 && z2 < g.lat.nz) {
        idx = v + g.off[e];
        const int64_t src = g.kind[e] == 1 ? v : idx;
        val = -what[src * g.lat.ndir + g.dir[e]];
      }
    }
    ell_idx[i * g.n + e] = idx;
    ell_val[i * g.n + e] = val;
  }
}

__device__ __forceinline__ int64_t find_seed(const int64_t* __restrict__ s, int64_t S, int64_t y) {
  int64_t lo = 0, hi = S;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (s[mid] < y) lo = mid + 1; else hi = mid;
  }
  return (lo < S && s[lo] == y) ? lo : -1;
}

// warp per seed
__global__ void seed_project_kernel(const double* __restrict__ V, int64_t ldv, int64_t row_base, int64_t own_begin,
                                    int64_t own_end, int64_t m, const int32_t* __restrict__ col_map,
                                    const int64_t* __restrict__ seed_idx, const int32_t* __restrict__ seed_lab,
                                    int64_t S, const int64_t* __restrict__ ell_idx, const double* __restrict__ ell_val,
                                    int64_t R, const double* __restrict__ d_sqrt, double dnorm, int64_t L,
                                    double* __restrict__ q_s, int64_t ldq, double* __restrict__ b_qn,
                                    double* __restrict__ bg, double* __restrict__ lsu, double* __restrict__ dsq_s) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  if (i >= S) return;
  const int64_t s = seed_idx[i];
  const bool owner = s >= own_begin && s < own_end;
  for (int64_t k = lane; k < L; k += 32) lsu[i * L + k] = 0.0;
  __syncwarp();
  double bgs = 0.0;
  if (lane == 0) {
    for (int64_t e = 0; e < R; ++e) {
      const int64_t y = ell_idx[i * R + e];
      if (y < 0) continue;
      const double val = ell_val[i * R + e];
      const int64_t t = find_seed(seed_idx, S, y);
      if (t >= 0) {
        if (owner) lsu[i * L + seed_lab[t]] += val * d_sqrt[y];  // l_s @ u_s_hat (fastrw.py:449)
      } else if (owner) {
        bgs += val * (d_sqrt[y] / dnorm);                       // seed_rows @ g_masked (:445)
      }
    }
    bg[i] = bgs;
    dsq_s[i] = owner ? d_sqrt[s] : 0.0;
  }
  for (int64_t j0 = 0; j0 < m; j0 += 32) {
    const int64_t j = j0 + lane;
    const bool act = j < m;
    const int64_t col = act ? (col_map ? col_map[j] : j) : 0;
    double acc = 0.0;
    for (int64_t e = 0; e < R; ++e) {
      const int64_t y = ell_idx[i * R + e];
      if (y < 0 || y < own_begin || y >= own_end) continue;
      if (find_seed(seed_idx, S, y) >= 0) continue;          // seed columns drop out of B
      const double val = ell_val[i * R + e];
      if (act) acc += val * V[(y - row_base) * ldv + col];
    }
    if (act) {
      b_qn[i * ldq + j] = acc;
      q_s[i * ldq + j] = owner ? V[(s - row_base) * ldv + col] : 0.0;
    }
  }
}

// ---------------------------------------------------------------------------
// small-system assembly helpers
// ---------------------------------------------------------------------------
__global__ void scale_cols_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t cols,
                                  const double* __restrict__ w, double* __restrict__ dst, int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / cols, c = e % cols;
    dst[r * ldd + c] = src[r * lds + c] * w[c];
  }
}

__global__ void transpose_kernel(const double* __restrict__ src, int64_t lds, int64_t rows, int64_t cols,
                                 double* __restrict__ dst, int64_t ldd) {
  __shared__ double tile[32][33];
  const int64_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = src[r * lds + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][k];
  }
}

__global__ void add_identity_kernel(double* __restrict__ A, int64_t lda, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    A[i * lda + i] += 1.0;
}

// border of the gamma = 0 system (fastrw.py:445-450) and its rhs
// A[:S,S] = -bg; A[S,:S] = -(gq*w)^T q_s^T; A[S,S] = g_s.g_s
// rhs[:S] = lsu; rhs[S,k] = sum_t g_s[t] [lab_t == k] dsq_s[t]
__global__ void border_kernel(int64_t S, int64_t m, int64_t L, const double* __restrict__ q_s, int64_t ldq,
                              const double* __restrict__ bg, const double* __restrict__ lsu,
                              const double* __restrict__ w, const double* __restrict__ gq,
                              const double* __restrict__ g_s, const double* __restrict__ dsq_s,
                              const int32_t* __restrict__ lab, double* __restrict__ A, int64_t lda,
                              double* __restrict__ rhs, int64_t ldr) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t t = wid; t < S; t += nwarps) {
    double acc = 0.0;
    for (int64_t j = lane; j < m; j += 32) acc += gq[j] * w[j] * q_s[t * ldq + j];
    acc = warp_sum(acc);
    if (lane == 0) {
      A[S * lda + t] = -acc;
      A[t * lda + S] = -bg[t];
    }
    for (int64_t k = lane; k < L; k += 32) rhs[t * ldr + k] = lsu[t * L + k];
  }
  if (blockIdx.x == 0) {
    __shared__ double red[32];
    double gg = 0.0;
    for (int64_t t = threadIdx.x; t < S; t += blockDim.x) gg += g_s[t] * g_s[t];
    gg = warp_sum(gg);
    if (lane == 0) red[threadIdx.x >> 5] = gg;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) s += red[q];
      A[S * lda + S] = s;
    }
    // rhs[S, k]: one warp per label, lanes over the seeds
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t k = warp; k < L; k += nw) {
      double a = 0.0;
      for (int64_t t = lane; t < S; t += 32)
        if (lab[t] == k) a += g_s[t] * dsq_s[t];
      a = warp_sum(a);
      if (lane == 0) rhs[S * ldr + k] = a;
    }
  }
}

// gamma > 0 rhs base: lsu + gamma * u_s_hat
__global__ void rhs_gamma_kernel(int64_t S, int64_t L, double gamma, const double* __restrict__ lsu,
                                 const double* __restrict__ dsq_s, const int32_t* __restrict__ lab,
                                 double* __restrict__ rhs, int64_t ldr) {
  const int64_t total = S * L;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = e / L, k = e % L;
    const double u = (lab[t] == k) ? dsq_s[t] : 0.0;
    rhs[t * ldr + k] = lsu[t * L + k] + gamma * u;
  }
}

// coeff = w * (proj [+ gamma t_p]); proj may be null (S == 0)
__global__ void coeff_kernel(int64_t m, int64_t L, const double* __restrict__ w, const double* __restrict__ proj,
                             int64_t ldp, const double* __restrict__ t_p, int64_t ldt, double gamma,
                             double* __restrict__ coeff) {
  const int64_t total = m * L;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / L, k = e % L;
    double v = proj ? proj[j * ldp + k] : 0.0;
    if (t_p) v = proj ? v + gamma * t_p[j * ldt + k] : gamma * t_p[j * ldt + k];
    coeff[j * L + k] = w[j] * v;
  }
}

__global__ void set_value_kernel(double* p, double v) { *p = v; }

// fastrw.py:399-403 spectral weights; g_s = d_sqrt[s]/||d_sqrt|| (fastrw.py:412, 442)
__global__ void weights_kernel(int64_t m, int64_t S, double gamma, const double* __restrict__ values,
                               const double* __restrict__ dsq_s, double dnorm, double* __restrict__ w,
                               double* __restrict__ g_s) {
  const int64_t t0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t t = t0; t < S; t += stride) g_s[t] = dsq_s[t] / dnorm;
  for (int64_t j = t0; j < m; j += stride) {
    const double v = values[j];
    w[j] = gamma == 0.0 ? (v > 1e-10 ? 1.0 / v : 0.0) : 1.0 / (v + gamma);
  }
}

// gq = V^T g_masked = (V^T g) - q_s^T g_s (fastrw.py:426):
// gq[j] = vtg[j] - sum_t q_s[t, j] g_s[t], g_s = dsq_s / dnorm: a (32 x 8)
// block per 32 columns, the 8 seed-row groups reduced in a fixed order
__global__ void __launch_bounds__(256) gq_kernel(int64_t m, int64_t S, const double* __restrict__ vtg,
                                                 const double* __restrict__ q_s, int64_t ldq,
                                                 const double* __restrict__ dsq_s, double dnorm,
                                                 double* __restrict__ gq) {
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j = blockIdx.x * 32 + tx;
  double s = 0.0;
  if (j < m)
    for (int64_t t = ty; t < S; t += 8) s += q_s[t * ldq + j] * (dsq_s[t] / dnorm);
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && j < m) {
    double a = red[0][tx];
#pragma unroll
    for (int g = 1; g < 8; ++g) a += red[g][tx];
    gq[j] = vtg[j] - a;
  }
}

__global__ void copy_row_kernel(const double* __restrict__ src, int64_t n, double* __restrict__ dst) {
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// ---------------------------------------------------------------------------
// pass 2: reconstruction + finalize + argmax
// ---------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ void finalize_row(double (&u)[L], int64_t r, int64_t r_begin, double* U, int64_t ldu,
                                             int32_t* labels, double* top2) {
  double sum = 0.0;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    u[k] = u[k] > 0.0 ? u[k] : (u[k] != u[k] ? u[k] : 0.0);  // np.clip(u, 0, None)
    sum += u[k];
  }
  if (sum == 0.0) {
#pragma unroll
    for (int k = 0; k < L; ++k) u[k] = 1.0 / double(L);
    sum = 1.0;
  }
  int best = 0;
  double p1 = -1.0, p2 = -1.0;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    u[k] = u[k] / sum;
    if (u[k] > p1) { p2 = p1; p1 = u[k]; best = k; }
    else if (u[k] > p2) p2 = u[k];
  }
  const int64_t o = r - r_begin;
  if (U) {
#pragma unroll
    for (int k = 0; k < L; ++k) U[o * ldu + k] = u[k];
  }
  labels[o] = best;
  if (top2) top2[o] = L > 1 ? p1 - p2 : 1.0;
}

constexpr int RC_WARPS = 8;

template <int L>
__global__ void __launch_bounds__(RC_WARPS * 32)
reconstruct_kernel(const double* __restrict__ V, int64_t ldv, int64_t row_base, int64_t r_begin, int64_t r_end,
                   int64_t mr, const double* __restrict__ coeff, const double* __restrict__ extra, double dnorm,
                   const double* __restrict__ d_sqrt, double* __restrict__ U, int64_t ldu,
                   int32_t* __restrict__ labels, double* __restrict__ top2) {
  extern __shared__ double cf[];  // mr x L
  for (int64_t e = threadIdx.x; e < mr * L; e += blockDim.x) cf[e] = coeff[e];
  double ex[L];
#pragma unroll
  for (int k = 0; k < L; ++k) ex[k] = extra ? extra[k] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const bool vec = ((ldv & 1) == 0) && ((reinterpret_cast<uintptr_t>(V) & 15) == 0);
  for (int64_t r = r_begin + gw; r < r_end; r += nw) {
    const double* row = V + (r - row_base) * ldv;
    double acc[L];
#pragma unroll
    for (int k = 0; k < L; ++k) acc[k] = 0.0;
    if (vec) {
      for (int64_t c = 2 * lane; c < mr; c += 64) {
        const double2 v = *reinterpret_cast<const double2*>(row + c);
        const double* a = cf + c * L;
#pragma unroll
        for (int k = 0; k < L; ++k) acc[k] += v.x * a[k];
        if (c + 1 < mr) {
#pragma unroll
          for (int k = 0; k < L; ++k) acc[k] += v.y * a[L + k];
        }
      }
    } else {
      for (int64_t c = lane; c < mr; c += 32) {
        const double v = row[c];
#pragma unroll
        for (int k = 0; k < L; ++k) acc[k] += v * cf[c * L + k];
      }
    }
#pragma unroll
    for (int k = 0; k < L; ++k) acc[k] = warp_sum(acc[k]);
    if (lane == 0) {
      const double ds = d_sqrt[r];
      const double g = ds / dnorm;
      double u[L];
#pragma unroll
      for (int k = 0; k < L; ++k) u[k] = (acc[k] + g * ex[k]) / ds;  // u_hat / d_sqrt (fastrw.py:462-464)
      finalize_row<L>(u, r, r_begin, U, ldu, labels, top2);
    }
  }
}

// Generic finalize for many labels: U already holds V*coeff (rows r_begin..).
// Register variant for L <= 32 * J: each lane keeps its J entries of the
// row in registers, so the row is read once and written once (the loop
// version reads it twice and writes it twice, with one row in flight per
// warp).  Same operations and order as finalize_many_kernel.
template <int J>
__global__ void finalize_many_reg_kernel(int64_t r_begin, int64_t r_end, int64_t L, const double* __restrict__ extra,
                                         double dnorm, const double* __restrict__ d_sqrt, double* __restrict__ U,
                                         int64_t ldu, int32_t* __restrict__ labels, double* __restrict__ top2) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  double ex[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int64_t k = lane + 32 * j;
    ex[j] = (extra && k < L) ? extra[k] : 0.0;
  }
  for (int64_t r = r_begin + gw; r < r_end; r += nw) {
    double* u = U + (r - r_begin) * ldu;
    double v[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int64_t k = lane + 32 * j;
      v[j] = k < L ? u[k] : 0.0;
    }
    const double ds = d_sqrt[r];
    const double g = ds / dnorm;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (lane + 32 * j < L) {
        double x = (v[j] + (extra ? g * ex[j] : 0.0)) / ds;
        x = x > 0.0 ? x : (x != x ? x : 0.0);
        v[j] = x;
        s += x;
      }
    }
    s = warp_sum(s);
    const bool dead = s == 0.0;
    if (dead) s = 1.0;
    double p1 = -1.0, p2 = -1.0;
    int best = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int64_t k = lane + 32 * j;
      if (k < L) {
        const double x = dead ? (1.0 / double(L)) : v[j] / s;
        u[k] = x;
        if (x > p1) { p2 = p1; p1 = x; best = static_cast<int>(k); }
        else if (x > p2) p2 = x;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double q1 = __shfl_xor_sync(0xffffffffu, p1, o);
      const double q2 = __shfl_xor_sync(0xffffffffu, p2, o);
      const int qb = __shfl_xor_sync(0xffffffffu, best, o);
      double n1, n2;
      int nb;
      if (q1 > p1 || (q1 == p1 && qb < best)) { n1 = q1; nb = qb; n2 = fmax(p1, q2); }
      else { n1 = p1; nb = best; n2 = fmax(p2, q1); }
      p1 = n1; p2 = n2; best = nb;
    }
    if (lane == 0) {
      labels[r - r_begin] = best;
      if (top2) top2[r - r_begin] = L > 1 ? p1 - p2 : 1.0;
    }
  }
}

__global__ void finalize_many_kernel(int64_t r_begin, int64_t r_end, int64_t L, const double* __restrict__ extra,
                                     double dnorm, const double* __restrict__ d_sqrt, double* __restrict__ U,
                                     int64_t ldu, int32_t* __restrict__ labels, double* __restrict__ top2) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = r_begin + gw; r < r_end; r += nw) {
    double* u = U + (r - r_begin) * ldu;
    const double ds = d_sqrt[r];
    const double g = ds / dnorm;
    double s = 0.0;
    for (int64_t k = lane; k < L; k += 32) {
      double v = (u[k] + (extra ? g * extra[k] : 0.0)) / ds;
      v = v > 0.0 ? v : (v != v ? v : 0.0);
      u[k] = v;
      s += v;
    }
    s = warp_sum(s);
    const bool dead = s == 0.0;
    if (dead) s = 1.0;
    double p1 = -1.0, p2 = -1.0;
    int best = 0x7fffffff;
    for (int64_t k = lane; k < L; k += 32) {
      const double v = dead ? (1.0 / double(L)) : u[k] / s;
      u[k] = v;
      if (v > p1) { p2 = p1; p1 = v; best = static_cast<int>(k); }
      else if (v > p2) p2 = v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double q1 = __shfl_xor_sync(0xffffffffu, p1, o);
      const double q2 = __shfl_xor_sync(0xffffffffu, p2, o);
      const int qb = __shfl_xor_sync(0xffffffffu, best, o);
      double n1, n2;
      int nb;
      if (q1 > p1 || (q1 == p1 && qb < best)) { n1 = q1; nb = qb; n2 = fmax(p1, q2); }
      else { n1 = p1; nb = best; n2 = fmax(p2, q1); }
      p1 = n1; p2 = n2; best = nb;
    }
    if (lane == 0) {
      labels[r - r_begin] = best;
      if (top2) top2[r - r_begin] = L > 1 ? p1 - p2 : 1.0;
    }
  }
}

__global__ void apply_seeds_kernel(const int64_t* __restrict__ seed_idx, const int32_t* __restrict__ seed_lab,
                                   int64_t S, int64_t r_begin, int64_t r_end, int64_t L, double* __restrict__ U,
                                   int64_t ldu, int32_t* __restrict__ labels, double* __restrict__ top2) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < S; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = seed_idx[i];
    if (s < r_begin || s >= r_end) continue;
    const int64_t o = s - r_begin;
    const int lab = seed_lab[i];
    if (U)
      for (int64_t k = 0; k < L; ++k) U[o * ldu + k] = (k == lab) ? 1.0 : 0.0;
    labels[o] = lab;
    if (top2) top2[o] = 1.0;
  }
}

__global__ void scatter_rows_kernel(const double* __restrict__ src, int64_t m, int64_t L,
                                    const int32_t* __restrict__ col_map, double* __restrict__ dst) {
  const int64_t total = m * L;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / L, k = e % L;
    dst[int64_t(col_map[j]) * L + k] = src[e];
  }
}

// DMMA-fed reconstruction for L <= 8 labels: a 128-row tile of V times the
// coefficient block (mr x L, zero-padded to 8 columns by the loader) on the
// FP64 tensor pipe (the K=400 reduction costs 2*8*K flops per voxel, far
// below the FP64 roof, so the kernel stays HBM-bound), 4-stage cp.async
// stream of V, and the finalize + argmax epilogue per row in registers.
constexpr int RD_WARPS = 8, RD_WTM = 2, RD_STAGES = 4;
using RdCfg = swb_core::Cfg<RD_WARPS, 1, RD_WTM, 1, RD_STAGES, false>;

__global__ void __launch_bounds__(RD_WARPS * 32)
reconstruct_dmma_kernel(const double* __restrict__ V, int64_t ldv, int64_t rows, int64_t mr,
                        const double* __restrict__ coeff, int64_t L, const double* __restrict__ extra, double dnorm,
                        const double* __restrict__ d_sqrt, double* __restrict__ U, int64_t ldu,
                        int32_t* __restrict__ labels, double* __restrict__ top2) {
  extern __shared__ __align__(16) double smem[];
  const int64_t m0 = int64_t(blockIdx.x) * RdCfg::BM;
  double acc[RD_WTM][1][2];
#pragma unroll
  for (int i = 0; i < RD_WTM; ++i) acc[i][0][0] = acc[i][0][1] = 0.0;
  swb_core::mainloop<RD_WARPS, 1, RD_WTM, 1, RD_STAGES, false>(acc, smem, V, ldv, coeff, L, 0, mr, m0, rows, 0, L);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 3;             // this lane holds labels 2q, 2q+1 of its row
  double ex0 = 0.0, ex1 = 0.0;
  if (extra) {
    if (2 * q < L) ex0 = extra[2 * q];
    if (2 * q + 1 < L) ex1 = extra[2 * q + 1];
  }
#pragma unroll
  for (int i = 0; i < RD_WTM; ++i) {
    const int64_t r = m0 + warp * RD_WTM * 8 + i * 8 + (lane >> 2);
    const bool row_ok = r < rows;
    // gather the row's 8 values into the quad leader (lane & 3 == 0)
    double v[8];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      v[2 * t] = __shfl_sync(0xffffffffu, acc[i][0][0], (lane & ~3) | t);
      v[2 * t + 1] = __shfl_sync(0xffffffffu, acc[i][0][1], (lane & ~3) | t);
    }
    double e[8];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      e[2 * t] = __shfl_sync(0xffffffffu, ex0, (lane & ~3) | t);
      e[2 * t + 1] = __shfl_sync(0xffffffffu, ex1, (lane & ~3) | t);
    }
    if (q != 0 || !row_ok) continue;
    const double ds = d_sqrt[r];
    const double g = ds / dnorm;
    double sum = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= L) break;
      double u = (v[k] + g * e[k]) / ds;                  // fastrw.py:462-464
      u = u > 0.0 ? u : (u != u ? u : 0.0);                // np.clip(u, 0, None)
      v[k] = u;
      sum += u;                                            // row sum in label order
    }
    if (sum == 0.0) {                                      // solver.py:63-65
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = 1.0 / double(L);
      sum = 1.0;
    }
    int best = 0;
    double p1 = -1.0, p2 = -1.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k >= L) break;
      const double p = v[k] / sum;
      v[k] = p;
      if (p > p1) { p2 = p1; p1 = p; best = k; } else if (p > p2) p2 = p;
    }
    labels[r] = best;
    if (top2) top2[r] = L > 1 ? p1 - p2 : 1.0;
    if (U) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k < L) U[r * ldu + k] = v[k];
    }
  }
}

template <int L>
int launch_reconstruct(const double* V, int64_t ldv, int64_t row_base, int64_t r_begin, int64_t r_end, int64_t mr,
                       const double* coeff, const double* extra, double dnorm, const double* d_sqrt, double* U,
                       int64_t ldu, int32_t* labels, double* top2, cudaStream_t st) {
  const size_t smem = sizeof(double) * size_t(mr) * L;
  auto kern = reconstruct_kernel<L>;
  if (smem > 48 * 1024)
    SWB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  SWB_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RC_WARPS * 32, smem));
  if (per_sm < 1) per_sm = 1;
  const int64_t rows = r_end - r_begin;
  int64_t grid = int64_t(swb_sm_count()) * per_sm;
  const int64_t need = (rows + RC_WARPS - 1) / RC_WARPS;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<static_cast<unsigned>(grid), RC_WARPS * 32, smem, st>>>(V, ldv, row_base, r_begin, r_end, mr, coeff, extra,
                                                                 dnorm, d_sqrt, U, ldu, labels, top2);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

}  // namespace

int swb_gemm_nn_alpha(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int64_t K,
                      int64_t M2, double* out, int64_t ldo, int accumulate, double alpha, cudaStream_t st);

extern "C" int swb_seed_rows(const swb_lattice* lat, const double* what, const double* diag, const int64_t* seed_idx,
                             int64_t S, int64_t* ell_idx, double* ell_val, void* stream) {
  SeedGeom g;
  int rc = make_seed_geom(lat, &g);
  if (rc) return rc;
  if (S < 0 || (S > 0 && (!what || !diag || !seed_idx || !ell_idx || !ell_val))) return SWB_INVALID_PARAM;
  if (S == 0) return SWB_OK;
  seed_rows_kernel<<<static_cast<unsigned>((S + 127) / 128), 128, 0, swb_stream(stream)>>>(g, what, diag, seed_idx, S,
                                                                                        ell_idx, ell_val);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_seed_project(const double* V, int64_t ldv, int64_t row_base, int64_t own_begin, int64_t own_end,
                                int64_t m, const int32_t* col_map, const int64_t* seed_idx, const int32_t* seed_lab,
                                int64_t S, const int64_t* ell_idx, const double* ell_val, int64_t R,
                                const double* d_sqrt, double dnorm, int64_t L, double* q_s, int64_t ldq,
                                double* b_qn, double* bg, double* lsu, double* dsq_s, void* stream) {
  if (S < 0 || m <= 0 || L <= 0 || R <= 0 || ldq < m) return SWB_INVALID_PARAM;
  if (S == 0) return SWB_OK;
  if (!V || !seed_idx || !seed_lab || !ell_idx || !ell_val || !d_sqrt || !q_s || !b_qn || !bg || !lsu || !dsq_s)
    return SWB_INVALID_PARAM;
  if (!(dnorm > 0.0)) return SWB_INVALID_PARAM;
  const int64_t threads = S * 32;
  seed_project_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, swb_stream(stream)>>>(
      V, ldv, row_base, own_begin, own_end, m, col_map, seed_idx, seed_lab, S, ell_idx, ell_val, R, d_sqrt, dnorm, L,
      q_s, ldq, b_qn, bg, lsu, dsq_s);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

// flag = 1 when the seeds break the kernels' precondition: seed_idx strictly
// ascending (sorted, unique) and in [0, n), labels in [0, L)
__global__ void check_seeds_kernel(const int64_t* __restrict__ seed_idx, const int32_t* __restrict__ seed_lab,
                                   int64_t S, int64_t n, int64_t L, double* __restrict__ flag) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < S; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = seed_idx[i];
    const int32_t l = seed_lab[i];
    const bool bad = s < 0 || s >= n || l < 0 || l >= L || (i + 1 < S && seed_idx[i + 1] <= s);
    if (bad) *flag = 1.0;
  }
}

extern "C" int swb_check_seeds(const int64_t* seed_idx, const int32_t* seed_lab, int64_t S, int64_t n, int64_t L,
                               double* flag_out, void* stream) {
  if (S < 0 || n <= 0 || L <= 0 || !flag_out || (S > 0 && (!seed_idx || !seed_lab))) return SWB_INVALID_PARAM;
  cudaStream_t st = swb_stream(stream);
  SWB_CUDA_TRY(cudaMemsetAsync(flag_out, 0, sizeof(double), st));
  if (S == 0) return SWB_OK;
  const int blocks = static_cast<int>(std::min<int64_t>((S + 255) / 256, 4 * swb_sm_count()));
  check_seeds_kernel<<<blocks, 256, 0, st>>>(seed_idx, seed_lab, S, n, L, flag_out);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

namespace {
struct SmallLayout {
  int64_t n, lda, ldr, ldm, lds;
  size_t off_A, off_rhs, off_bw, off_qt, off_piv, off_anorm, off_lu, off_tn, off_proj, off_w, off_rs, total;
  // Woodbury path (A = I - Ut Vt^T of rank r << n): Ut, Vt (n x ldw), K (r x ldk), its pivots / LU / solve
  // scratch, t (r x ldr), the TN GEMM scratch, gecon scratch
  int64_t r, ldw, ldk;
  size_t off_ut, off_vt, off_k, off_pk, off_luk, off_t, off_rsk, off_tnw, off_gw, off_nrm;
};

SmallLayout small_layout(int64_t S, int64_t m, int64_t L, int gamma_zero) {
  SmallLayout Ly{};
  Ly.n = gamma_zero ? S + 1 : S;
  Ly.lda = (Ly.n + 7) / 8 * 8;
  Ly.ldr = (L + 1) / 2 * 2;
  Ly.ldm = (m + 1) / 2 * 2;
  Ly.lds = (S + 1) / 2 * 2;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t at = o; o = swb_align_up(o + bytes, 256); return at; };
  Ly.off_A = take(sizeof(double) * size_t(Ly.n) * Ly.lda);
  Ly.off_rhs = take(sizeof(double) * size_t(Ly.n) * Ly.ldr);
  Ly.off_bw = take(sizeof(double) * size_t(S) * Ly.ldm);
  Ly.off_qt = take(sizeof(double) * size_t(m) * Ly.lds);
  Ly.off_piv = take(sizeof(int32_t) * size_t(Ly.n + 1));
  Ly.off_anorm = take(sizeof(double) * 2);
  Ly.off_lu = take(swb_lu_workspace_bytes(Ly.n));
  Ly.off_proj = take(sizeof(double) * size_t(m) * Ly.ldr);
  Ly.off_w = take(sizeof(double) * size_t(2 * m + S + 1));
  Ly.off_rs = take(swb_lu_solve_workspace_bytes(Ly.n, L));
  Ly.off_tn = take(S > 0 ? swb_gemm_tn_workspace_bytes(S, m, L) : 0);
  Ly.r = gamma_zero ? m + 2 : m;
  Ly.ldw = (Ly.r + 1) / 2 * 2;
  Ly.ldk = (Ly.r + 7) / 8 * 8;
  Ly.off_ut = take(sizeof(double) * size_t(Ly.n) * Ly.ldw);
  Ly.off_vt = take(sizeof(double) * size_t(Ly.n) * Ly.ldw);
  Ly.off_k = take(sizeof(double) * size_t(Ly.r) * Ly.ldk);
  Ly.off_pk = take(sizeof(int32_t) * size_t(Ly.r + 1));
  Ly.off_luk = take(swb_lu_workspace_bytes(Ly.r));
  Ly.off_t = take(sizeof(double) * size_t(Ly.r) * Ly.ldr);
  Ly.off_rsk = take(swb_lu_solve_workspace_bytes(Ly.r, L));
  Ly.off_tnw = take(std::max(swb_gemm_tn_workspace_bytes(Ly.n, Ly.r, Ly.r), swb_gemm_tn_workspace_bytes(Ly.n, Ly.r, L)));
  Ly.off_gw = take(swb_gecon_wb_workspace_bytes(Ly.n, Ly.r));
  Ly.off_nrm = take(sizeof(double) * size_t(Ly.n + 1));
  Ly.total = o;
  return Ly;
}

// Woodbury factors of the seed system (fastrw.py:430-450): A = I - Ut Vt^T.
// gamma > 0: Ut = (b_qn w), Vt = q_s (r = m).  gamma = 0, bordered
// (S+1) x (S+1) (r = m + 2): the border column -bg and corner alpha = g_s.g_s
// join the low-rank part as two extra columns,
//   Ut = [[b_qn w, bg, 0], [(gq w)^T, 0, 1]],  Vt = [[q_s, 0, 0], [0, 1, 1 - alpha]],
// so I - Ut Vt^T reproduces A[:S,:S] = I - (b_qn w) q_s^T, A[:S,S] = -bg,
// A[S,:S] = -(gq w)^T q_s^T and A[S,S] = alpha exactly.
__global__ void wb_factors_kernel(int64_t S, int64_t m, int g0, const double* __restrict__ Bw, int64_t ldm,
                                  const double* __restrict__ q_s, int64_t ldq, const double* __restrict__ bg,
                                  const double* __restrict__ w, const double* __restrict__ gq,
                                  const double* __restrict__ A, int64_t lda, double* __restrict__ Ut,
                                  double* __restrict__ Vt, int64_t ldw) {
  const int64_t n = g0 ? S + 1 : S, r = g0 ? m + 2 : m;
  const double alpha = g0 ? A[S * lda + S] : 0.0;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n * r; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / r, j = e % r;
    double u, v;
    if (i < S) {
      u = j < m ? Bw[i * ldm + j] : (j == m ? bg[i] : 0.0);
      v = j < m ? q_s[i * ldq + j] : 0.0;
    } else {
      u = j < m ? gq[j] * w[j] : (j == m ? 0.0 : 1.0);
      v = j < m ? 0.0 : (j == m ? 1.0 : 1.0 - alpha);
    }
    Ut[i * ldw + j] = u;
    Vt[i * ldw + j] = v;
  }
}

__global__ void eye_minus_kernel(double* __restrict__ K, int64_t ldk, int64_t r) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < r * r; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / r, j = e % r;
    K[i * ldk + j] = (i == j ? 1.0 : 0.0) - K[i * ldk + j];
  }
}
}  // namespace

extern "C" int swb_small_solve_ex(double gamma, int64_t S, int64_t m, int64_t L, const double* q_s,
                                  const double* b_qn, int64_t ldq, const double* bg, const double* lsu,
                                  const double* dsq_s, double dnorm, const int32_t* seed_lab, const double* values,
                                  const double* vtg, const double* t_p, int64_t ldt, double* coeff, double* extra,
                                  double* rcond_out, void* workspace, size_t workspace_bytes, void* stream,
                                  void* rcond_stream, void* rcond_event);

extern "C" int swb_small_dense_solve(double* A, int64_t n, int64_t lda, int32_t* piv, double* B, int64_t nrhs,
                                     int64_t ldb, double* anorm_out, double* rcond_out, void* stream);

extern "C" size_t swb_small_solve_workspace_bytes(int64_t S, int64_t m, int64_t L) {
  const SmallLayout a = small_layout(S, m, L, 1), b = small_layout(S, m, L, 0);
  return a.total > b.total ? a.total : b.total;
}

extern "C" int swb_small_solve(double gamma, int64_t S, int64_t m, int64_t L, const double* q_s, const double* b_qn,
                               int64_t ldq, const double* bg, const double* lsu, const double* dsq_s, double dnorm,
                               const int32_t* seed_lab, const double* values, const double* vtg, const double* t_p,
                               int64_t ldt, double* coeff, double* extra, double* rcond_out, void* workspace,
                               size_t workspace_bytes, void* stream) {
  return swb_small_solve_ex(gamma, S, m, L, q_s, b_qn, ldq, bg, lsu, dsq_s, dnorm, seed_lab, values, vtg, t_p, ldt,
                            coeff, extra, rcond_out, workspace, workspace_bytes, stream, nullptr, nullptr);
}

extern "C" int swb_small_solve_ex(double gamma, int64_t S, int64_t m, int64_t L, const double* q_s,
                                  const double* b_qn, int64_t ldq, const double* bg, const double* lsu,
                                  const double* dsq_s, double dnorm, const int32_t* seed_lab, const double* values,
                                  const double* vtg, const double* t_p, int64_t ldt, double* coeff, double* extra,
                                  double* rcond_out, void* workspace, size_t workspace_bytes, void* stream,
                                  void* rcond_stream, void* rcond_event) {
  if (!(gamma >= 0.0) || S < 0 || m <= 0 || L <= 0 || !values || !coeff || !rcond_out) return SWB_INVALID_PARAM;
  if (!(dnorm > 0.0)) return SWB_INVALID_PARAM;
  const int g0 = gamma == 0.0;
  if (g0 && (S == 0 || !vtg || !extra)) return SWB_INVALID_PARAM;  // solver.py:33-34 SingularSystem upstream
  if (!g0 && !t_p) return SWB_INVALID_PARAM;
  if (S > 0 && (!q_s || !b_qn || !lsu || !dsq_s || !seed_lab || (g0 && !bg))) return SWB_INVALID_PARAM;
  const SmallLayout Ly = small_layout(S, m, L, g0);
  if (!workspace || workspace_bytes < Ly.total) return SWB_WORKSPACE_TOO_SMALL;
  cudaStream_t st = swb_stream(stream);
  char* base = static_cast<char*>(workspace);
  double* A = reinterpret_cast<double*>(base + Ly.off_A);
  double* rhs = reinterpret_cast<double*>(base + Ly.off_rhs);
  double* Bw = reinterpret_cast<double*>(base + Ly.off_bw);
  double* qT = reinterpret_cast<double*>(base + Ly.off_qt);
  int32_t* piv = reinterpret_cast<int32_t*>(base + Ly.off_piv);
  double* anorm = reinterpret_cast<double*>(base + Ly.off_anorm);
  void* luws = base + Ly.off_lu;
  double* proj = reinterpret_cast<double*>(base + Ly.off_proj);
  void* tnws = base + Ly.off_tn;
  double* w = reinterpret_cast<double*>(base + Ly.off_w);
  double* gq = w + m;
  double* g_s = gq + m;
  const int grid = swb_sm_count() * 4;
  if (S > 0 && (ldq < m || (ldq & 1))) return SWB_INVALID_PARAM;
  if (!g0 && ldt < L) return SWB_INVALID_PARAM;

  weights_kernel<<<std::max<int64_t>(1, std::min<int64_t>((std::max(m, S) + 255) / 256, 1024)), 256, 0, st>>>(
      m, S, gamma, values, dsq_s, dnorm, w, g_s);
  SWB_CHECK_LAUNCH();
  if (g0) {
    gq_kernel<<<static_cast<unsigned>((m + 31) / 32), 256, 0, st>>>(m, S, vtg, q_s, ldq, dsq_s, dnorm, gq);
    SWB_CHECK_LAUNCH();
  }
  if (S == 0) {  // gamma > 0, no seeds: coeff = w * gamma t_p (fastrw.py:437-438)
    coeff_kernel<<<grid, 256, 0, st>>>(m, L, w, nullptr, 0, t_p, ldt, gamma, coeff);
    SWB_CHECK_LAUNCH();
    set_value_kernel<<<1, 1, 0, st>>>(rcond_out, 1.0);
    SWB_CHECK_LAUNCH();
    return SWB_OK;
  }
  // Bw = b_qn * w ; qT = q_s^T
  scale_cols_kernel<<<grid, 256, 0, st>>>(b_qn, ldq, S, m, w, Bw, Ly.ldm);
  SWB_CHECK_LAUNCH();
  {
    dim3 tb(32, 8), tg(static_cast<unsigned>((m + 31) / 32), static_cast<unsigned>((S + 31) / 32));
    transpose_kernel<<<tg, tb, 0, st>>>(q_s, ldq, S, m, qT, Ly.lds);
    SWB_CHECK_LAUNCH();
  }
  // A[:S,:S] = I - Bw q_s^T
  int rc = swb_gemm_nn_alpha(Bw, Ly.ldm, qT, Ly.lds, S, m, S, A, Ly.lda, 0, -1.0, st);
  if (rc) return rc;
  add_identity_kernel<<<grid, 256, 0, st>>>(A, Ly.lda, S);
  SWB_CHECK_LAUNCH();
  if (g0) {
    border_kernel<<<grid, 256, 0, st>>>(S, m, L, q_s, ldq, bg, lsu, w, gq, g_s, dsq_s, seed_lab, A, Ly.lda, rhs, Ly.ldr);
    SWB_CHECK_LAUNCH();
  } else {
    rhs_gamma_kernel<<<grid, 256, 0, st>>>(S, L, gamma, lsu, dsq_s, seed_lab, rhs, Ly.ldr);
    SWB_CHECK_LAUNCH();
    rc = swb_gemm_nn_alpha(Bw, Ly.ldm, t_p, ldt, S, m, L, rhs, Ly.ldr, 1, gamma, st);  // + gamma (Bw) t_p
    if (rc) return rc;
  }
  // A = I - Ut Vt^T has rank-r structure (r = m or m + 2): when r is well
  // below n, factor the r x r K = I - Vt^T Ut instead of A (Woodbury):
  // f = rhs + Ut K^-1 (Vt^T rhs), rcond of A from the same identity
  // (SWB_WOODBURY=0: always the LU of A)
  static const bool wb_env = [] { const char* e = getenv("SWB_WOODBURY"); return !(e && e[0] == '0'); }();
  const bool wood = wb_env && Ly.n >= Ly.r + 64;
  // systems up to 160 unknowns whose [A | rhs] fits in shared memory: one launch on column-owner threads
  // (lu.cu; faster than the blocked LU there; SWB_SMALL_LU=0: blocked path)
  static const bool small_env = [] { const char* e = getenv("SWB_SMALL_LU"); return !(e && e[0] == '0'); }();
  const bool small_n = !wood && small_env && Ly.n <= 160 && Ly.n + L <= 256 &&
                       sizeof(double) * size_t(Ly.n + 8) * size_t((Ly.n + L) | 1) <= size_t(220) * 1024;
  double* Ut = reinterpret_cast<double*>(base + Ly.off_ut);
  double* Vt = reinterpret_cast<double*>(base + Ly.off_vt);
  double* Kf = reinterpret_cast<double*>(base + Ly.off_k);
  int32_t* pk = reinterpret_cast<int32_t*>(base + Ly.off_pk);
  if (wood) {
    wb_factors_kernel<<<grid, 256, 0, st>>>(S, m, g0, Bw, Ly.ldm, q_s, ldq, bg, w, gq, A, Ly.lda, Ut, Vt, Ly.ldw);
    SWB_CHECK_LAUNCH();
    void* tnw = base + Ly.off_tnw;
    const size_t tnw_bytes = std::max(swb_gemm_tn_workspace_bytes(Ly.n, Ly.r, Ly.r),
                                      swb_gemm_tn_workspace_bytes(Ly.n, Ly.r, L));
    if ((rc = swb_gemm_tn(Vt, Ly.ldw, Ut, Ly.ldw, Ly.n, Ly.r, Ly.r, 0, Kf, Ly.ldk, tnw, tnw_bytes, stream))) return rc;
    eye_minus_kernel<<<grid, 256, 0, st>>>(Kf, Ly.ldk, Ly.r);
    SWB_CHECK_LAUNCH();
    if ((rc = swb_norm1(A, Ly.n, Ly.lda, anorm, base + Ly.off_nrm, sizeof(double) * size_t(Ly.n + 1), stream)))
      return rc;
    double* tb = reinterpret_cast<double*>(base + Ly.off_t);
    // K of up to 160 unknowns (c3: r = m + 2 <= 152): factors, pivots and K^-1 (Vt^T rhs) in one launch on
    // column-owner threads (lu.cu); larger K (c4: r = 402): the blocked LU
    const bool small_k = small_env && Ly.r <= 160 && Ly.r + L <= 256 &&
                         sizeof(double) * size_t(Ly.r + 8) * size_t((Ly.r + L) | 1) <= size_t(220) * 1024;
    if (small_k) {
      if ((rc = swb_gemm_tn(Vt, Ly.ldw, rhs, Ly.ldr, Ly.n, Ly.r, L, 0, tb, Ly.ldr, tnw, tnw_bytes, stream))) return rc;
      double* knorm = reinterpret_cast<double*>(base + Ly.off_luk);   // ||K||_1: not used (rcond is A's, below)
      if ((rc = swb_small_dense_solve(Kf, Ly.r, Ly.ldk, pk, tb, L, Ly.ldr, knorm, nullptr, stream))) return rc;
    } else {
      if ((rc = swb_lu_factor(Kf, Ly.r, Ly.ldk, pk, nullptr, base + Ly.off_luk, swb_lu_workspace_bytes(Ly.r), stream)))
        return rc;
      if ((rc = swb_gemm_tn(Vt, Ly.ldw, rhs, Ly.ldr, Ly.n, Ly.r, L, 0, tb, Ly.ldr, tnw, tnw_bytes, stream))) return rc;
      if ((rc = swb_lu_solve(Kf, Ly.r, Ly.ldk, pk, tb, L, Ly.ldr, base + Ly.off_rsk,
                             swb_lu_solve_workspace_bytes(Ly.r, L), stream)))
        return rc;
    }
    if ((rc = swb_gemm_nn_alpha(Ut, Ly.ldw, tb, Ly.ldr, Ly.n, Ly.r, L, rhs, Ly.ldr, 1, 1.0, st))) return rc;
  } else if (small_n) {
    // one launch: 1-norm, LU and the solve (lu.cu); gecon below, as for the blocked LU
    if ((rc = swb_small_dense_solve(A, Ly.n, Ly.lda, piv, rhs, L, Ly.ldr, anorm, nullptr, stream))) return rc;
  } else {
    rc = swb_lu_factor(A, Ly.n, Ly.lda, piv, anorm, luws, swb_lu_workspace_bytes(Ly.n), stream);
    if (rc) return rc;
    rc = swb_lu_solve(A, Ly.n, Ly.lda, piv, rhs, L, Ly.ldr, base + Ly.off_rs, swb_lu_solve_workspace_bytes(Ly.n, L),
                      stream);
    if (rc) return rc;
  }
  // proj = q_s^T f_s (m x L), reduction over the S seed rows
  rc = swb_gemm_tn(q_s, ldq, rhs, Ly.ldr, S, m, L, 0, proj, Ly.ldr, tnws, swb_gemm_tn_workspace_bytes(S, m, L), stream);
  if (rc) return rc;
  coeff_kernel<<<grid, 256, 0, st>>>(m, L, w, proj, Ly.ldr, g0 ? nullptr : t_p, ldt, gamma, coeff);
  SWB_CHECK_LAUNCH();
  if (g0) {
    copy_row_kernel<<<1, 128, 0, st>>>(rhs + S * Ly.ldr, L, extra);
    SWB_CHECK_LAUNCH();
  }
  if (rcond_stream && rcond_event) {
    // condition estimate concurrently with whatever the caller enqueues next
    // (the reconstruction); the caller joins rcond_stream before reusing the
    // workspace or reading rcond_out
    SWB_CUDA_TRY(cudaEventRecord(reinterpret_cast<cudaEvent_t>(rcond_event), st));
    SWB_CUDA_TRY(cudaStreamWaitEvent(swb_stream(rcond_stream), reinterpret_cast<cudaEvent_t>(rcond_event), 0));
  }
  void* rs_stream = (rcond_stream && rcond_event) ? rcond_stream : stream;
  if (wood)
    return swb_gecon_wb(Ly.n, Ly.r, Ut, Vt, Ly.ldw, Kf, Ly.ldk, pk, anorm, rcond_out, base + Ly.off_gw,
                        swb_gecon_wb_workspace_bytes(Ly.n, Ly.r), rs_stream);
  return swb_lu_rcond(A, Ly.n, Ly.lda, piv, anorm, rcond_out, luws, swb_lu_workspace_bytes(Ly.n), rs_stream);
}

extern "C" int swb_reconstruct_label(const double* V, int64_t ldv, int64_t row_base, int64_t r_begin, int64_t r_end,
                                     int64_t mr, const double* coeff, const double* extra, double dnorm,
                                     const double* d_sqrt, int64_t L, double* U, int64_t ldu, int32_t* labels,
                                     double* top2, void* stream) {
  if (!V || !coeff || !d_sqrt || !labels || mr <= 0 || L <= 0 || r_end < r_begin || r_begin < row_base)
    return SWB_INVALID_PARAM;
  if (!(dnorm > 0.0) || (U && ldu < L)) return SWB_INVALID_PARAM;
  if (r_end == r_begin) return SWB_OK;
  cudaStream_t st = swb_stream(stream);
  const size_t smem = sizeof(double) * size_t(mr) * L;
  if (L <= 8 && (ldv % 2) == 0 && (reinterpret_cast<uintptr_t>(V) & 15) == 0) {
    static unsigned long long attr = 0;
    if (swb_first_on_device(&attr)) {
      SWB_CUDA_TRY(cudaFuncSetAttribute(reconstruct_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(RdCfg::SMEM)));
    }
    const int64_t rows = r_end - r_begin;
    const int64_t grid = (rows + RdCfg::BM - 1) / RdCfg::BM;
    reconstruct_dmma_kernel<<<static_cast<unsigned>(grid), RdCfg::THREADS, RdCfg::SMEM, st>>>(
        V + (r_begin - row_base) * ldv, ldv, rows, mr, coeff, L, extra, dnorm, d_sqrt + r_begin, U, ldu, labels, top2);
    SWB_CHECK_LAUNCH();
    return SWB_OK;
  }
  if (L <= 8 && smem <= 200 * 1024) {
    switch (L) {
#define SWB_RC(n) case n: return launch_reconstruct<n>(V, ldv, row_base, r_begin, r_end, mr, coeff, extra, dnorm, d_sqrt, U, ldu, labels, top2, st);
      SWB_RC(1) SWB_RC(2) SWB_RC(3) SWB_RC(4) SWB_RC(5) SWB_RC(6) SWB_RC(7) SWB_RC(8)
#undef SWB_RC
      default: break;
    }
  }
  // many labels: DMMA GEMM into U, then a row-wise finalize
  if (!U || (ldu & 1) || (ldv & 1)) return SWB_INVALID_PARAM;  // U doubles as the GEMM output
  int rc = swb_gemm_nn_alpha(V + (r_begin - row_base) * ldv, ldv, coeff, L, r_end - r_begin, mr, L, U, ldu, 0, 1.0, st);
  if (rc) return rc;
  const int fg = swb_sm_count() * 8;
  if (L <= 32) finalize_many_reg_kernel<1><<<fg, 256, 0, st>>>(r_begin, r_end, L, extra, dnorm, d_sqrt, U, ldu, labels, top2);
  else if (L <= 64) finalize_many_reg_kernel<2><<<fg, 256, 0, st>>>(r_begin, r_end, L, extra, dnorm, d_sqrt, U, ldu, labels, top2);
  else if (L <= 128) finalize_many_reg_kernel<4><<<fg, 256, 0, st>>>(r_begin, r_end, L, extra, dnorm, d_sqrt, U, ldu, labels, top2);
  else if (L <= 256) finalize_many_reg_kernel<8><<<fg, 256, 0, st>>>(r_begin, r_end, L, extra, dnorm, d_sqrt, U, ldu, labels, top2);
  else finalize_many_kernel<<<fg, 256, 0, st>>>(r_begin, r_end, L, extra, dnorm, d_sqrt, U, ldu, labels, top2);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

// finalize + argmax of a reconstruction computed elsewhere (update_and_solve:
// the rotation GEMM's extra columns hold V (C coeff) = V' coeff): one thread
// per row, the same operations in the same order as reconstruct_dmma_kernel's
// epilogue (fastrw.py:462-464, solver.py:55-66, images.py:128-130).
template <int L>
__global__ void __launch_bounds__(256) finalize_rows_kernel(int64_t rows, const double* __restrict__ uraw,
                                                             int64_t ldr, const double* __restrict__ extra,
                                                             double dnorm, const double* __restrict__ d_sqrt,
                                                             double* __restrict__ U, int64_t ldu,
                                                             int32_t* __restrict__ labels, double* __restrict__ top2) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  double v[L];
#pragma unroll
  for (int k = 0; k < L; ++k) v[k] = uraw[r * ldr + k];
  const double ds = d_sqrt[r];
  const double g = ds / dnorm;
  double sum = 0.0;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    double u = (v[k] + g * (extra ? extra[k] : 0.0)) / ds;
    u = u > 0.0 ? u : (u != u ? u : 0.0);
    v[k] = u;
    sum += u;
  }
  if (sum == 0.0) {
#pragma unroll
    for (int k = 0; k < L; ++k) v[k] = 1.0 / double(L);
    sum = 1.0;
  }
  int best = 0;
  double p1 = -1.0, p2 = -1.0;
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const double p = v[k] / sum;
    v[k] = p;
    if (p > p1) { p2 = p1; p1 = p; best = k; } else if (p > p2) p2 = p;
  }
  labels[r] = best;
  if (top2) top2[r] = L > 1 ? p1 - p2 : 1.0;
  if (U) {
#pragma unroll
    for (int k = 0; k < L; ++k) U[r * ldu + k] = v[k];
  }
}

extern "C" int swb_finalize_label(int64_t r_begin, int64_t r_end, int64_t L, const double* uraw, int64_t ldr,
                                  const double* extra, double dnorm, const double* d_sqrt, double* U, int64_t ldu,
                                  int32_t* labels, double* top2, void* stream) {
  if (!uraw || !d_sqrt || !labels || L <= 0 || r_end < r_begin || ldr < L || !(dnorm > 0.0) || (U && ldu < L))
    return SWB_INVALID_PARAM;
  const int64_t rows = r_end - r_begin;
  if (rows == 0) return SWB_OK;
  cudaStream_t st = swb_stream(stream);
  const double* ds = d_sqrt + r_begin;
  if (L <= 8) {
    const unsigned grid = static_cast<unsigned>((rows + 255) / 256);
    switch (L) {
#define SWB_FR(n) case n: finalize_rows_kernel<n><<<grid, 256, 0, st>>>(rows, uraw, ldr, extra, dnorm, ds, U, ldu, labels, top2); break;
      SWB_FR(1) SWB_FR(2) SWB_FR(3) SWB_FR(4) SWB_FR(5) SWB_FR(6) SWB_FR(7) SWB_FR(8)
#undef SWB_FR
      default: break;
    }
    SWB_CHECK_LAUNCH();
    return SWB_OK;
  }
  // many labels: in place (U must be the raw buffer), warp per row
  if (U != uraw || ldu != ldr) return SWB_INVALID_PARAM;
  const int fg = swb_sm_count() * 8;
  if (L <= 32) finalize_many_reg_kernel<1><<<fg, 256, 0, st>>>(r_begin, r_end, L, extra, dnorm, d_sqrt, U, ldu, labels, top2);
  else if (L <= 64) finalize_many_reg_kernel<2><<<fg, 256, 0, st>>>(r_begin, r_end, L, extra, dnorm, d_sqrt, U, ldu, labels, top2);
  else if (L <= 128) finalize_many_reg_kernel<4><<<fg, 256, 0, st>>>(r_begin, r_end, L, extra, dnorm, d_sqrt, U, ldu, labels, top2);
  else if (L <= 256) finalize_many_reg_kernel<8><<<fg, 256, 0, st>>>(r_begin, r_end, L, extra, dnorm, d_sqrt, U, ldu, labels, top2);
  else finalize_many_kernel<<<fg, 256, 0, st>>>(r_begin, r_end, L, extra, dnorm, d_sqrt, U, ldu, labels, top2);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_apply_seeds(const int64_t* seed_idx, const int32_t* seed_lab, int64_t S, int64_t r_begin,
                               int64_t r_end, int64_t L, double* U, int64_t ldu, int32_t* labels, double* top2,
                               void* stream) {
  if (S < 0 || !labels || (S > 0 && (!seed_idx || !seed_lab))) return SWB_INVALID_PARAM;
  if (S == 0) return SWB_OK;
  apply_seeds_kernel<<<static_cast<unsigned>((S + 255) / 256), 256, 0, swb_stream(stream)>>>(
      seed_idx, seed_lab, S, r_begin, r_end, L, U, ldu, labels, top2);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_scatter_rows(const double* src, int64_t m, int64_t L, const int32_t* col_map, double* dst,
                                int64_t mr, void* stream) {
  if (!src || !col_map || !dst || m <= 0 || L <= 0 || mr <= 0) return SWB_INVALID_PARAM;
  cudaStream_t st = swb_stream(stream);
  SWB_CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(double) * size_t(mr) * L, st));
  scatter_rows_kernel<<<swb_sm_count() * 2, 256, 0, st>>>(src, m, L, col_map, dst);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

namespace {
__global__ void gather_rows_kernel(const double* __restrict__ src, int64_t lds, const int32_t* __restrict__ row_map,
                                   int64_t m, int64_t ncols, double* __restrict__ dst, int64_t ldd) {
  const int64_t total = m * ncols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / ncols, k = e % ncols;
    dst[j * ldd + k] = src[int64_t(row_map[j]) * lds + k];
  }
}
}  // namespace

extern "C" int swb_gather_rows(const double* src, int64_t lds, const int32_t* row_map, int64_t m, int64_t ncols,
                               double* dst, int64_t ldd, void* stream) {
  if (!src || !row_map || !dst || m < 0 || ncols <= 0 || ldd < ncols) return SWB_INVALID_PARAM;
  if (m == 0) return SWB_OK;
  gather_rows_kernel<<<swb_sm_count() * 2, 256, 0, swb_stream(stream)>>>(src, lds, row_map, m, ncols, dst, ldd);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

namespace {
// P^_masked = priors * d_sqrt, seed rows zeroed (fastrw.py:395-397)
__global__ void prior_hat_kernel(const double* __restrict__ priors, int64_t ldp, int64_t N, int64_t L,
                                 const double* __restrict__ d_sqrt, double* __restrict__ out, int64_t ldo) {
  const int64_t total = N * L;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / L, k = e % L;
    out[r * ldo + k] = priors[r * ldp + k] * d_sqrt[r];
  }
}

__global__ void zero_rows_kernel(const int64_t* __restrict__ rows, int64_t S, int64_t row_begin, int64_t row_end,
                                 int64_t L, double* __restrict__ out, int64_t ldo) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < S * L; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = rows[i / L];
    if (r >= row_begin && r < row_end) out[(r - row_begin) * ldo + i % L] = 0.0;
  }
}

// hard labels of an existing field (images.py:128-130): argmax, ties lowest
__global__ void argmax_rows_kernel(const double* __restrict__ U, int64_t ldu, int64_t N, int64_t L,
                                   int32_t* __restrict__ labels, double* __restrict__ top2) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < N; r += int64_t(gridDim.x) * blockDim.x) {
    const double* u = U + r * ldu;
    int best = 0;
    double p1 = u[0], p2 = -__longlong_as_double(0x7ff0000000000000LL);
    for (int64_t k = 1; k < L; ++k) {
      const double v = u[k];
      if (v > p1) { p2 = p1; p1 = v; best = static_cast<int>(k); }
      else if (v > p2) p2 = v;
    }
    labels[r] = best;
    if (top2) top2[r] = L > 1 ? p1 - p2 : 1.0;
  }
}
}  // namespace

extern "C" int swb_prior_hat(const double* priors, int64_t ldp, int64_t row_begin, int64_t row_end, int64_t L,
                             const double* d_sqrt, const int64_t* seed_idx, int64_t S, double* out, int64_t ldo,
                             void* stream) {
  if (!priors || !d_sqrt || !out || L <= 0 || ldp < L || ldo < L || row_end < row_begin) return SWB_INVALID_PARAM;
  if (S > 0 && !seed_idx) return SWB_INVALID_PARAM;
  cudaStream_t st = swb_stream(stream);
  const int64_t N = row_end - row_begin;
  if (N == 0) return SWB_OK;
  prior_hat_kernel<<<swb_sm_count() * 8, 256, 0, st>>>(priors, ldp, N, L, d_sqrt + row_begin, out, ldo);
  SWB_CHECK_LAUNCH();
  if (S > 0) {
    zero_rows_kernel<<<static_cast<unsigned>(std::min<int64_t>((S * L + 255) / 256, 4096)), 256, 0, st>>>(
        seed_idx, S, row_begin, row_end, L, out, ldo);
    SWB_CHECK_LAUNCH();
  }
  return SWB_OK;
}

extern "C" int swb_argmax_rows(const double* U, int64_t ldu, int64_t N, int64_t L, int32_t* labels, double* top2,
                               void* stream) {
  if (!U || !labels || L <= 0 || ldu < L || N < 0) return SWB_INVALID_PARAM;
  if (N == 0) return SWB_OK;
  argmax_rows_kernel<<<swb_sm_count() * 8, 256, 0, swb_stream(stream)>>>(U, ldu, N, L, labels, top2);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}
