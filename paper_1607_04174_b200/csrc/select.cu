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
#include "swb_common.cuh"

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

// Round-robin tournament: round rd, slot p of n (even) players
__device__ __forceinline__ void rr_pair(int rd, int p, int n, int& a, int& b) {
  // player 0 fixed, others rotate
  auto pos = [&](int k) { return k == 0 ? 0 : 1 + ((k - 1 + rd) % (n - 1)); };
  a = pos(p);
  b = pos(n - 1 - p);
}

// One CTA per scheduled m.  W (m_pad x r) = R_m^T in shared or global
// scratch; sigma, b, f outputs per step.
__global__ void __launch_bounds__(512) jacobi_fit_kernel(const double* __restrict__ At, int64_t S, int64_t M,
                                                         const double* __restrict__ Ut, int64_t K,
                                                         const int32_t* __restrict__ steps,
                                                         const double* __restrict__ uu, double bound,
                                                         double* __restrict__ scratch, int64_t scratch_stride,
                                                         double* __restrict__ f_out) {
  extern __shared__ double sm[];
  __shared__ int rotated;
  const int st = blockIdx.x;
  const int64_t m = steps[st];
  const int64_t r = (S < m ? S : m);  // rows of R_m
  const int n = static_cast<int>((m + 1) / 2 * 2);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool in_smem = size_t(n) * r * sizeof(double) + size_t(m) * 2 * sizeof(double) <= 200 * 1024;
  double* W = in_smem ? sm : scratch + st * scratch_stride;  // n x r, row j = column j of R_m
  double* nrm = in_smem ? sm + size_t(n) * r : scratch + st * scratch_stride + size_t(n) * r;
  for (int64_t e = threadIdx.x; e < int64_t(n) * r; e += blockDim.x) {
    const int64_t j = e / r, i = e % r;
    W[e] = (j < m && i <= j) ? At[j * S + i] : 0.0;
  }
  __syncthreads();
  // one-sided Jacobi sweeps
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int rd = 0; rd < n - 1; ++rd) {
      for (int p = warp; p < n / 2; p += nw) {
        int a, b;
        rr_pair(rd, p, n, a, b);
        if (a > b) { const int t = a; a = b; b = t; }
        double* wa = W + int64_t(a) * r;
        double* wb = W + int64_t(b) * r;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int64_t i = lane; i < r; i += 32) {
          const double x = wa[i], y = wb[i];
          al += x * x; be += y * y; ga += x * y;
        }
        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
        if (fabs(ga) > 1e-15 * sqrt(al * be) && ga != 0.0) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int64_t i = lane; i < r; i += 32) {
            const double x = wa[i], y = wb[i];
            wa[i] = c * x - s * y;
            wb[i] = s * x + c * y;
          }
          if (lane == 0) rotated = 1;
        }
      }
      __syncthreads();
    }
    const int any = rotated;
    __syncthreads();
    if (!any) break;
  }
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
  return swb_align_up(sizeof(double) * size_t(M + K) * S, 256) + swb_align_up(sizeof(double) * size_t(K), 256) +
         swb_align_up(sizeof(double) * size_t(n_steps) * (size_t(n) * r + 2 * size_t(M) + 2), 256);
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
  const int64_t sstride = n * r + 2 * M + 2;
  seed_block_kernel<<<swb_sm_count() * 2, 256, 0, st>>>(V, ldv, col_map, seed_idx, seed_lab, d_sqrt, S, M, K, At, Ut, uu);
  SWB_CHECK_LAUNCH();
  householder_kernel<<<1, 1024, 0, st>>>(At, S, M, Ut, K);
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
                                                                       sstride, f_out);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}
