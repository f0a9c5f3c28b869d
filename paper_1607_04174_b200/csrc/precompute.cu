// Column kernels of the offline eigensolver (reference
// precompute fastrw.py:200-221, smallest_eigs linalg.py:98-175,
// _canonical_signs linalg.py:90-95, _snap_null_vector fastrw.py:180-197).
//
// The solver itself (Chebyshev-filtered subspace iteration over the stencil
// apply pass and the DMMA GEMMs) is driven from paper_1607_04174_b200/
// precompute.py; the kernels here are the N-length column reductions it
// needs, all with fixed-order (deterministic) partial sums:
//   swb_ritz_residuals   res2_j = || Y_j - theta_j X_j ||^2
//   swb_column_dots      h_j    = a^T X_j      (a = nullptr: ||X_j||^2)
//   swb_column_update    X_j    = (X_j - a * h_j) * s_j
//   swb_canonical_signs  flip X_j so its largest-|.| entry (first index on
//                        ties, numpy argmax) is positive
#include "swb_common.cuh"

namespace {

constexpr int CK_THREADS = 256;
constexpr int CK_BLOCKS = 296;   // partial-sum rows (fixed, so the reduction order is fixed)

// part[b][j] = sum over the block's rows of f(row, j); threads stride columns
template <int MODE>
__global__ void col_partial_kernel(const double* __restrict__ X, int64_t ldx, const double* __restrict__ Y,
                                   int64_t ldy, const double* __restrict__ vec, int64_t N, int64_t k,
                                   double* __restrict__ part) {
  const int64_t per = (N + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(N, r0 + per);
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    double s = 0.0;
    const double th = MODE == 0 ? vec[j] : 0.0;
    for (int64_t r = r0; r < r1; ++r) {
      const double x = X[r * ldx + j];
      if (MODE == 0) {            // residual: (Y - theta X)^2
        const double d = Y[r * ldy + j] - th * x;
        s = fma(d, d, s);
      } else if (MODE == 1) {     // dot with a row vector a[r]
        s = fma(vec[r], x, s);
      } else if (MODE == 3) {     // column dot of X and Y
        s = fma(x, Y[r * ldy + j], s);
      } else {                    // sum of squares
        s = fma(x, x, s);
      }
    }
    part[int64_t(blockIdx.x) * k + j] = s;
  }
}

__global__ void col_reduce_kernel(const double* __restrict__ part, int nb, int64_t k, double* __restrict__ out) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < k; j += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[int64_t(b) * k + j];
    out[j] = s;
  }
}

__global__ void col_update_kernel(double* __restrict__ X, int64_t ldx, int64_t N, int64_t k,
                                  const double* __restrict__ a, const double* __restrict__ h,
                                  const double* __restrict__ scale) {
  const int64_t total = N * k;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / k, j = e % k;
    double v = X[r * ldx + j];
    if (a) v = fma(-a[r], h[j], v);
    if (scale) v *= scale[j];
    X[r * ldx + j] = v;
  }
}

// per block: (max |x|, first row attaining it) per column
__global__ void col_absmax_partial_kernel(const double* __restrict__ X, int64_t ldx, int64_t N, int64_t k,
                                          double* __restrict__ pmax, int64_t* __restrict__ pidx) {
  const int64_t per = (N + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * per, r1 = min(N, r0 + per);
  for (int64_t j = threadIdx.x; j < k; j += blockDim.x) {
    double best = -1.0;
    int64_t bi = -1;
    for (int64_t r = r0; r < r1; ++r) {
      const double a = fabs(X[r * ldx + j]);
      if (a > best) { best = a; bi = r; }
    }
    pmax[int64_t(blockIdx.x) * k + j] = best;
    pidx[int64_t(blockIdx.x) * k + j] = bi;
  }
}

// sign of the entry at the global first argmax; flip the column if negative
__global__ void col_sign_kernel(const double* __restrict__ X, int64_t ldx, int nb, int64_t k,
                                const double* pmax, const int64_t* __restrict__ pidx, double* sign) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < k; j += int64_t(gridDim.x) * blockDim.x) {
    double best = -1.0;
    int64_t bi = -1;
    for (int b = 0; b < nb; ++b) {   // blocks cover increasing rows: strict > keeps the first index
      const double m = pmax[int64_t(b) * k + j];
      if (m > best) { best = m; bi = pidx[int64_t(b) * k + j]; }
    }
    const double v = bi >= 0 ? X[bi * ldx + j] : 0.0;
    sign[j] = v < 0.0 ? -1.0 : 1.0;   // np.sign(0) = 0 -> treated as +1
  }
}

int col_partials(int mode, const double* X, int64_t ldx, const double* Y, int64_t ldy, const double* vec, int64_t N,
                 int64_t k, double* out, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!X || !out || N < 0 || k <= 0 || ldx < k) return SWB_INVALID_PARAM;
  const size_t need = sizeof(double) * size_t(CK_BLOCKS) * size_t(k);
  if (!ws || ws_bytes < need) return SWB_WORKSPACE_TOO_SMALL;
  double* part = static_cast<double*>(ws);
  if (mode == 0) col_partial_kernel<0><<<CK_BLOCKS, CK_THREADS, 0, st>>>(X, ldx, Y, ldy, vec, N, k, part);
  else if (mode == 1) col_partial_kernel<1><<<CK_BLOCKS, CK_THREADS, 0, st>>>(X, ldx, Y, ldy, vec, N, k, part);
  else if (mode == 2) col_partial_kernel<2><<<CK_BLOCKS, CK_THREADS, 0, st>>>(X, ldx, Y, ldy, vec, N, k, part);
  else col_partial_kernel<3><<<CK_BLOCKS, CK_THREADS, 0, st>>>(X, ldx, Y, ldy, vec, N, k, part);
  SWB_CHECK_LAUNCH();
  col_reduce_kernel<<<static_cast<unsigned>((k + 255) / 256), 256, 0, st>>>(part, CK_BLOCKS, k, out);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

}  // namespace

extern "C" size_t swb_column_workspace_bytes(int64_t k) {
  return (sizeof(double) + sizeof(int64_t)) * size_t(CK_BLOCKS) * size_t(k > 0 ? k : 1) + 256;
}

extern "C" int swb_ritz_residuals(const double* X, int64_t ldx, const double* Y, int64_t ldy, const double* theta,
                                  int64_t N, int64_t k, double* res2, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  if (!Y || !theta || ldy < k) return SWB_INVALID_PARAM;
  return col_partials(0, X, ldx, Y, ldy, theta, N, k, res2, workspace, workspace_bytes, swb_stream(stream));
}

extern "C" int swb_column_dots(const double* X, int64_t ldx, const double* a, int64_t N, int64_t k, double* out,
                               void* workspace, size_t workspace_bytes, void* stream) {
  return col_partials(a ? 1 : 2, X, ldx, nullptr, 0, a, N, k, out, workspace, workspace_bytes, swb_stream(stream));
}

extern "C" int swb_column_products(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t N, int64_t k,
                                   double* out, void* workspace, size_t workspace_bytes, void* stream) {
  if (!Y || ldy < k) return SWB_INVALID_PARAM;
  return col_partials(3, X, ldx, Y, ldy, nullptr, N, k, out, workspace, workspace_bytes, swb_stream(stream));
}

extern "C" int swb_column_update(double* X, int64_t ldx, int64_t N, int64_t k, const double* a, const double* h,
                                 const double* scale, void* stream) {
  if (!X || N < 0 || k <= 0 || ldx < k || (a && !h)) return SWB_INVALID_PARAM;
  if (N == 0) return SWB_OK;
  col_update_kernel<<<swb_sm_count() * 8, 256, 0, swb_stream(stream)>>>(X, ldx, N, k, a, h, scale);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_canonical_signs(double* X, int64_t ldx, int64_t N, int64_t k, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  if (!X || N <= 0 || k <= 0 || ldx < k) return SWB_INVALID_PARAM;
  if (!workspace || workspace_bytes < swb_column_workspace_bytes(k)) return SWB_WORKSPACE_TOO_SMALL;
  cudaStream_t st = swb_stream(stream);
  double* pmax = static_cast<double*>(workspace);
  int64_t* pidx = reinterpret_cast<int64_t*>(pmax + size_t(CK_BLOCKS) * k);
  col_absmax_partial_kernel<<<CK_BLOCKS, CK_THREADS, 0, st>>>(X, ldx, N, k, pmax, pidx);
  SWB_CHECK_LAUNCH();
  // sign[j] overwrites block 0's partial of column j, which only column j's thread reads
  double* sign = pmax;
  col_sign_kernel<<<static_cast<unsigned>((k + 255) / 256), 256, 0, st>>>(X, ldx, CK_BLOCKS, k, pmax, pidx, sign);
  SWB_CHECK_LAUNCH();
  col_update_kernel<<<swb_sm_count() * 8, 256, 0, st>>>(X, ldx, N, k, nullptr, nullptr, sign);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}
