// Eigen-update coefficients (M x M, tiny): the refresh eigenvalues + stable
// sort (reference refresh.py:78-79) and the first-order rotation matrix
// (no reference function; SURVEY.md §7 "Recommended update definition").
#include "swb_common.cuh"

namespace {

// numpy ordering for the refreshed values: NaN sorts last, ties keep index order
__device__ __forceinline__ bool before(double a, int ia, double b, int ib) {
  const bool na = a != a, nb = b != b;
  if (na || nb) return (!na && nb) || (na && nb && ia < ib);
  return a < b || (a == b && ia < ib);
}

// lam_hat = max(quad/norm2, 0); rank by stable order; order[rank] = j
__global__ void refresh_sort_kernel(const double* __restrict__ quad, const double* __restrict__ norm2,
                                    int64_t M, double* __restrict__ lam_new, int64_t* __restrict__ order,
                                    double* __restrict__ lam_hat_scratch) {
  extern __shared__ double lam[];
  for (int64_t j = threadIdx.x; j < M; j += blockDim.x) {
    const double v = quad[j] / norm2[j];
    lam[j] = (v != v) ? v : fmax(v, 0.0);  // np.maximum propagates NaN
  }
  __syncthreads();
  for (int64_t j = threadIdx.x; j < M; j += blockDim.x) {
    const double a = lam[j];
    int64_t rank = 0;
    for (int64_t i = 0; i < M; ++i) rank += before(lam[i], static_cast<int>(i), a, static_cast<int>(j));
    order[rank] = j;
    lam_new[rank] = a;
    if (lam_hat_scratch) lam_hat_scratch[j] = a;
  }
}

// Column k of C = column i = order[k] of Cfo scaled by 1/||Cfo[:, i]||.
// One block per output column; the norm is a fixed-order tree reduction.
__global__ void first_order_c_kernel(const double* __restrict__ P, int64_t ldp,
                                     const double* __restrict__ lam, const int64_t* __restrict__ order,
                                     int64_t M, double gap_guard, double* __restrict__ C, int64_t ldc) {
  __shared__ double red[256];
  const int64_t k = blockIdx.x;
  const int64_t i = order[k];
  const double li = lam[i];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < M; j += blockDim.x) {
    double c;
    if (j == i) {
      c = 1.0;
    } else {
      const double gap = li - lam[j];
      const double p = P[j * ldp + i];
      c = (gap != 0.0 && fabs(p) <= gap_guard * fabs(gap)) ? p / gap : 0.0;
    }
    s += c * c;
    C[j * ldc + k] = c;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double scale = 1.0 / sqrt(red[0]);
  for (int64_t j = threadIdx.x; j < M; j += blockDim.x) C[j * ldc + k] *= scale;
}

}  // namespace

extern "C" int swb_update_coeffs(int method, const double* P, int64_t ldp, const double* lam_old,
                                 const double* quad, const double* norm2, int64_t M, double gap_guard,
                                 double* C, int64_t ldc, double* lam_new, int64_t* order, void* stream) {
  if (M <= 0 || M > 8192 || !quad || !norm2 || !lam_new || !order) return SWB_INVALID_PARAM;
  if (method != 0 && method != 1) return SWB_INVALID_PARAM;
  if (method == 1 && (!P || !lam_old || !C || ldp < M || ldc < M || !(gap_guard >= 0.0)))
    return SWB_INVALID_PARAM;
  cudaStream_t st = swb_stream(stream);
  const size_t smem = sizeof(double) * size_t(M);
  if (smem > 48 * 1024) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(refresh_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
  }
  refresh_sort_kernel<<<1, 1024, smem, st>>>(quad, norm2, M, lam_new, order, nullptr);
  SWB_CHECK_LAUNCH();
  if (method == 1) {
    first_order_c_kernel<<<static_cast<unsigned>(M), 256, 0, st>>>(P, ldp, lam_old, order, M, gap_guard,
                                                                   C, ldc);
    SWB_CHECK_LAUNCH();
  }
  return SWB_OK;
}
