// Registration data term on the GPU (reference registration.py:95-129):
//   s_k(x) = mean over patch offsets o of |F(clamp(x+o)) - M(clamp(x+o+d_k))|
//   sigma  = max(mean_x min_k s_k(x), 1e-8)
//   p_k(x) = softmax_k(-(s_k(x)/sigma)^2)
// Offsets run in the reference's meshgrid order (first axis slowest) and the
// per-voxel sums are sequential in that order, so s_k matches bit for bit.
#include "swb_common.cuh"

namespace {

__device__ __forceinline__ int64_t clampi(int64_t v, int64_t n) { return v < 0 ? 0 : (v >= n ? n - 1 : v); }

// one thread per (voxel, label); scores written row-major N x ld
__global__ void patch_scores_kernel(const double* __restrict__ F, const double* __restrict__ Mv, int64_t nx,
                                    int64_t ny, int64_t nz, int ndim, const int32_t* __restrict__ disp, int64_t K,
                                    int radius, double* __restrict__ scores, int64_t ld) {
  const int64_t N = nx * ny * nz;
  const int64_t total = N * K;
  const int w = 2 * radius + 1;
  const int n_off = ndim == 3 ? w * w * w : w * w;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t v = e / K, k = e % K;
    const int64_t x = v % nx, y = (v / nx) % ny, z = v / (nx * ny);
    const int64_t dx = disp[k * 3 + 0], dy = disp[k * 3 + 1], dz = ndim == 3 ? disp[k * 3 + 2] : 0;
    double acc = 0.0;
    for (int t = 0; t < n_off; ++t) {
      // meshgrid(..., indexing="ij").reshape(-1, d): first axis varies slowest
      int ox, oy, oz;
      if (ndim == 3) { ox = t / (w * w) - radius; oy = (t / w) % w - radius; oz = t % w - radius; }
      else { ox = t / w - radius; oy = t % w - radius; oz = 0; }
      const int64_t fx = clampi(x + ox, nx), fy = clampi(y + oy, ny), fz = ndim == 3 ? clampi(z + oz, nz) : 0;
      const int64_t mx = clampi(x + ox + dx, nx), my = clampi(y + oy + dy, ny),
                    mz = ndim == 3 ? clampi(z + oz + dz, nz) : 0;
      acc += fabs(F[fx + nx * (fy + ny * fz)] - Mv[mx + nx * (my + ny * mz)]);
    }
    scores[v * ld + k] = acc / double(n_off);
  }
}

// per-voxel min over labels, summed in fixed order per block (deterministic)
__global__ void rowmin_sum_kernel(const double* __restrict__ scores, int64_t N, int64_t K, int64_t ld,
                                  double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < N; v += int64_t(gridDim.x) * blockDim.x) {
    double mn = scores[v * ld];
    for (int64_t k = 1; k < K; ++k) mn = fmin(mn, scores[v * ld + k]);
    s += mn;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void sigma_kernel(const double* __restrict__ part, int n_part, int64_t N, double* __restrict__ sigma) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n_part; ++i) s += part[i];
    *sigma = fmax(s / double(N), 1e-8);
  }
}

// warp per voxel: logits = -(s/sigma)^2, subtract the max, exp, normalise
__global__ void softmax_kernel(const double* __restrict__ scores, int64_t N, int64_t K, int64_t ld,
                               const double* __restrict__ sigma_p, double* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const double sigma = *sigma_p;
  for (int64_t v = gw; v < N; v += nw) {
    double mx = -__longlong_as_double(0x7ff0000000000000LL);
    for (int64_t k = lane; k < K; k += 32) {
      const double r = scores[v * ld + k] / sigma;
      mx = fmax(mx, -(r * r));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double s = 0.0;
    for (int64_t k = lane; k < K; k += 32) {
      const double r = scores[v * ld + k] / sigma;
      const double e = exp(-(r * r) - mx);
      out[v * ldo + k] = e;
      s += e;
    }
    s = warp_sum(s);
    for (int64_t k = lane; k < K; k += 32) out[v * ldo + k] /= s;
  }
}
}  // namespace

extern "C" size_t swb_similarity_priors_workspace_bytes(int64_t N, int64_t K) {
  return swb_align_up(sizeof(double) * size_t(N) * size_t(K), 256) + sizeof(double) * 1024;
}

extern "C" int swb_similarity_priors(const double* fixed, const double* moving, int64_t nx, int64_t ny, int64_t nz,
                                     int32_t ndim, const int32_t* disp, int64_t K, int32_t patch_radius,
                                     double* priors, int64_t ldp, double* sigma_out, void* workspace,
                                     size_t workspace_bytes, void* stream) {
  if (!fixed || !moving || !disp || !priors || !sigma_out || K <= 0 || patch_radius < 0 || ldp < K)
    return SWB_INVALID_PARAM;
  if ((ndim != 2 && ndim != 3) || nx <= 0 || ny <= 0 || nz <= 0 || (ndim == 2 && nz != 1)) return SWB_INVALID_PARAM;
  const int64_t N = nx * ny * nz;
  if (!workspace || workspace_bytes < swb_similarity_priors_workspace_bytes(N, K)) return SWB_WORKSPACE_TOO_SMALL;
  cudaStream_t st = swb_stream(stream);
  double* scores = static_cast<double*>(workspace);
  double* part = reinterpret_cast<double*>(static_cast<char*>(workspace) +
                                           swb_align_up(sizeof(double) * size_t(N) * size_t(K), 256));
  const int grid = swb_sm_count() * 8;
  patch_scores_kernel<<<grid, 256, 0, st>>>(fixed, moving, nx, ny, nz, ndim, disp, K, patch_radius, scores, K);
  SWB_CHECK_LAUNCH();
  rowmin_sum_kernel<<<512, 256, 0, st>>>(scores, N, K, K, part);
  SWB_CHECK_LAUNCH();
  sigma_kernel<<<1, 32, 0, st>>>(part, 512, N, sigma_out);
  SWB_CHECK_LAUNCH();
  softmax_kernel<<<grid, 256, 0, st>>>(scores, N, K, K, sigma_out, priors, ldp);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}
