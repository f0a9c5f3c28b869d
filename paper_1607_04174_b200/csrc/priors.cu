// Registration data term on the GPU (reference registration.py:95-129):
//   s_k(x) = mean over patch offsets o of |F(clamp(x+o)) - M(clamp(x+o+d_k))|
//   sigma  = max(mean_x min_k s_k(x), 1e-8)
//   p_k(x) = softmax_k(-(s_k(x)/sigma)^2)
//
// The summand depends only on the unclamped point y = x + o:
//   E_k(y) = |F(clamp(y)) - M(clamp(y + d_k))|,
// so the patch sum is a box filter of E_k over the halo-extended grid and is
// separable.  box_scores_kernel stages E_k for a (32 x 8 x 4)-voxel tile plus
// halo in shared memory and runs the three 1-D box passes there (15 adds per
// voxel instead of 125 strided gathers at r = 2); a CTA walks a chunk of
// SC_KC labels and writes each voxel's chunk of scores as one 32-byte row
// segment.  Only the summation order differs from the reference's
// sequential meshgrid-order sum (relative difference ~1e-16).  Radii whose
// tile does not fit in shared memory use the direct per-(voxel, label)
// kernel, which keeps the reference order.
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

constexpr int SC_TX = 32, SC_KC = 4, SC_THREADS = 256;

struct BoxGeom {
  int tx, ty, tz;      // output tile
  int r, rz;           // halo (rz = 0 for 2-D)
  int ex, ey, ez;      // extended tile
  __host__ __device__ constexpr int n_e() const { return ex * ey * ez; }
  __host__ __device__ constexpr int n_bx() const { return tx * ey * ez; }
  __host__ __device__ constexpr int n_t() const { return tx * ty * tz; }
};

__host__ __device__ constexpr BoxGeom box_geom(int ndim, int r) {
  BoxGeom g{};
  g.tx = SC_TX;
  g.ty = ndim == 3 ? 8 : 32;
  g.tz = ndim == 3 ? 4 : 1;
  g.r = r;
  g.rz = ndim == 3 ? r : 0;
  g.ex = g.tx + 2 * r;
  g.ey = g.ty + 2 * r;
  g.ez = g.tz + 2 * g.rz;
  return g;
}

inline size_t box_smem_bytes(const BoxGeom& g) {
  return sizeof(double) * (size_t(g.n_e()) + size_t(g.n_bx()) + size_t(g.n_t()) * SC_KC);
}

// CT_NDIM / CT_R > 0: the tile geometry is a compile-time constant (every
// index split below divides by constants); CT_NDIM = 0: the runtime geometry.
template <int CT_NDIM, int CT_R>
__global__ void __launch_bounds__(SC_THREADS) box_scores_kernel(const double* __restrict__ F,
                                                                 const double* __restrict__ Mv, int nx, int ny,
                                                                 int nz, int ndim_rt, const int32_t* __restrict__ disp,
                                                                 int K, int radius_rt, double* __restrict__ scores,
                                                                 int64_t ld) {
  extern __shared__ double sm[];
  const int ndim = CT_NDIM ? CT_NDIM : ndim_rt;
  const int radius = CT_NDIM ? CT_R : radius_rt;
  const BoxGeom g = CT_NDIM ? box_geom(CT_NDIM ? CT_NDIM : 3, CT_R) : box_geom(ndim_rt, radius_rt);
  double* E = sm;                     // extended tile; reused for the y-pass output
  double* Bx = E + g.n_e();
  double* res = Bx + g.n_bx();        // [voxel][SC_KC]
  const int ntx = (nx + g.tx - 1) / g.tx, nty = (ny + g.ty - 1) / g.ty;
  const int tile = blockIdx.x;
  const int x0 = (tile % ntx) * g.tx, y0 = ((tile / ntx) % nty) * g.ty, z0 = (tile / (ntx * nty)) * g.tz;
  const int k0 = blockIdx.y * SC_KC;
  const int kc = min(SC_KC, K - k0);
  const int w = 2 * radius + 1;
  const double inv_off = 1.0 / double(ndim == 3 ? w * w * w : w * w);
  const int64_t plane = int64_t(nx) * ny;
  for (int kk = 0; kk < kc; ++kk) {
    const int dx = disp[(k0 + kk) * 3 + 0], dy = disp[(k0 + kk) * 3 + 1], dz = ndim == 3 ? disp[(k0 + kk) * 3 + 2] : 0;
    // E on the extended tile
    for (int i = threadIdx.x; i < g.n_e(); i += SC_THREADS) {
      const int ix = i % g.ex, iy = (i / g.ex) % g.ey, iz = i / (g.ex * g.ey);
      const int yx = x0 - g.r + ix, yy = y0 - g.r + iy, yz = z0 - g.rz + iz;
      const int fx = min(max(yx, 0), nx - 1), fy = min(max(yy, 0), ny - 1), fz = min(max(yz, 0), nz - 1);
      const int mx = min(max(yx + dx, 0), nx - 1), my = min(max(yy + dy, 0), ny - 1),
                mz = min(max(yz + dz, 0), nz - 1);
      E[i] = fabs(__ldg(F + fx + int64_t(nx) * fy + plane * fz) - __ldg(Mv + mx + int64_t(nx) * my + plane * mz));
    }
    __syncthreads();
    // x pass: Bx[(iz*ey + iy)*tx + ox]
    for (int i = threadIdx.x; i < g.n_bx(); i += SC_THREADS) {
      const int ox = i % g.tx, row = i / g.tx;
      const double* e = E + row * g.ex + ox;
      double a = e[0];
      for (int j = 1; j < w; ++j) a += e[j];
      Bx[i] = a;
    }
    __syncthreads();
    // y pass into E: By[(iz*ty + oy)*tx + ox]
    for (int i = threadIdx.x; i < g.tx * g.ty * g.ez; i += SC_THREADS) {
      const int ox = i % g.tx, oy = (i / g.tx) % g.ty, iz = i / (g.tx * g.ty);
      const double* b = Bx + (iz * g.ey + oy) * g.tx + ox;
      double a = b[0];
      for (int j = 1; j < w; ++j) a += b[j * g.tx];
      E[i] = a;
    }
    __syncthreads();
    // z pass + mean
    const int wz = 2 * g.rz + 1;
    for (int i = threadIdx.x; i < g.n_t(); i += SC_THREADS) {
      const double* b = E + i;
      double a = b[0];
      for (int j = 1; j < wz; ++j) a += b[j * g.tx * g.ty];
      res[i * SC_KC + kk] = a * inv_off;
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < g.n_t() * SC_KC; i += SC_THREADS) {
    const int v = i / SC_KC, kk = i % SC_KC;
    const int ox = v % g.tx, oy = (v / g.tx) % g.ty, oz = v / (g.tx * g.ty);
    const int x = x0 + ox, y = y0 + oy, z = z0 + oz;
    if (kk < kc && x < nx && y < ny && z < nz) scores[(x + int64_t(nx) * y + plane * z) * ld + k0 + kk] = res[i];
  }
}

// warp per voxel, the row in registers (K <= 32 * J): min over labels,
// accumulated per warp in a fixed voxel order, then per block in warp order
template <int J>
__global__ void rowmin_reg_kernel(const double* __restrict__ scores, int64_t N, int64_t K, int64_t ld,
                                  double* __restrict__ part) {
  __shared__ double wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  double acc = 0.0;
  for (int64_t v = gw; v < N; v += nw) {
    double mn = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int64_t k = lane + 32 * j;
      if (k < K) mn = fmin(mn, scores[v * ld + k]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    acc += mn;
  }
  if (lane == 0) wsum[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += wsum[w];
    part[blockIdx.x] = s;
  }
}

// warp per voxel, row in registers: logits = -(s/sigma)^2, max, exp, normalise
template <int J>
__global__ void softmax_reg_kernel(const double* __restrict__ scores, int64_t N, int64_t K, int64_t ld,
                                   const double* __restrict__ sigma_p, double* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const double sigma = *sigma_p;
  for (int64_t v = gw; v < N; v += nw) {
    double lg[J];
    double mx = -__longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int64_t k = lane + 32 * j;
      if (k < K) {
        const double r = scores[v * ld + k] / sigma;
        lg[j] = -(r * r);
        mx = fmax(mx, lg[j]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (lane + 32 * j < K) {
        lg[j] = exp(lg[j] - mx);
        s += lg[j];
      }
    }
    s = warp_sum(s);
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int64_t k = lane + 32 * j;
      if (k < K) out[v * ldo + k] = lg[j] / s;
    }
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
  const int64_t ld = (K + SC_KC - 1) / SC_KC * SC_KC;
  return swb_align_up(sizeof(double) * size_t(N) * size_t(ld), 256) + sizeof(double) * 1024;
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
  if (nx > INT32_MAX / 2 || ny > INT32_MAX / 2 || nz > INT32_MAX / 2 || K > INT32_MAX) return SWB_INVALID_PARAM;
  cudaStream_t st = swb_stream(stream);
  const int64_t ld = (K + SC_KC - 1) / SC_KC * SC_KC;
  double* scores = static_cast<double*>(workspace);
  double* part = reinterpret_cast<double*>(static_cast<char*>(workspace) +
                                           swb_align_up(sizeof(double) * size_t(N) * size_t(ld), 256));
  const int grid = swb_sm_count() * 8;
  const BoxGeom g = box_geom(ndim, patch_radius);
  const size_t smem = box_smem_bytes(g);
  const int64_t tiles = int64_t((nx + g.tx - 1) / g.tx) * ((ny + g.ty - 1) / g.ty) * ((nz + g.tz - 1) / g.tz);
  if (smem <= 227 * 1024 && tiles < INT32_MAX && (K + SC_KC - 1) / SC_KC <= 65535) {
    dim3 bg(unsigned(tiles), unsigned((K + SC_KC - 1) / SC_KC));
#define SWB_BOX(ND, R)                                                                                            \
  do {                                                                                                            \
    if (smem > 48 * 1024)                                                                                         \
      SWB_CUDA_TRY(cudaFuncSetAttribute(box_scores_kernel<ND, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                        int(smem)));                                                              \
    box_scores_kernel<ND, R><<<bg, SC_THREADS, smem, st>>>(fixed, moving, int(nx), int(ny), int(nz), ndim, disp,  \
                                                           int(K), patch_radius, scores, ld);                     \
  } while (0)
    if (ndim == 3 && patch_radius == 1) SWB_BOX(3, 1);
    else if (ndim == 3 && patch_radius == 2) SWB_BOX(3, 2);
    else if (ndim == 2 && patch_radius == 1) SWB_BOX(2, 1);
    else if (ndim == 2 && patch_radius == 2) SWB_BOX(2, 2);
    else SWB_BOX(0, 0);
#undef SWB_BOX
  } else {
    patch_scores_kernel<<<grid, 256, 0, st>>>(fixed, moving, nx, ny, nz, ndim, disp, K, patch_radius, scores, ld);
  }
  SWB_CHECK_LAUNCH();
  if (K <= 128) rowmin_reg_kernel<4><<<512, 256, 0, st>>>(scores, N, K, ld, part);
  else rowmin_sum_kernel<<<512, 256, 0, st>>>(scores, N, K, ld, part);
  SWB_CHECK_LAUNCH();
  sigma_kernel<<<1, 32, 0, st>>>(part, 512, N, sigma_out);
  SWB_CHECK_LAUNCH();
  if (K <= 32) softmax_reg_kernel<1><<<grid, 256, 0, st>>>(scores, N, K, ld, sigma_out, priors, ldp);
  else if (K <= 128) softmax_reg_kernel<4><<<grid, 256, 0, st>>>(scores, N, K, ld, sigma_out, priors, ldp);
  else softmax_kernel<<<grid, 256, 0, st>>>(scores, N, K, ld, sigma_out, priors, ldp);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}
