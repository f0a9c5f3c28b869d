// Super-vertex aggregation (reference aggregation.py:89-216).
//
//   swb_build_aggregation  greedy region growing, restated exactly
//                          (aggregation.py:89-127).  Inherently sequential
//                          (flat scan order + FIFO BFS decide membership),
//                          so it runs as native host code on host buffers;
//                          the L1 prior distance uses numpy's pairwise
//                          summation so threshold decisions match bit for bit.
//   swb_delta_weights      2 per lattice neighbour in another cluster
//                          (aggregation.py:130-139), one thread per voxel.
//   swb_cluster_rows       out[c] = sum over members x (ascending) of
//                          (1/|c|) * (X[x] * w[x])  -- eta_bar^T (w X), the
//                          CSR order of aggregation.py:173-174 / 207-209.
//   swb_csr_spmm           Y = A X for a host-assembled CSR (the aggregate
//                          Laplacian), CSR order, one warp per row.
#include <deque>
#include <vector>

#include "swb_common.cuh"

namespace {

// numpy's pairwise summation for contiguous float64 (PW_BLOCKSIZE = 128)
double np_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

__global__ void delta_weights_kernel(LatticeDev L, const int32_t* __restrict__ cid, double* __restrict__ delta) {
  const int64_t N = L.nx * L.ny * L.nz;
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < N; v += int64_t(gridDim.x) * blockDim.x) {
    const int64_t x = v % L.nx, y = (v / L.nx) % L.ny, z = v / (L.nx * L.ny);
    const int32_t c = cid[v];
    double d = 0.0;
    for (int k = 0; k < L.ndir; ++k) {
      for (int s = -1; s <= 1; s += 2) {
        const int64_t x2 = x + s * L.dx[k], y2 = y + s * L.dy[k], z2 = z + s * L.dz[k];
        if (x2 < 0 || x2 >= L.nx || y2 < 0 || y2 >= L.ny || z2 < 0 || z2 >= L.nz) continue;
        if (cid[x2 + L.nx * (y2 + L.ny * z2)] != c) d += 2.0;
      }
    }
    delta[v] = d;
  }
}

// one warp per cluster, lanes over columns
__global__ void cluster_rows_kernel(const double* __restrict__ X, int64_t ldx, int64_t m, const double* __restrict__ w,
                                    const int64_t* __restrict__ order, const int64_t* __restrict__ off,
                                    int64_t n_super, double* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t c = gw; c < n_super; c += nw) {
    const int64_t b = off[c], e = off[c + 1];
    const double inv = 1.0 / double(e - b);
    for (int64_t j = lane; j < m; j += 32) {
      double s = 0.0;
      for (int64_t t = b; t < e; ++t) {
        const int64_t x = order[t];
        const double v = w ? __dmul_rn(X[x * ldx + j], w[x]) : X[x * ldx + j];
        s = __dadd_rn(s, __dmul_rn(inv, v));
      }
      out[c * ldo + j] = s;
    }
  }
}

__global__ void csr_spmm_kernel(const int64_t* __restrict__ indptr, const int64_t* __restrict__ indices,
                                const double* __restrict__ data, int64_t nrows, const double* __restrict__ X,
                                int64_t ldx, int64_t m, double* __restrict__ Y, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = gw; r < nrows; r += nw) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    for (int64_t j = lane; j < m; j += 32) {
      double s = 0.0;
      for (int64_t t = b; t < e; ++t) s = __dadd_rn(s, __dmul_rn(data[t], X[indices[t] * ldx + j]));
      Y[r * ldy + j] = s;
    }
  }
}

}  // namespace

extern "C" int swb_build_aggregation(const double* priors, int64_t ldp, int64_t L, const int64_t* dims, int32_t ndim,
                                     int32_t max_cluster_radius, double similarity_tol, int32_t* cluster_ids,
                                     int64_t* n_super) {
  if (!priors || !dims || !cluster_ids || !n_super || ndim < 1 || ndim > 3 || L <= 0 || ldp < L ||
      max_cluster_radius < 0)
    return SWB_INVALID_PARAM;
  int64_t n = 1;
  int64_t stride[3] = {1, 1, 1};
  for (int a = 0; a < ndim; ++a) {
    if (dims[a] <= 0) return SWB_INVALID_PARAM;
    stride[a] = n;
    n *= dims[a];
  }
  std::vector<double> diff(static_cast<size_t>(L));
  for (int64_t i = 0; i < n; ++i) cluster_ids[i] = -1;
  int64_t next_id = 0;
  std::deque<int64_t> queue;
  auto coord = [&](int64_t v, int a) { return (v / stride[a]) % dims[a]; };
  for (int64_t start = 0; start < n; ++start) {
    if (cluster_ids[start] >= 0) continue;
    if (next_id > INT32_MAX) return SWB_INVALID_PARAM;
    cluster_ids[start] = static_cast<int32_t>(next_id);
    const double* ps = priors + start * ldp;
    int64_t cs[3] = {0, 0, 0};
    for (int a = 0; a < ndim; ++a) cs[a] = coord(start, a);
    queue.clear();
    queue.push_back(start);
    while (!queue.empty()) {
      const int64_t x = queue.front();
      queue.pop_front();
      for (int a = 0; a < ndim; ++a) {
        const int64_t cx = coord(x, a);
        for (int step = -1; step <= 1; step += 2) {
          if (cx + step < 0 || cx + step >= dims[a]) continue;
          const int64_t y = x + step * stride[a];
          if (cluster_ids[y] >= 0) continue;
          int64_t cheb = 0;
          for (int b = 0; b < ndim; ++b) {
            const int64_t d = coord(y, b) - cs[b];
            cheb = std::max<int64_t>(cheb, d < 0 ? -d : d);
          }
          if (cheb > max_cluster_radius) continue;
          const double* py = priors + y * ldp;
          for (int64_t k = 0; k < L; ++k) diff[k] = fabs(py[k] - ps[k]);
          if (np_pairwise_sum(diff.data(), L) > similarity_tol) continue;
          cluster_ids[y] = static_cast<int32_t>(next_id);
          queue.push_back(y);
        }
      }
    }
    ++next_id;
  }
  *n_super = next_id;
  return SWB_OK;
}

extern "C" int swb_delta_weights(const swb_lattice* lat, const int32_t* cluster_ids, double* delta, void* stream) {
  LatticeDev L;
  if (swb_make_lattice(lat, &L) || !cluster_ids || !delta) return SWB_INVALID_PARAM;
  delta_weights_kernel<<<swb_sm_count() * 8, 256, 0, swb_stream(stream)>>>(L, cluster_ids, delta);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_cluster_rows(const double* X, int64_t ldx, int64_t m, const double* w, const int64_t* order,
                                const int64_t* offsets, int64_t n_super, double* out, int64_t ldo, void* stream) {
  if (!X || !order || !offsets || !out || m <= 0 || ldx < m || ldo < m || n_super < 0) return SWB_INVALID_PARAM;
  if (n_super == 0) return SWB_OK;
  cluster_rows_kernel<<<swb_sm_count() * 8, 256, 0, swb_stream(stream)>>>(X, ldx, m, w, order, offsets, n_super, out,
                                                                          ldo);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_csr_spmm(const int64_t* indptr, const int64_t* indices, const double* data, int64_t nrows,
                            const double* X, int64_t ldx, int64_t m, double* Y, int64_t ldy, void* stream) {
  if (!indptr || !X || !Y || nrows < 0 || m <= 0 || ldx < m || ldy < m) return SWB_INVALID_PARAM;
  if (nrows == 0) return SWB_OK;
  csr_spmm_kernel<<<swb_sm_count() * 8, 256, 0, swb_stream(stream)>>>(indptr, indices, data, nrows, X, ldx, m, Y,
                                                                      ldy);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}
