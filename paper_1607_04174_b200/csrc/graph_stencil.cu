// Graph coefficients and the grid-stencil passes over the eigenbasis.
//
// graph:   reference graphs.py:127-140 (build_graph) + :143-159
//          (laplacian_from_weights, NORMALIZED).  The Laplacian is never
//          materialised as CSR: per voxel we keep the normalised forward
//          edge weights what[x*ndir+d] and the diagonal, and every consumer
//          recomputes L^ rows on the fly.
// stencil: refresh.py:75-77 (quad = diag(V^T L'V), norms = diag(V^T V)) and
//          the difference stencil W = (L^new - L^old) V of the first-order
//          update, HBM-bound.  One warp owns a 32-column block of one x-line
//          (nx consecutive voxel rows); all warps sweep the column blocks in
//          lockstep so the +-y / +-z neighbour rows of a line are being read
//          by other warps at the same time and hit in L2.
//
// The arithmetic that feeds reference-visible values (degrees, d_sqrt,
// L^ entries, the L^ v row sums) uses explicit _rn intrinsics so nvcc cannot
// contract it into FMAs: it mirrors scipy's evaluation order exactly.
#include "swb_common.cuh"

namespace {

constexpr double W_MIN = 1e-8;  // graphs.py:20

// Neighbour entries of one row, sorted by flat-offset (the CSR column order of
// the reference Laplacian, graphs.py:122-123 sort_indices): kind 0 = diag,
// kind 1 = forward edge d of x, kind 2 = backward edge d (stored at x-off).
struct NbrList {
  int n;
  int64_t off[9];
  int dir[9];
  int kind[9];
  int dx[9], dy[9], dz[9];
};

int build_nbr_list(const LatticeDev& L, NbrList* out) {
  NbrList nl{};
  struct E { int64_t off; int dir, kind, dx, dy, dz; };
  E es[9];
  int n = 0;
  for (int d = 0; d < L.ndir; ++d) {
    int64_t o = L.dx[d] + L.nx * (L.dy[d] + L.ny * int64_t(L.dz[d]));
    es[n++] = {o, d, 1, L.dx[d], L.dy[d], L.dz[d]};
    es[n++] = {-o, d, 2, -L.dx[d], -L.dy[d], -L.dz[d]};
  }
  es[n++] = {0, -1, 0, 0, 0, 0};
  for (int i = 1; i < n; ++i)  // insertion sort by offset
    for (int j = i; j > 0 && es[j].off < es[j - 1].off; --j) { E t = es[j]; es[j] = es[j - 1]; es[j - 1] = t; }
  nl.n = n;
  for (int i = 0; i < n; ++i) {
    nl.off[i] = es[i].off; nl.dir[i] = es[i].dir; nl.kind[i] = es[i].kind;
    nl.dx[i] = es[i].dx; nl.dy[i] = es[i].dy; nl.dz[i] = es[i].dz;
  }
  *out = nl;
  return SWB_OK;
}

// Lattice + sorted neighbour list travel as by-value kernel parameters
// (param space), so concurrent calls with different lattices cannot race.
struct StencilGeom {
  LatticeDev lat;
  NbrList nbr;
};

int make_geom(const swb_lattice* lat, StencilGeom* g) {
  int rc = swb_make_lattice(lat, &g->lat);
  if (rc) return rc;
  return build_nbr_list(g->lat, &g->nbr);
}

__device__ __forceinline__ bool in_grid(const LatticeDev& L, int64_t x, int64_t y, int64_t z) {
  return x >= 0 && x < L.nx && y >= 0 && y < L.ny && z >= 0 && z < L.nz;
}

// --- graph build -----------------------------------------------------------

__global__ void edge_weight_kernel(const StencilGeom g, const double* __restrict__ I, double beta, int weight_mode,
                                   const uint8_t* __restrict__ cut, double* __restrict__ w, int64_t N) {
  const int nd = g.lat.ndir;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < N * nd;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t v = e / nd;
    const int d = static_cast<int>(e % nd);
    const int64_t x = v % g.lat.nx, y = (v / g.lat.nx) % g.lat.ny, z = v / (g.lat.nx * g.lat.ny);
    const int64_t x2 = x + g.lat.dx[d], y2 = y + g.lat.dy[d], z2 = z + g.lat.dz[d];
    double out = 0.0;
    if (in_grid(g.lat, x2, y2, z2) && !(cut && cut[e])) {
      const int64_t u = x2 + g.lat.nx * (y2 + g.lat.ny * z2);
      const double diff = __dadd_rn(I[v], -I[u]);
      const double arg = weight_mode == 0 ? fabs(diff) : __dmul_rn(diff, diff);
      out = fmax(exp(__dmul_rn(-beta, arg)), W_MIN);  // graphs.py:136
    }
    w[e] = out;
  }
}

// degrees in increasing neighbour-index order (scipy csr row sum), d_sqrt,
// diag = (inv*d)*inv with inv = 1/d_sqrt (graphs.py:154-158)
__global__ void degree_kernel(const StencilGeom g, const double* __restrict__ w, double* __restrict__ d_sqrt,
                              double* __restrict__ diag, int32_t* __restrict__ degenerate, int64_t N) {
  const int nd = g.lat.ndir;
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < N;
       v += int64_t(gridDim.x) * blockDim.x) {
    const int64_t x = v % g.lat.nx, y = (v / g.lat.nx) % g.lat.ny, z = v / (g.lat.nx * g.lat.ny);
    double deg = 0.0;
    for (int e = 0; e < g.nbr.n; ++e) {
      const int kind = g.nbr.kind[e];
      if (kind == 0) continue;
      const int64_t x2 = x + g.nbr.dx[e], y2 = y + g.nbr.dy[e], z2 = z + g.nbr.dz[e];
      if (!in_grid(g.lat, x2, y2, z2)) continue;
      const int d = g.nbr.dir[e];
      const double we = kind == 1 ? w[v * nd + d] : w[(v + g.nbr.off[e]) * nd + d];
      deg = __dadd_rn(deg, we);
    }
    if (!(deg > 0.0)) {
      atomicExch(degenerate, 1);
      d_sqrt[v] = 0.0;
      diag[v] = 0.0;
      continue;
    }
    const double ds = sqrt(deg);
    const double inv = 1.0 / ds;
    d_sqrt[v] = ds;
    diag[v] = __dmul_rn(__dmul_rn(inv, deg), inv);
  }
}

// what = 0.5*((inv_x*w)*inv_y + (inv_y*w)*inv_x), in place over w
__global__ void normalize_kernel(const StencilGeom g, double* __restrict__ w, const double* __restrict__ d_sqrt, int64_t N) {
  const int nd = g.lat.ndir;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < N * nd;
       e += int64_t(gridDim.x) * blockDim.x) {
    const double we = w[e];
    if (we == 0.0) continue;
    const int64_t v = e / nd;
    const int d = static_cast<int>(e % nd);
    const int64_t u = v + g.lat.dx[d] + g.lat.nx * (g.lat.dy[d] + g.lat.ny * int64_t(g.lat.dz[d]));
    const double iv = 1.0 / d_sqrt[v], iu = 1.0 / d_sqrt[u];
    const double a = __dmul_rn(__dmul_rn(iv, we), iu);
    const double b = __dmul_rn(__dmul_rn(iu, we), iv);
    w[e] = __dmul_rn(__dadd_rn(a, b), 0.5);
  }
}

// --- stencil passes --------------------------------------------------------

constexpr int ST_WARPS = 8;
constexpr int ST_CTAS_PER_SM = 4;

// One warp: column block cb (32 columns, lane = column), one x-line.
// Accumulates per-column partials in registers; flushes them into
// slots[warp][col][3] whenever the warp moves to another column block.
template <bool DELTA>
__global__ void __launch_bounds__(ST_WARPS * 32)
stencil_kernel(const StencilGeom g, const double* __restrict__ V, int64_t ldv, int64_t row_base, int64_t line_begin,
               int64_t n_lines, int64_t M, int n_cb,
               const double* __restrict__ what_new, const double* __restrict__ diag_new,
               const double* __restrict__ what_old, const double* __restrict__ diag_old,
               const double* __restrict__ d_sqrt, double* __restrict__ W, int64_t ldw,
               int64_t w_row0, double* __restrict__ slots, int64_t slot_ld) {
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t n_items = int64_t(n_cb) * n_lines;
  const int64_t nx = g.lat.nx;
  const int nd = g.lat.ndir;
  const int nn = g.nbr.n;

  double q = 0.0, s2 = 0.0, sd = 0.0;
  int cur_cb = -1;
  for (int64_t it = gwarp; it < n_items; it += n_warps) {
    const int cb = static_cast<int>(it / n_lines);
    const int64_t line = line_begin + it % n_lines;
    if (cb != cur_cb) {
      if (cur_cb >= 0) {
        double* sl = slots + gwarp * slot_ld * 3 + int64_t(cur_cb * 32 + lane) * 3;
        sl[0] = q; sl[1] = s2; sl[2] = sd;
      }
      q = s2 = sd = 0.0;
      cur_cb = cb;
    }
    const int64_t col = int64_t(cb) * 32 + lane;
    const bool active = col < M;
    const int64_t r0 = line * nx;
    const int64_t yz = line;  // y + ny*z
    const int64_t y = yz % g.lat.ny, z = yz / g.lat.ny;
#pragma unroll 2
    for (int64_t xi = 0; xi < nx; ++xi) {
      const int64_t r = r0 + xi;
      const double* vrow = V + (r - row_base) * ldv;
      const double c = active ? vrow[col] : 0.0;
      double lv = 0.0, dw = 0.0;
      for (int e = 0; e < nn; ++e) {
        const int kind = g.nbr.kind[e];
        if (kind == 0) {
          const double dn = diag_new[r];
          lv = __dadd_rn(lv, __dmul_rn(dn, c));
          if (DELTA) dw += (dn - diag_old[r]) * c;
          continue;
        }
        const int64_t x2 = xi + g.nbr.dx[e], y2 = y + g.nbr.dy[e], z2 = z + g.nbr.dz[e];
        if (!in_grid(g.lat, x2, y2, z2)) continue;
        const int d = g.nbr.dir[e];
        const int64_t cidx = (kind == 1 ? r : r + g.nbr.off[e]) * nd + d;
        const double an = what_new[cidx];
        const double ao = DELTA ? what_old[cidx] : 0.0;
        if (an == 0.0 && ao == 0.0) continue;
        const double vn = active ? V[(r + g.nbr.off[e] - row_base) * ldv + col] : 0.0;
        lv = __dadd_rn(lv, __dmul_rn(-an, vn));
        if (DELTA) dw -= (an - ao) * vn;
      }
      q += c * lv;
      s2 += c * c;
      sd += c * d_sqrt[r];
      if (DELTA && active) W[(r - w_row0) * ldw + col] = dw;
    }
  }
  if (cur_cb >= 0) {
    double* sl = slots + gwarp * slot_ld * 3 + int64_t(cur_cb * 32 + lane) * 3;
    sl[0] = q; sl[1] = s2; sl[2] = sd;
  }
}

// out[col] = sum over warps (fixed order) of slots[w][col][k]
__global__ void slot_reduce_kernel(const double* __restrict__ slots, int64_t slot_ld, int64_t n_warps,
                                   int64_t M, double* __restrict__ quad, double* __restrict__ norm2,
                                   double* __restrict__ vtd) {
  const int64_t col = blockIdx.x;
  const int k = blockIdx.y;
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t w = threadIdx.x; w < n_warps; w += blockDim.x) s += slots[(w * slot_ld + col) * 3 + k];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0 && col < M) {
    double* dst = k == 0 ? quad : (k == 1 ? norm2 : vtd);
    if (dst) dst[col] = red[0];
  }
}

int64_t stencil_grid() { return int64_t(swb_sm_count()) * ST_CTAS_PER_SM; }

template <bool DELTA>
int run_stencil(const swb_lattice* lat, const double* V, int64_t ldv, int64_t row_base,
                int64_t r_begin, int64_t r_end, int64_t M, const double* what_new,
                const double* diag_new, const double* what_old, const double* diag_old,
                const double* d_sqrt, double* W, int64_t ldw, double* quad, double* norm2, double* vtd,
                void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = swb_stream(stream);
  StencilGeom g;
  int rc = make_geom(lat, &g);
  if (rc) return rc;
  const LatticeDev& L = g.lat;
  if (!V || M <= 0 || ldv < M || r_begin < row_base || r_end < r_begin) return SWB_INVALID_PARAM;
  if (r_begin % L.nx || r_end % L.nx) return SWB_INVALID_PARAM;  // whole x-lines
  if (r_end > L.nx * L.ny * L.nz) return SWB_INVALID_PARAM;
  const size_t need = swb_stencil_workspace_bytes(M);
  if (!ws || ws_bytes < need) return SWB_WORKSPACE_TOO_SMALL;
  const int n_cb = static_cast<int>((M + 31) / 32);
  const int64_t slot_ld = int64_t(n_cb) * 32;
  const int64_t grid = stencil_grid();
  const int64_t n_warps = grid * ST_WARPS;
  double* slots = static_cast<double*>(ws);
  SWB_CUDA_TRY(cudaMemsetAsync(slots, 0, sizeof(double) * n_warps * slot_ld * 3, st));
  const int64_t n_lines = (r_end - r_begin) / L.nx;
  if (n_lines > 0) {
    stencil_kernel<DELTA><<<static_cast<unsigned>(grid), ST_WARPS * 32, 0, st>>>(
        g, V, ldv, row_base, r_begin / L.nx, n_lines, M, n_cb, what_new, diag_new, what_old, diag_old,
        d_sqrt, W, ldw, r_begin, slots, slot_ld);
    SWB_CHECK_LAUNCH();
  }
  dim3 rg(static_cast<unsigned>(M), 3);
  slot_reduce_kernel<<<rg, 256, 0, st>>>(slots, slot_ld, n_warps, M, quad, norm2, vtd);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

__global__ void sumsq_partial_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    s += v[i] * v[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

__global__ void gather_columns_kernel(const double* __restrict__ src, int64_t lds, int64_t rows,
                                      const int32_t* __restrict__ col_map, int64_t m,
                                      double* __restrict__ dst, int64_t ldd) {
  const int64_t total = rows * m;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / m, j = e % m;
    dst[r * ldd + j] = src[r * lds + col_map[j]];
  }
}

}  // namespace

extern "C" int swb_num_directions(const swb_lattice* lat) {
  LatticeDev L;
  if (swb_make_lattice(lat, &L)) return -1;
  return L.ndir;
}

extern "C" int swb_graph_build(const swb_lattice* lat, const double* intensities, double beta,
                               const uint8_t* cut_mask, double* what, double* diag, double* d_sqrt,
                               int32_t* degenerate_flag, void* stream) {
  if (!(beta >= 0.0)) return SWB_INVALID_PARAM;  // graphs.py:130-131
  if (!intensities || !what || !diag || !d_sqrt || !degenerate_flag) return SWB_INVALID_PARAM;
  cudaStream_t st = swb_stream(stream);
  StencilGeom g;
  int rc = make_geom(lat, &g);
  if (rc) return rc;
  const int64_t N = g.lat.nx * g.lat.ny * g.lat.nz;
  const int grid = swb_sm_count() * 8;
  SWB_CUDA_TRY(cudaMemsetAsync(degenerate_flag, 0, sizeof(int32_t), st));
  edge_weight_kernel<<<grid, 256, 0, st>>>(g, intensities, beta, lat->weight_mode, cut_mask, what, N);
  SWB_CHECK_LAUNCH();
  degree_kernel<<<grid, 256, 0, st>>>(g, what, d_sqrt, diag, degenerate_flag, N);
  SWB_CHECK_LAUNCH();
  normalize_kernel<<<grid, 256, 0, st>>>(g, what, d_sqrt, N);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" size_t swb_stencil_workspace_bytes(int64_t M) {
  const int64_t n_cb = (M + 31) / 32;
  return sizeof(double) * size_t(stencil_grid() * ST_WARPS) * size_t(n_cb * 32) * 3;
}

extern "C" int swb_stencil_rayleigh(const swb_lattice* lat, const double* V, int64_t ldv,
                                    int64_t row_base, int64_t r_begin, int64_t r_end, int64_t M,
                                    const double* what, const double* diag, const double* d_sqrt,
                                    double* quad, double* norm2, double* vtd, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  if (!what || !diag || !d_sqrt) return SWB_INVALID_PARAM;
  return run_stencil<false>(lat, V, ldv, row_base, r_begin, r_end, M, what, diag, nullptr, nullptr,
                            d_sqrt, nullptr, 0, quad, norm2, vtd, workspace, workspace_bytes, stream);
}

extern "C" int swb_stencil_delta(const swb_lattice* lat, const double* V, int64_t ldv, int64_t row_base,
                                 int64_t r_begin, int64_t r_end, int64_t M, const double* what_old,
                                 const double* diag_old, const double* what_new, const double* diag_new,
                                 const double* d_sqrt_new, double* W, int64_t ldw, double* quad,
                                 double* norm2, double* vtd, void* workspace, size_t workspace_bytes,
                                 void* stream) {
  if (!what_old || !diag_old || !what_new || !diag_new || !d_sqrt_new || !W || ldw < M)
    return SWB_INVALID_PARAM;
  return run_stencil<true>(lat, V, ldv, row_base, r_begin, r_end, M, what_new, diag_new, what_old,
                           diag_old, d_sqrt_new, W, ldw, quad, norm2, vtd, workspace, workspace_bytes,
                           stream);
}

extern "C" int swb_sumsq(const double* v, int64_t n, double* out, void* workspace, size_t workspace_bytes,
                         void* stream) {
  const int parts = 256;
  if (!v || !out || n < 0) return SWB_INVALID_PARAM;
  if (!workspace || workspace_bytes < parts * sizeof(double)) return SWB_WORKSPACE_TOO_SMALL;
  cudaStream_t st = swb_stream(stream);
  double* part = static_cast<double*>(workspace);
  sumsq_partial_kernel<<<parts, 256, 0, st>>>(v, n, part);
  SWB_CHECK_LAUNCH();
  sum_parts_kernel<<<1, 256, 0, st>>>(part, parts, out);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_gather_columns(const double* src, int64_t lds, int64_t rows, const int32_t* col_map,
                                  int64_t m, double* dst, int64_t ldd, void* stream) {
  if (!src || !dst || !col_map || m <= 0 || rows < 0 || ldd < m) return SWB_INVALID_PARAM;
  if (rows == 0) return SWB_OK;
  cudaStream_t st = swb_stream(stream);
  gather_columns_kernel<<<swb_sm_count() * 8, 256, 0, st>>>(src, lds, rows, col_map, m, dst, ldd);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}
