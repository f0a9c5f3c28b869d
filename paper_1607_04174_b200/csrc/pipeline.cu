// Composite entry points: the whole first-order update and the whole RW
// solve as single C calls, for hosts that bind the library directly (cgo /
// JNI / ctypes) instead of going through the Python layer.  They sequence the
// same ABI kernels in the same order as paper_1607_04174_b200/api.py
// (update_basis first-order branch; solve_fast), with caller-owned device
// buffers and one caller workspace carved into the pieces each step needs.
//
//   swb_update_first_order   graphs.py:127-159 (both betas) + the first-order
//                            update of SURVEY §7 (stencil, DMMA projection,
//                            refresh / coefficients refresh.py:75-79, rotation)
//   swb_rw_solve             fastrw.py:352-467 + solver.py:55-66 +
//                            images.py:128-130 (labels), with the reference's
//                            SingularSmallSystem check (fastrw.py:340)
//   swb_update_and_solve     the two in one call with one pass less over the
//                            basis (api.update_and_solve): seed system first,
//                            reconstruction as extra rotation columns
#include "swb_common.cuh"
#include <algorithm>
#include <cstdlib>

extern "C" size_t swb_oz_gemm_nn_workspace_bytes(int64_t rows, int64_t K, int64_t M2);
extern "C" int swb_oz_gemm_nn(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int64_t K,
                              int64_t M2, double* out, int64_t ldo, void* workspace, size_t workspace_bytes,
                              void* stream);

namespace {

struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    off = swb_align_up(off, 256);
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += sizeof(T) * count;
    return p;
  }
};

// vtg[j] = (sum_i vtd[i] C[i, j]) / ||d_sqrt||, dnorm from sum d_sqrt^2
__global__ void vtg_kernel(const double* __restrict__ vtd, const double* __restrict__ C, int64_t ldc, int64_t M,
                           const double* __restrict__ dsq_sum, double* __restrict__ vtg, double* __restrict__ dnorm) {
  const double dn = sqrt(*dsq_sum);
  if (blockIdx.x == 0 && threadIdx.x == 0 && dnorm) *dnorm = dn;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < M; j += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int64_t i = 0; i < M; ++i) s = fma(vtd[i], C[i * ldc + j], s);
    vtg[j] = s / dn;
  }
}

__global__ void zero_cols_kernel(double* __restrict__ V, int64_t ldv, int64_t N, int64_t M) {
  const int64_t w = ldv - M;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < N * w; e += int64_t(gridDim.x) * blockDim.x)
    V[(e / w) * ldv + M + e % w] = 0.0;
}

struct UpdateLayout {
  double *what_o, *diag_o, *dsq_o, *what_n, *diag_n, *quad, *norm2, *vtd, *P, *C, *dsum;
  int32_t* flag;
  void* st_ws;
  size_t st_bytes;
  void* tn_ws;
  size_t tn_bytes;
  void* ss_ws;
  void* oz_ws;
  size_t oz_bytes;
  size_t total;
};

// The rotation V' = V C runs on the INT8 tensor cores (ozaki.cu) when the
// basis has at most 512 columns; SWB_ROTATION=dmma selects the FP64 DMMA
// GEMM instead (measurement knob).
bool rotation_on_int8(int64_t M) {
  static const bool dmma = [] {
    const char* e = getenv("SWB_ROTATION");
    return e && e[0] == 'd';
  }();
  return !dmma && M <= 512;
}

UpdateLayout update_layout(const swb_lattice* lat, int64_t M, void* ws, bool rotation_ws = true) {
  LatticeDev L{};
  swb_make_lattice(lat, &L);
  const int64_t N = L.nx * L.ny * L.nz;
  const int64_t ldp = (M + 1) / 2 * 2;
  Carver c{static_cast<char*>(ws)};
  UpdateLayout u{};
  u.what_o = c.take<double>(size_t(N) * L.ndir);
  u.diag_o = c.take<double>(N);
  u.dsq_o = c.take<double>(N);
  u.what_n = c.take<double>(size_t(N) * L.ndir);
  u.diag_n = c.take<double>(N);
  u.quad = c.take<double>(M);
  u.norm2 = c.take<double>(M);
  u.vtd = c.take<double>(M);
  u.P = c.take<double>(size_t(M) * ldp);
  u.C = c.take<double>(size_t(M) * ldp);
  u.dsum = c.take<double>(1);
  u.flag = c.take<int32_t>(4);
  u.st_bytes = swb_stencil_workspace_bytes(lat, M);
  u.st_ws = c.take<char>(u.st_bytes);
  u.tn_bytes = swb_gemm_tn_workspace_bytes(N, M, M);
  u.tn_ws = c.take<char>(u.tn_bytes);
  u.ss_ws = c.take<char>(256 * 8);
  u.oz_bytes = rotation_ws && rotation_on_int8(M) ? swb_oz_gemm_nn_workspace_bytes(N, M, M) : 0;
  u.oz_ws = c.take<char>(u.oz_bytes);
  u.total = c.off + 256;
  return u;
}

}  // namespace

extern "C" size_t swb_update_workspace_bytes(const swb_lattice* lat, int64_t M) {
  LatticeDev L;
  if (swb_make_lattice(lat, &L) || M <= 0) return 0;
  return update_layout(lat, M, nullptr).total;
}

extern "C" int swb_update_first_order(const swb_lattice* lat, const double* image, double beta_old,
                                      double beta_new, const uint8_t* cut_old, const uint8_t* cut_new,
                                      const double* V, int64_t ldv, const double* lambda_old, int64_t M,
                                      double gap_guard, double* V_out, double* lambda_out, int64_t* order_out,
                                      double* d_sqrt_out, double* vtg_out, double* dnorm_out,
                                      int32_t* degenerate_out, void* workspace, size_t workspace_bytes,
                                      void* stream) {
  LatticeDev L;
  if (swb_make_lattice(lat, &L) || !image || !V || !V_out || V == V_out || !lambda_old || !lambda_out ||
      !order_out || !d_sqrt_out || M <= 0 || ldv < M || (ldv & 1))
    return SWB_INVALID_PARAM;
  if (!workspace || workspace_bytes < swb_update_workspace_bytes(lat, M)) return SWB_WORKSPACE_TOO_SMALL;
  cudaStream_t st = swb_stream(stream);
  const int64_t N = L.nx * L.ny * L.nz;
  const int64_t ldp = (M + 1) / 2 * 2;
  UpdateLayout u = update_layout(lat, M, workspace);
  int rc;
  if ((rc = swb_graph_build(lat, image, beta_old, cut_old, u.what_o, u.diag_o, u.dsq_o, u.flag, stream))) return rc;
  if ((rc = swb_graph_build(lat, image, beta_new, cut_new, u.what_n, u.diag_n, d_sqrt_out, u.flag + 1, stream)))
    return rc;
  if (degenerate_out) {
    SWB_CUDA_TRY(cudaMemcpyAsync(degenerate_out, u.flag, 2 * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  }
  // W = dL V in V_out's buffer (dead after the projection, then the rotation target)
  if ((rc = swb_stencil_delta(lat, V, ldv, 0, 0, N, M, u.what_o, u.diag_o, u.what_n, u.diag_n, d_sqrt_out, V_out,
                              ldv, u.quad, u.norm2, u.vtd, u.st_ws, u.st_bytes, stream)))
    return rc;
  if ((rc = swb_gemm_tn(V, ldv, V_out, ldv, N, M, M, 1, u.P, ldp, u.tn_ws, u.tn_bytes, stream))) return rc;
  if ((rc = swb_update_coeffs(1, u.P, ldp, lambda_old, u.quad, u.norm2, M, gap_guard, u.C, ldp, lambda_out, order_out,
                              stream)))
    return rc;
  if ((rc = swb_sumsq(d_sqrt_out, N, u.dsum, u.ss_ws, 256 * 8, stream))) return rc;
  if (vtg_out || dnorm_out) {
    double* vtg_tmp = vtg_out ? vtg_out : u.quad;   // quad is dead after the coefficients
    vtg_kernel<<<static_cast<unsigned>((M + 255) / 256), 256, 0, st>>>(u.vtd, u.C, ldp, M, u.dsum, vtg_tmp, dnorm_out);
    SWB_CHECK_LAUNCH();
  }
  if (u.oz_bytes) {
    if ((rc = swb_oz_gemm_nn(V, ldv, u.C, ldp, N, M, M, V_out, ldv, u.oz_ws, u.oz_bytes, stream))) return rc;
  } else {
    if ((rc = swb_gemm_nn(V, ldv, u.C, ldp, N, M, M, V_out, ldv, 0, stream))) return rc;
  }
  if (ldv > M) {
    zero_cols_kernel<<<swb_sm_count() * 4, 256, 0, st>>>(V_out, ldv, N, M);
    SWB_CHECK_LAUNCH();
  }
  return SWB_OK;
}

// ---------------------------------------------------------------------------
// whole solve
// ---------------------------------------------------------------------------
namespace {

struct SolveLayout {
  int64_t *ell_idx;
  double *ell_val, *q_s, *b_qn, *bg, *lsu, *dsq_s, *ph, *t_p, *coeff, *extra, *dsum;
  void *tn_ws, *ss_ws, *sum_ws;
  size_t tn_bytes, ss_bytes, total;
};

SolveLayout solve_layout(const LatticeDev& L, int64_t M, int64_t m_use, int64_t S, int64_t K, bool priors,
                         void* ws) {
  const int64_t N = L.nx * L.ny * L.nz;
  const int64_t R = 2 * L.ndir + 1;
  const int64_t sa = S > 0 ? S : 1;
  const int64_t ldq = (m_use + 1) / 2 * 2, ldt = (K + 1) / 2 * 2;
  Carver c{static_cast<char*>(ws)};
  SolveLayout s{};
  s.ell_idx = c.take<int64_t>(size_t(sa) * R);
  s.ell_val = c.take<double>(size_t(sa) * R);
  s.q_s = c.take<double>(size_t(sa) * ldq);
  s.b_qn = c.take<double>(size_t(sa) * ldq);
  s.bg = c.take<double>(sa);
  s.lsu = c.take<double>(size_t(sa) * K);
  s.dsq_s = c.take<double>(sa);
  s.ph = priors ? c.take<double>(size_t(N) * ldt) : nullptr;
  s.t_p = c.take<double>(size_t(m_use) * ldt);
  s.coeff = c.take<double>(size_t(m_use) * K);
  s.extra = c.take<double>(K);
  s.dsum = c.take<double>(3);   // ||d_sqrt||^2, rcond, seed-check flag
  s.tn_bytes = priors ? swb_gemm_tn_workspace_bytes(N, m_use, K) : 0;
  s.tn_ws = c.take<char>(s.tn_bytes);
  s.ss_bytes = swb_small_solve_workspace_bytes(S, m_use, K);
  s.ss_ws = c.take<char>(s.ss_bytes);
  s.sum_ws = c.take<char>(256 * 8);
  s.total = c.off + 256;
  return s;
}

}  // namespace

extern "C" size_t swb_rw_solve_workspace_bytes(const swb_lattice* lat, int64_t M, int64_t m_use, int64_t S,
                                               int64_t K, int with_priors) {
  LatticeDev L;
  if (swb_make_lattice(lat, &L) || M <= 0 || m_use <= 0 || m_use > M || S < 0 || K <= 0) return 0;
  return solve_layout(L, M, m_use, S, K, with_priors != 0, nullptr).total;
}

extern "C" int swb_rw_solve(const swb_lattice* lat, const double* what, const double* diag, const double* d_sqrt,
                            const double* V, int64_t ldv, const double* values, const double* vtg, int64_t M,
                            int64_t m_use, const int64_t* seed_idx, const int32_t* seed_lab, int64_t S, int64_t K,
                            double gamma, const double* priors, int64_t ldp, int32_t* labels_out, double* top2_out,
                            double* U_out, int64_t ldu, double* rcond_host, void* workspace, size_t workspace_bytes,
                            void* stream) {
  LatticeDev L;
  if (swb_make_lattice(lat, &L) || !what || !diag || !d_sqrt || !V || !values || !labels_out || M <= 0 ||
      m_use <= 0 || m_use > M || S < 0 || K <= 0 || !(gamma >= 0.0) || (S > 0 && (!seed_idx || !seed_lab)))
    return SWB_INVALID_PARAM;
  if (m_use < K) return SWB_INSUFFICIENT_BASIS;
  if (K > 8 && (!U_out || ldu < K || (ldu & 1))) return SWB_INVALID_PARAM;   // many labels: the field is needed
  if (gamma == 0.0 && (S == 0 || !vtg)) return SWB_INVALID_PARAM;
  if (gamma > 0.0 && (!priors || ldp < K)) return SWB_INVALID_PARAM;
  const bool with_priors = gamma > 0.0;
  if (!workspace || workspace_bytes < swb_rw_solve_workspace_bytes(lat, M, m_use, S, K, with_priors))
    return SWB_WORKSPACE_TOO_SMALL;
  cudaStream_t st = swb_stream(stream);
  const int64_t N = L.nx * L.ny * L.nz;
  const int64_t R = 2 * L.ndir + 1;
  const int64_t ldq = (m_use + 1) / 2 * 2, ldt = (K + 1) / 2 * 2;
  SolveLayout w = solve_layout(L, M, m_use, S, K, with_priors, workspace);
  int rc;
  // ||d_sqrt|| (a host scalar of the kernels below): one synchronous read
  if ((rc = swb_sumsq(d_sqrt, N, w.dsum, w.sum_ws, 256 * 8, stream))) return rc;
  // the seed kernels binary-search seed_idx: validate sorted / unique / in range
  if ((rc = swb_check_seeds(seed_idx, seed_lab, S, N, K, w.dsum + 2, stream))) return rc;
  double hs[3] = {0.0, 0.0, 0.0};
  SWB_CUDA_TRY(cudaMemcpyAsync(hs, w.dsum, sizeof(hs), cudaMemcpyDeviceToHost, st));
  SWB_CUDA_TRY(cudaStreamSynchronize(st));
  if (hs[2] != 0.0) return SWB_INVALID_PARAM;
  const double dnorm = sqrt(hs[0]);
  if (S > 0) {
    if ((rc = swb_seed_rows(lat, what, diag, seed_idx, S, w.ell_idx, w.ell_val, stream))) return rc;
    if ((rc = swb_seed_project(V, ldv, 0, 0, N, m_use, nullptr, seed_idx, seed_lab, S, w.ell_idx, w.ell_val, R,
                               d_sqrt, dnorm, K, w.q_s, ldq, w.b_qn, w.bg, w.lsu, w.dsq_s, stream)))
      return rc;
  }
  const double* t_p = nullptr;
  if (with_priors) {
    if ((rc = swb_prior_hat(priors, ldp, 0, N, K, d_sqrt, seed_idx, S, w.ph, ldt, stream))) return rc;
    if ((rc = swb_gemm_tn(V, ldv, w.ph, ldt, N, m_use, K, 0, w.t_p, ldt, w.tn_ws, w.tn_bytes, stream))) return rc;
    t_p = w.t_p;
  }
  double* rcond_dev = w.dsum + 1;
  if ((rc = swb_small_solve(gamma, S, m_use, K, w.q_s, w.b_qn, ldq, w.bg, w.lsu, w.dsq_s, dnorm, seed_lab, values,
                            with_priors ? nullptr : vtg, t_p, ldt, w.coeff, with_priors ? nullptr : w.extra, rcond_dev,
                            w.ss_ws, w.ss_bytes, stream)))
    return rc;
  if ((rc = swb_reconstruct_label(V, ldv, 0, 0, N, m_use, w.coeff, with_priors ? nullptr : w.extra, dnorm, d_sqrt, K,
                                  U_out, ldu, labels_out, top2_out, stream)))
    return rc;
  if ((rc = swb_apply_seeds(seed_idx, seed_lab, S, 0, N, K, U_out, ldu, labels_out, top2_out, stream))) return rc;
  double rc_h = 0.0;
  SWB_CUDA_TRY(cudaMemcpyAsync(&rc_h, rcond_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
  SWB_CUDA_TRY(cudaStreamSynchronize(st));
  if (rcond_host) *rcond_host = rc_h;
  return swb_check_rcond(rc_h);
}

// ---------------------------------------------------------------------------
// update + solve in one pass over the basis (api.update_and_solve)
// ---------------------------------------------------------------------------
extern "C" int swb_oz_gemm_nn_split(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows,
                                    int64_t K, int64_t M2, int64_t ncol_main, double* out, int64_t ldo, double* out2,
                                    int64_t ldo2, void* workspace, size_t workspace_bytes, void* stream);

namespace {

// row e = s R + t of the seed stencil neighbourhoods: ell_idx[e], or the seed
// itself for an off-grid (-1) entry
__device__ __forceinline__ int64_t ell_row(const int64_t* ell_idx, const int64_t* seed_idx, int64_t e, int64_t R) {
  const int64_t r = ell_idx[e];
  return r >= 0 ? r : seed_idx[e / R];
}

// local row of entry e in a buffer holding global rows [row_base, row_base +
// local_rows) (a slab shard: rows outside are clamped in, every write then
// stores that local row's correct value)
__device__ __forceinline__ int64_t ell_local(const int64_t* ell_idx, const int64_t* seed_idx, int64_t e, int64_t R,
                                             int64_t row_base, int64_t local_rows) {
  const int64_t y = ell_row(ell_idx, seed_idx, e, R) - row_base;
  return y < 0 ? 0 : (y >= local_rows ? local_rows - 1 : y);
}

__global__ void gather_ell_rows_kernel(const double* __restrict__ V, int64_t ldv, int64_t row_base, int64_t local_rows,
                                       const int64_t* __restrict__ ell_idx, const int64_t* __restrict__ seed_idx,
                                       int64_t E, int64_t R, int64_t M, double* __restrict__ out) {
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    const double* src = V + ell_local(ell_idx, seed_idx, e, R, row_base, local_rows) * ldv;
    for (int64_t j = threadIdx.x; j < ldv; j += blockDim.x) out[e * ldv + j] = j < M ? src[j] : 0.0;
  }
}

// identical rows may appear several times: every writer stores the same values
__global__ void scatter_ell_rows_kernel(const double* __restrict__ src, int64_t ldv, int64_t row_base,
                                        int64_t local_rows, const int64_t* __restrict__ ell_idx,
                                        const int64_t* __restrict__ seed_idx, int64_t E, int64_t R, int64_t M,
                                        double* __restrict__ V) {
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    double* dst = V + ell_local(ell_idx, seed_idx, e, R, row_base, local_rows) * ldv;
    for (int64_t j = threadIdx.x; j < M; j += blockDim.x) dst[j] = src[e * ldv + j];
  }
}

// C_aug[i, :] = [C[i, :M] | ccf[i, :K] | 0]
__global__ void aug_kernel(const double* __restrict__ C, int64_t ldp, const double* __restrict__ ccf, int64_t ldk,
                           int64_t M, int64_t K, double* __restrict__ caug, int64_t ldca) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < M * ldca; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / ldca, j = e % ldca;
    caug[e] = j < M ? C[i * ldp + j] : (j < M + K ? ccf[i * ldk + (j - M)] : 0.0);
  }
}

struct FusedLayout {
  UpdateLayout u;
  SolveLayout s;
  double *rows_v, *rows_vp, *ccf, *caug, *uraw, *dnorm;
  void* oz_ws;
  size_t oz_bytes, total;
};

FusedLayout fused_layout(const swb_lattice* lat, int64_t M, int64_t m_use, int64_t S, int64_t K, int64_t ldv,
                         void* ws) {
  LatticeDev L{};
  swb_make_lattice(lat, &L);
  const int64_t N = L.nx * L.ny * L.nz;
  const int64_t R = 2 * L.ndir + 1;
  FusedLayout f{};
  f.u = update_layout(lat, M, ws, false);   // the split-output rotation below has its own workspace
  char* base = ws ? static_cast<char*>(ws) + f.u.total : nullptr;
  f.s = solve_layout(L, M, m_use, S, K, false, base);
  Carver c{base ? base + f.s.total : nullptr};
  const int64_t ldca = (M + K + 1) / 2 * 2, ldk = (K + 1) / 2 * 2;
  f.rows_v = c.take<double>(size_t(S) * R * ldv);
  f.rows_vp = c.take<double>(size_t(S) * R * ldv);
  f.ccf = c.take<double>(size_t(M) * ldk);
  f.caug = c.take<double>(size_t(M) * ldca);
  f.uraw = c.take<double>(size_t(N) * ldk);
  f.dnorm = c.take<double>(1);
  f.oz_bytes = rotation_on_int8(M) ? swb_oz_gemm_nn_workspace_bytes(N, M, M + K) : 0;
  f.oz_ws = c.take<char>(f.oz_bytes);
  f.total = f.u.total + f.s.total + c.off + 256;
  return f;
}

}  // namespace

extern "C" size_t swb_update_and_solve_workspace_bytes(const swb_lattice* lat, int64_t M, int64_t m_use, int64_t S,
                                                       int64_t K, int64_t ldv) {
  LatticeDev L;
  if (swb_make_lattice(lat, &L) || M <= 0 || m_use <= 0 || m_use > M || S <= 0 || K <= 0 || ldv < M) return 0;
  return fused_layout(lat, M, m_use, S, K, ldv, nullptr).total;
}

extern "C" int swb_update_and_solve(const swb_lattice* lat, const double* image, double beta_old, double beta_new,
                                    const uint8_t* cut_old, const uint8_t* cut_new, const double* V, int64_t ldv,
                                    const double* lambda_old, int64_t M, double gap_guard, double* V_out,
                                    double* lambda_out, int64_t* order_out, double* d_sqrt_out, double* vtg_out,
                                    int64_t m_use, const int64_t* seed_idx, const int32_t* seed_lab, int64_t S,
                                    int64_t K, int32_t* labels_out, double* top2_out, double* U_out, int64_t ldu,
                                    double* rcond_host, void* workspace, size_t workspace_bytes, void* stream) {
  LatticeDev L;
  if (swb_make_lattice(lat, &L) || !image || !V || !V_out || V == V_out || !lambda_old || !lambda_out ||
      !order_out || !d_sqrt_out || !vtg_out || M <= 0 || ldv < M || (ldv & 1) || m_use <= 0 || m_use > M || S <= 0 ||
      K <= 0 || !seed_idx || !seed_lab || !labels_out)
    return SWB_INVALID_PARAM;
  if (m_use < K) return SWB_INSUFFICIENT_BASIS;
  if (K > 8 && (!U_out || ldu < K || (ldu & 1))) return SWB_INVALID_PARAM;
  if (!workspace || workspace_bytes < swb_update_and_solve_workspace_bytes(lat, M, m_use, S, K, ldv))
    return SWB_WORKSPACE_TOO_SMALL;
  cudaStream_t st = swb_stream(stream);
  const int64_t N = L.nx * L.ny * L.nz;
  const int64_t R = 2 * L.ndir + 1, E = S * R;
  const int64_t ldp = (M + 1) / 2 * 2, ldq = (m_use + 1) / 2 * 2, ldt = (K + 1) / 2 * 2;
  const int64_t ldca = (M + K + 1) / 2 * 2, ldk = (K + 1) / 2 * 2;
  FusedLayout f = fused_layout(lat, M, m_use, S, K, ldv, workspace);
  const UpdateLayout& u = f.u;
  const SolveLayout& w = f.s;
  int rc;
  // ---- the update up to the rotation (swb_update_first_order's sequence) ----
  if ((rc = swb_graph_build(lat, image, beta_old, cut_old, u.what_o, u.diag_o, u.dsq_o, u.flag, stream))) return rc;
  if ((rc = swb_graph_build(lat, image, beta_new, cut_new, u.what_n, u.diag_n, d_sqrt_out, u.flag + 1, stream)))
    return rc;
  if ((rc = swb_stencil_delta(lat, V, ldv, 0, 0, N, M, u.what_o, u.diag_o, u.what_n, u.diag_n, d_sqrt_out, V_out,
                              ldv, u.quad, u.norm2, u.vtd, u.st_ws, u.st_bytes, stream)))
    return rc;
  if ((rc = swb_gemm_tn(V, ldv, V_out, ldv, N, M, M, 1, u.P, ldp, u.tn_ws, u.tn_bytes, stream))) return rc;
  if ((rc = swb_update_coeffs(1, u.P, ldp, lambda_old, u.quad, u.norm2, M, gap_guard, u.C, ldp, lambda_out, order_out,
                              stream)))
    return rc;
  if ((rc = swb_sumsq(d_sqrt_out, N, u.dsum, u.ss_ws, 256 * 8, stream))) return rc;
  vtg_kernel<<<static_cast<unsigned>((M + 255) / 256), 256, 0, st>>>(u.vtd, u.C, ldp, M, u.dsum, vtg_out, f.dnorm);
  SWB_CHECK_LAUNCH();
  if (ldv > M) {   // V' pad columns (the seed-row scatter and the rotation write [0, M) only)
    zero_cols_kernel<<<swb_sm_count() * 4, 256, 0, st>>>(V_out, ldv, N, M);
    SWB_CHECK_LAUNCH();
  }
  // host scalars: ||d_sqrt||, the degenerate-graph flags, seed validity
  if ((rc = swb_check_seeds(seed_idx, seed_lab, S, N, K, w.dsum + 2, stream))) return rc;
  double hs[2] = {0.0, 0.0};
  int32_t hf[2] = {0, 0};
  SWB_CUDA_TRY(cudaMemcpyAsync(hs, f.dnorm, sizeof(double), cudaMemcpyDeviceToHost, st));
  SWB_CUDA_TRY(cudaMemcpyAsync(hs + 1, w.dsum + 2, sizeof(double), cudaMemcpyDeviceToHost, st));
  SWB_CUDA_TRY(cudaMemcpyAsync(hf, u.flag, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SWB_CUDA_TRY(cudaStreamSynchronize(st));
  if (hf[0] || hf[1]) return SWB_DEGENERATE_GRAPH;
  if (hs[1] != 0.0) return SWB_INVALID_PARAM;
  const double dnorm = hs[0];
  // ---- the seed system on V' rows formed as V[rows] C ----
  if ((rc = swb_seed_rows(lat, u.what_n, u.diag_n, seed_idx, S, w.ell_idx, w.ell_val, stream))) return rc;
  const unsigned eg = static_cast<unsigned>(E < 65535 ? E : 65535);
  gather_ell_rows_kernel<<<eg, 128, 0, st>>>(V, ldv, 0, N, w.ell_idx, seed_idx, E, R, M, f.rows_v);
  SWB_CHECK_LAUNCH();
  if ((rc = swb_gemm_nn(f.rows_v, ldv, u.C, ldp, E, M, M, f.rows_vp, ldv, 0, stream))) return rc;
  scatter_ell_rows_kernel<<<eg, 128, 0, st>>>(f.rows_vp, ldv, 0, N, w.ell_idx, seed_idx, E, R, M, V_out);
  SWB_CHECK_LAUNCH();
  if ((rc = swb_seed_project(V_out, ldv, 0, 0, N, m_use, nullptr, seed_idx, seed_lab, S, w.ell_idx, w.ell_val, R,
                             d_sqrt_out, dnorm, K, w.q_s, ldq, w.b_qn, w.bg, w.lsu, w.dsq_s, stream)))
    return rc;
  double* rcond_dev = w.dsum + 1;
  if ((rc = swb_small_solve(0.0, S, m_use, K, w.q_s, w.b_qn, ldq, w.bg, w.lsu, w.dsq_s, dnorm, seed_lab, lambda_out,
                            vtg_out, nullptr, ldt, w.coeff, w.extra, rcond_dev, w.ss_ws, w.ss_bytes, stream)))
    return rc;
  // ---- C_aug = [C | C[:, :m_use] coeff]; the rotation emits V' and V' coeff ----
  if ((rc = swb_gemm_nn(u.C, ldp, w.coeff, K, M, m_use, K, f.ccf, ldk, 0, stream))) return rc;
  aug_kernel<<<swb_sm_count() * 4, 256, 0, st>>>(u.C, ldp, f.ccf, ldk, M, K, f.caug, ldca);
  SWB_CHECK_LAUNCH();
  if (f.oz_bytes) {
    if ((rc = swb_oz_gemm_nn_split(V, ldv, f.caug, ldca, N, M, M + K, M, V_out, ldv, f.uraw, ldk, f.oz_ws,
                                   f.oz_bytes, stream)))
      return rc;
  } else {
    if ((rc = swb_gemm_nn(V, ldv, u.C, ldp, N, M, M, V_out, ldv, 0, stream))) return rc;
    if ((rc = swb_gemm_nn(V, ldv, f.ccf, ldk, N, M, K, f.uraw, ldk, 0, stream))) return rc;
  }
  // ---- finalize + argmax + seeds ----
  if (K > 8) {   // the many-label finalize works in place in U
    SWB_CUDA_TRY(cudaMemcpy2DAsync(U_out, ldu * sizeof(double), f.uraw, ldk * sizeof(double), K * sizeof(double), N,
                                   cudaMemcpyDeviceToDevice, st));
    if ((rc = swb_finalize_label(0, N, K, U_out, ldu, w.extra, dnorm, d_sqrt_out, U_out, ldu, labels_out, top2_out,
                                 stream)))
      return rc;
  } else if ((rc = swb_finalize_label(0, N, K, f.uraw, ldk, w.extra, dnorm, d_sqrt_out, U_out, ldu, labels_out,
                                      top2_out, stream))) {
    return rc;
  }
  if ((rc = swb_apply_seeds(seed_idx, seed_lab, S, 0, N, K, U_out, ldu, labels_out, top2_out, stream))) return rc;
  double rc_h = 0.0;
  SWB_CUDA_TRY(cudaMemcpyAsync(&rc_h, rcond_dev, sizeof(double), cudaMemcpyDeviceToHost, st));
  SWB_CUDA_TRY(cudaStreamSynchronize(st));
  if (rcond_host) *rcond_host = rc_h;
  return swb_check_rcond(rc_h);
}

// ---------------------------------------------------------------------------
// pieces of update_and_solve for the host layer (one launch each)
// ---------------------------------------------------------------------------
extern "C" int swb_ell_rows_gather(const double* V, int64_t ldv, int64_t row_base, int64_t local_rows,
                                   const int64_t* ell_idx, const int64_t* seed_idx, int64_t S, int64_t R, int64_t M,
                                   double* out, void* stream) {
  if (!V || !ell_idx || !seed_idx || !out || S < 0 || R <= 0 || M <= 0 || ldv < M || local_rows <= 0)
    return SWB_INVALID_PARAM;
  const int64_t E = S * R;
  if (E == 0) return SWB_OK;
  gather_ell_rows_kernel<<<static_cast<unsigned>(E < 65535 ? E : 65535), 128, 0, swb_stream(stream)>>>(
      V, ldv, row_base, local_rows, ell_idx, seed_idx, E, R, M, out);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_ell_rows_scatter(const double* src, int64_t ldv, int64_t row_base, int64_t local_rows,
                                    const int64_t* ell_idx, const int64_t* seed_idx, int64_t S, int64_t R, int64_t M,
                                    double* V, void* stream) {
  if (!V || !ell_idx || !seed_idx || !src || S < 0 || R <= 0 || M <= 0 || ldv < M || local_rows <= 0)
    return SWB_INVALID_PARAM;
  const int64_t E = S * R;
  if (E == 0) return SWB_OK;
  scatter_ell_rows_kernel<<<static_cast<unsigned>(E < 65535 ? E : 65535), 128, 0, swb_stream(stream)>>>(
      src, ldv, row_base, local_rows, ell_idx, seed_idx, E, R, M, V);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_build_caug(const double* C, int64_t ldp, const double* ccf, int64_t ldk, int64_t M, int64_t K,
                              double* caug, int64_t ldca, void* stream) {
  if (!C || !ccf || !caug || M <= 0 || K <= 0 || ldp < M || ldk < K || ldca < M + K) return SWB_INVALID_PARAM;
  const int64_t total = M * ldca;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, int64_t(swb_sm_count()) * 8));
  aug_kernel<<<grid, 256, 0, swb_stream(stream)>>>(C, ldp, ccf, ldk, M, K, caug, ldca);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}
