/*
 * specwalk-b200 — C ABI of the B200 (sm_100a) online hot path of the
 * adaptable-precomputation random walker (arXiv 1607.04174).
 *
 * Every entry point is `extern "C"`, returns an int status (SWB_OK == 0),
 * takes plain device pointers, int64 extents and a cudaStream_t passed as
 * `void*`.  Nothing allocates: scratch comes from a caller-provided
 * workspace whose size is given by the matching *_workspace_bytes query.
 * Calls are stream-ordered and stateless; concurrent calls on different
 * streams with disjoint buffers are safe.  No C++ exception crosses the ABI.
 *
 * Layouts
 *   - Voxels are flat x-fastest indices x + nx*(y + ny*z)
 *     (reference pkg/src/specwalk/indexing.py:1-6).
 *   - The eigenbasis V is ROW-MAJOR N x M float64 with leading dimension
 *     ldv >= M (even), one row per voxel.  (The reference keeps V
 *     column-major, fastrw.py:243; row-major gives coalesced stencil and
 *     row-tile access on the GPU.)  `row_base` is the global voxel index of
 *     row 0 of the V pointer, so a z-slab shard with a one-plane halo passes
 *     V at its first halo row.
 *   - Stencil coefficients: what[x*ndir + d] = magnitude of the normalized
 *     Laplacian off-diagonal between voxel x and its forward neighbour in
 *     direction d (L^_{x,y} = -what), 0 for edges off the grid or cut;
 *     diag[x] = L^_{x,x}.
 *
 * Status codes map 1:1 onto the reference exception taxonomy
 * (pkg/src/specwalk/errors.py:1-76).
 */
#ifndef SPECWALK_B200_H
#define SPECWALK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWB_OK 0
#define SWB_INVALID_PARAM 1          /* errors.InvalidParam          */
#define SWB_INSUFFICIENT_BASIS 2     /* errors.InsufficientBasis     */
#define SWB_SINGULAR_SMALL_SYSTEM 3  /* errors.SingularSmallSystem   */
#define SWB_DEGENERATE_GRAPH 4       /* errors.DegenerateGraph       */
#define SWB_CUDA_ERROR 5             /* device / launch failure      */
#define SWB_WORKSPACE_TOO_SMALL 6    /* caller workspace too small   */
#define SWB_COMM_ERROR 7             /* NCCL failure / unavailable    */

/* Lattice description.  connectivity: 4 (2-D, reference), 8 (2-D,
 * BASELINE config-2 extension) or 6 (3-D, reference); nz == 1 in 2-D.
 * weight_mode: 0 = max(exp(-beta*|dI|), 1e-8) (reference graphs.py:134-136),
 * 1 = max(exp(-beta*dI^2), 1e-8) (BASELINE configs).
 * Forward directions d: 4-conn {+x,+y}; 6-conn {+x,+y,+z};
 * 8-conn {+x, +y, (+1,+1), (-1,+1)}. */
typedef struct swb_lattice {
  int64_t nx, ny, nz;
  int32_t connectivity;
  int32_t weight_mode;
} swb_lattice;

int swb_abi_version(void);
const char* swb_status_string(int status);
const char* swb_last_cuda_error(void);
int swb_num_directions(const swb_lattice* lat);
/* Number of kernels this library has launched in the process (bench
 * accounting: gpu_launches). */
unsigned long long swb_launch_count(void);

/* ---- graph (replaces graphs.py:127-140 build_graph + :143-159
 *      laplacian_from_weights, NORMALIZED mode) ------------------------ */
/* cut_mask (nullable): N*ndir bytes, nonzero = forward edge removed
 * (topology-change extension).  degenerate_flag: device int32, set to 1
 * when some degree <= 0 (DegenerateGraph); the caller reads it. */
int swb_graph_build(const swb_lattice* lat, const double* intensities, double beta,
                    const uint8_t* cut_mask, double* what, double* diag, double* d_sqrt,
                    int32_t* degenerate_flag, void* stream);

/* ---- stencil passes over V (refresh.py:75-77) ----------------------- */
/* rows [r_begin, r_end) (global voxel indices) are processed; neighbour rows
 * are read from V (which must hold them: halo planes for shards).
 * Outputs are per-column sums over the processed rows, written (not
 * accumulated) to quad/norm2/vtd (M each):
 *   quad_j = sum_x v_xj (L^ v_j)_x,  norm2_j = sum_x v_xj^2,
 *   vtd_j  = sum_x v_xj d_sqrt_x.
 * Deterministic (fixed reduction order). */
size_t swb_stencil_workspace_bytes(const swb_lattice* lat, int64_t M);
int swb_stencil_rayleigh(const swb_lattice* lat, const double* V, int64_t ldv, int64_t row_base,
                         int64_t r_begin, int64_t r_end, int64_t M,
                         const double* what, const double* diag, const double* d_sqrt,
                         double* quad, double* norm2, double* vtd,
                         void* workspace, size_t workspace_bytes, void* stream);
/* Same pass, also materialising W = (L^new - L^old) V for rows
 * [r_begin, r_end) into W (row r at W + (r - r_begin)*ldw);
 * quad uses L^new. */
int swb_stencil_delta(const swb_lattice* lat, const double* V, int64_t ldv, int64_t row_base,
                      int64_t r_begin, int64_t r_end, int64_t M,
                      const double* what_old, const double* diag_old,
                      const double* what_new, const double* diag_new, const double* d_sqrt_new,
                      double* W, int64_t ldw, double* quad, double* norm2, double* vtd,
                      void* workspace, size_t workspace_bytes, void* stream);

/* Apply pass (polynomial filters of the offline eigensolver):
 * out = a * (L^ V) + b * V + g * Z over rows [r_begin, r_end) (Z optional,
 * same row indexing as out: row r at out + (r - r_begin)*ldo); also
 * returns quad = diag(V^T L^ V) and norm2 = diag(V^T V) over those rows. */
int swb_stencil_apply(const swb_lattice* lat, const double* V, int64_t ldv, int64_t row_base,
                      int64_t r_begin, int64_t r_end, int64_t M, const double* what, const double* diag,
                      const double* d_sqrt, double a, double b, const double* Z, int64_t ldz, double g,
                      double* out, int64_t ldo, double* quad, double* norm2, void* workspace,
                      size_t workspace_bytes, void* stream);

/* ---- FP64 tensor-core (DMMA) GEMMs ---------------------------------- */
/* out[M1 x M2] = X^T Y, X rows x M1 (ldx), Y rows x M2 (ldy), reduction
 * over rows; symmetric != 0 computes the upper triangle blocks only and
 * mirrors (X == Y columns assumed to give a symmetric result).
 * Deterministic split-row reduction through the workspace. */
size_t swb_gemm_tn_workspace_bytes(int64_t rows, int64_t M1, int64_t M2);
int swb_gemm_tn(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t rows,
                int64_t M1, int64_t M2, int symmetric, double* out, int64_t ldo,
                void* workspace, size_t workspace_bytes, void* stream);
/* out[rows x M2] = A[rows x K] B[K x M2] (+ out when accumulate != 0).  A row-major (lda), B row-major (ldb), out (ldo);
 * out must not alias A. */
int swb_gemm_nn(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows,
                int64_t K, int64_t M2, double* out, int64_t ldo, int accumulate, void* stream);
/* out = alpha * A B (+ out when accumulate != 0) — e.g. the prior residual
 * update r -= V_new (V_new^T r) of adaptive.py:129. */
int swb_gemm_nn_ex(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows,
                   int64_t K, int64_t M2, double* out, int64_t ldo, int accumulate, double alpha,
                   void* stream);

/* out[rows x M2] = A[rows x K] B[K x M2] in FP64 on the INT8 tcgen05 tensor
 * cores (Ozaki split-integer scheme: 7 digits per operand, 28 digit products,
 * row / column power-of-two scaling; error ~2^-53 K max|A[r,:]| max|B[:,c]|).
 * K <= 512 (larger K: INVALID_PARAM; use swb_gemm_nn); the workspace holds the
 * digit planes of a row chunk. */
size_t swb_oz_gemm_nn_workspace_bytes(int64_t rows, int64_t K, int64_t M2);
int swb_oz_gemm_nn(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int64_t K,
                   int64_t M2, double* out, int64_t ldo, void* workspace, size_t workspace_bytes, void* stream);
/* The same with the product's columns [ncol_main, M2) written to out2 (ld
 * ldo2) instead of out (swb_update_and_solve's extra columns C coeff). */
int swb_oz_gemm_nn_split(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int64_t K,
                         int64_t M2, int64_t ncol_main, double* out, int64_t ldo, double* out2, int64_t ldo2,
                         void* workspace, size_t workspace_bytes, void* stream);
/* The same in parts (the host loop of swb_oz_gemm_nn, exposed so callers can
 * time the digit split and the GEMM separately): B's planes once, then per
 * row chunk of at most swb_oz_chunk_rows(rows, K, M2) rows the chunk's A
 * planes and the GEMM.  `rows` (total) sizes the workspace layout; when rows
 * exceed one chunk the workspace holds two A-plane buffers (buf 0 / 1) so the
 * split of chunk i+1 can run on another stream during the GEMM of chunk i
 * (what swb_oz_gemm_nn does). */
int64_t swb_oz_chunk_rows(int64_t rows, int64_t K, int64_t M2);
int swb_oz_split_cols(const double* B, int64_t ldb, int64_t rows, int64_t K, int64_t M2, void* workspace,
                      size_t workspace_bytes, void* stream);
int swb_oz_split_rows(const double* A_chunk, int64_t lda, int64_t chunk_rows, int64_t rows, int64_t K, int64_t M2,
                      int buf, void* workspace, size_t workspace_bytes, void* stream);
int swb_oz_gemm_planes(int64_t chunk_rows, int64_t rows, int64_t K, int64_t M2, int buf, double* out_chunk,
                       int64_t ldo, void* workspace, size_t workspace_bytes, void* stream);
/* The same GEMM with the product's columns split between two outputs:
 * [0, ncol_main) -> out_chunk (ldo), [ncol_main, M2) -> out2_chunk (ldo2).
 * Extra B columns appended after the K rotation columns ride in the last
 * column tile's padding (64-column tiles), so e.g. V (C coeff) -- the RW
 * solve's reconstruction V' coeff -- comes out of the rotation at no extra
 * tensor-core work (update_and_solve). */
int swb_oz_gemm_planes_split(int64_t chunk_rows, int64_t rows, int64_t K, int64_t M2, int buf, double* out_chunk,
                             int64_t ldo, int64_t ncol_main, double* out2_chunk, int64_t ldo2, void* workspace,
                             size_t workspace_bytes, void* stream);
/* The split-output GEMM that also records row_amax[r] = bits of
 * max_{c < ncol_main} |out[r, c]| (atomicMax; row_amax zeroed by the caller,
 * indexed from out_chunk's first row): the next rotation's row scales. */
int swb_oz_gemm_planes_ex(int64_t chunk_rows, int64_t rows, int64_t K, int64_t M2, int buf, double* out_chunk,
                          int64_t ldo, int64_t ncol_main, double* out2_chunk, int64_t ldo2,
                          unsigned long long* row_amax_chunk, void* workspace, size_t workspace_bytes, void* stream);
/* A workspace with one A-plane buffer per row chunk (buf 0 .. chunks-1: all
 * of A's planes resident, e.g. emitted by swb_gemm_tn_sym_emit), and the
 * plane geometry for such producers: info[5] = {chunk_rows, nkc, byte
 * offset of buffer 0's planes, bytes of a buffer's planes (its row scales
 * follow), byte stride between buffers}. */
size_t swb_oz_gemm_nn_workspace_bytes_full(int64_t rows, int64_t K, int64_t M2);
int swb_oz_layout_info(int64_t rows, int64_t K, int64_t M2, int64_t* info);
/* measurement: back-to-back INT8 tcgen05 MMAs (M 128, N 256, K 32) on every
 * SM; *ops_out = 2 x MACs issued (bench.py's live INT8 roofline) */
int swb_int8_peak_probe(int iters, double* ops_out, void* stream);
/* measurement: the rotation GEMM's MMA pattern alone (M 128, N 64, K 32, SS,
 * 28 MMAs per K chunk into seven TMEM accumulators) on every SM -- the
 * ceiling of the digit-product scheme; *ops_out = 2 x MACs issued */
int swb_int8_scheme_probe(int iters, double* ops_out, void* stream);
/* the two probes with a choice of operands: pattern 0 = the dense M128 N256
 * probe, 1 = the scheme probe; seed 0 = zero operands (burst figure), else
 * pseudo-random operand bytes (the data-dependent power of real operands:
 * run long enough, this is the sustained, power-capped figure) */
int swb_int8_probe_ex(int pattern, int iters, unsigned int seed, double* ops_out, void* stream);
/* diagnostics: the seven int32 digit-product group sums of the first row
 * chunk, raw[(g * rows_p + r) * np + c], rows_p / np padded to 128 / 64 */
int swb_oz_gemm_nn_raw(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int64_t K,
                       int64_t M2, int32_t* raw, void* workspace, size_t workspace_bytes, void* stream);

/* ---- eigen update coefficients (refresh.py:78-79 + first-order) ------ */
/* method 0 (rayleigh, reference refresh): lam_new = sort(max(quad/norm2,0)),
 *   order = stable argsort; C untouched.
 * method 1 (first_order): additionally C[M x M] (row-major, ldc) =
 *   Cfo[:, order] * s[order] with Cfo_ii = 1,
 *   Cfo_ji = P_ji/(lam_i - lam_j) if |P_ji| <= gap_guard*|lam_i-lam_j| else 0,
 *   s_i = 1/||Cfo[:, i]||.  P row-major (ldp), lam_old the stored values. */
int swb_update_coeffs(int method, const double* P, int64_t ldp, const double* lam_old,
                      const double* quad, const double* norm2, int64_t M, double gap_guard,
                      double* C, int64_t ldc, double* lam_new, int64_t* order, void* stream);

/* ---- reduced-basis RW solve (fastrw.py:352-467) ---------------------- */
/* Seed rows of L^ in ELL form (S x R, R = 2*ndir+1), from the stencil. */
int swb_seed_rows(const swb_lattice* lat, const double* what, const double* diag,
                  const int64_t* seed_idx, int64_t S, int64_t* ell_idx, double* ell_val,
                  void* stream);
/* Pass 1 seed projections (fastrw.py:405-422, 428, 445, 449);
 * q_s / b_qn rows have leading dimension ldq, lsu is S x L:
 *   q_s[i,j]   = V[s_i, col(j)]
 *   b_qn[i,j]  = sum_{y in row s_i, y not a seed} L^_{s_i,y} V[y, col(j)]
 *   bg[i]      = sum_{y in row s_i, y not a seed} L^_{s_i,y} g_y
 *   lsu[i,k]   = sum_{t seed in row s_i} L^_{s_i,s_t} [lab_t == k] d_sqrt_{s_t}
 *   dsq_s[i]   = d_sqrt[s_i]
 * col(j) = col_map ? col_map[j] : j; g = d_sqrt / dnorm (dnorm = ||d_sqrt||).
 * Rows not in [own_begin, own_end) contribute zero (z-slab shards).
 * PRECONDITION: seed_idx strictly ascending (sorted, unique), as
 * SeedPartition guarantees (graphs.py:51-98) -- seed membership is a binary
 * search; unsorted input gives wrong results.  swb_check_seeds validates it
 * on the device; swb_rw_solve calls it and returns SWB_INVALID_PARAM. */
int swb_seed_project(const double* V, int64_t ldv, int64_t row_base, int64_t own_begin,
                     int64_t own_end, int64_t m, const int32_t* col_map,
                     const int64_t* seed_idx, const int32_t* seed_lab, int64_t S,
                     const int64_t* ell_idx, const double* ell_val, int64_t R,
                     const double* d_sqrt, double dnorm, int64_t L, double* q_s,
                     int64_t ldq, double* b_qn, double* bg, double* lsu, double* dsq_s,
                     void* stream);
/* dgecon of A = I - Ut Vt^T (n x n; Ut, Vt n x r, ld ldr) from the LU of
 * K = I_r - Vt^T Ut (swb_lu_factor: K, pivots pk) via the Woodbury identity;
 * anorm = ||A||_1 (device).  The seed systems use it when r << n. */
size_t swb_gecon_wb_workspace_bytes(int64_t n, int64_t r);
int swb_gecon_wb(int64_t n, int64_t r, const double* Ut, const double* Vt, int64_t ldr, const double* K, int64_t ldk,
                 const int32_t* pk, const double* anorm, double* rcond_out, void* workspace, size_t workspace_bytes,
                 void* stream);
/* *out = ||A||_1 (device double; workspace n + 1 doubles) */
int swb_norm1(const double* A, int64_t n, int64_t lda, double* out, void* workspace, size_t workspace_bytes,
              void* stream);
/* *flag_out (device double) = 1.0 when seed_idx is not strictly ascending
 * or not in [0, n), or a label is not in [0, L); else 0.0 (stream-ordered). */
int swb_check_seeds(const int64_t* seed_idx, const int32_t* seed_lab, int64_t S, int64_t n, int64_t L,
                    double* flag_out, void* stream);
/* Dense seed system of fastrw.py:399-454 + LU/rcond/solve of :332-344.
 * Computes the spectral weights w from values (m; 1/(lam+gamma), or the
 * deflated 1/lam for lam > 1e-10 at gamma == 0), g_s = dsq_s/dnorm,
 * gq = vtg - q_s^T g_s (gamma == 0; vtg[j] = sum_x V[x,col(j)] g_x), builds
 * the (S+1)^2 bordered (gamma == 0) or S^2 system, factors and solves it and
 * returns coeff (m x L, ld L) and extra (L; gamma == 0).
 * q_s, b_qn: S x m (ld ldq, even); lsu: S x L; t_p: m x L (ld ldt, gamma > 0).
 * rcond_out: device double; swb_check_rcond maps it to
 * SWB_SINGULAR_SMALL_SYSTEM after the stream is synchronised. */
size_t swb_small_solve_workspace_bytes(int64_t S, int64_t m, int64_t L);
int swb_small_solve(double gamma, int64_t S, int64_t m, int64_t L, const double* q_s,
                    const double* b_qn, int64_t ldq, const double* bg, const double* lsu,
                    const double* dsq_s, double dnorm, const int32_t* seed_lab,
                    const double* values, const double* vtg, const double* t_p, int64_t ldt,
                    double* coeff, double* extra, double* rcond_out,
                    void* workspace, size_t workspace_bytes, void* stream);
/* Same, with the condition estimate enqueued on rcond_stream after
 * rcond_event (a cudaEvent_t) is recorded on stream, so it overlaps the
 * caller's next work (the reconstruction).  The caller must join
 * rcond_stream before reading rcond_out or reusing the workspace. */
int swb_small_solve_ex(double gamma, int64_t S, int64_t m, int64_t L, const double* q_s,
                       const double* b_qn, int64_t ldq, const double* bg, const double* lsu,
                       const double* dsq_s, double dnorm, const int32_t* seed_lab,
                       const double* values, const double* vtg, const double* t_p, int64_t ldt,
                       double* coeff, double* extra, double* rcond_out,
                       void* workspace, size_t workspace_bytes, void* stream,
                       void* rcond_stream, void* rcond_event);
int swb_check_rcond(double rcond);

/* Dense LU with partial pivoting, 1-norm rcond (Hager/Higham) and solve.
 * A is n x n row-major (lda); replaced by its LU factors. */
size_t swb_lu_workspace_bytes(int64_t n);
int swb_lu_factor(double* A, int64_t n, int64_t lda, int32_t* piv, double* anorm_out,
                  void* workspace, size_t workspace_bytes, void* stream);
int swb_lu_rcond(const double* LU, int64_t n, int64_t lda, const int32_t* piv,
                 const double* anorm, double* rcond_out, void* workspace,
                 size_t workspace_bytes, void* stream);
/* n <= 160 in one launch: anorm_out = ||A||_1, A <- its LU factors (piv),
 * B <- A^-1 B, and (rcond_out non-null) rcond_out = dgecon's estimate.
 * swb_small_solve uses it for seed systems of up to 160 unknowns, with
 * rcond_out null and swb_lu_rcond on its side stream. */
int swb_small_dense_solve(double* A, int64_t n, int64_t lda, int32_t* piv, double* B, int64_t nrhs, int64_t ldb,
                          double* anorm_out, double* rcond_out, void* stream);
size_t swb_lu_solve_workspace_bytes(int64_t n, int64_t nrhs);
int swb_lu_solve(const double* LU, int64_t n, int64_t lda, const int32_t* piv, double* B,
                 int64_t nrhs, int64_t ldb, void* workspace, size_t workspace_bytes, void* stream);

/* Pass 2 + finalize + hard labels (fastrw.py:456-466, solver.py:55-66,
 * images.py:128-130) for rows [r_begin, r_end):
 *   u = (V[x, :mr] coeff + g_x*extra) / d_sqrt_x, clip >= 0, dead row ->
 *   1/L, normalise; label = argmax (ties -> lowest), top2 = p1 - p2.
 * coeff is mr x L (ld L) in V-column space: a permuted / truncated basis
 * passes its coefficients through swb_scatter_rows first.  g = d_sqrt/dnorm.
 * Seed rows are then overwritten by swb_apply_seeds.  U (nullable for
 * L <= 8; required, ldu even, for more labels), labels (int32), top2
 * (nullable) are indexed by (r - r_begin). */
int swb_reconstruct_label(const double* V, int64_t ldv, int64_t row_base, int64_t r_begin,
                          int64_t r_end, int64_t mr, const double* coeff, const double* extra,
                          double dnorm, const double* d_sqrt, int64_t L, double* U, int64_t ldu,
                          int32_t* labels, double* top2, void* stream);
/* dst[j, :ncols] = src[row_map[j], :ncols], j < m. */
int swb_gather_rows(const double* src, int64_t lds, const int32_t* row_map, int64_t m,
                    int64_t ncols, double* dst, int64_t ldd, void* stream);
/* dst (mr x L, zeroed) row col_map[j] = src row j, j < m. */
int swb_scatter_rows(const double* src, int64_t m, int64_t L, const int32_t* col_map,
                     double* dst, int64_t mr, void* stream);
int swb_apply_seeds(const int64_t* seed_idx, const int32_t* seed_lab, int64_t S,
                    int64_t r_begin, int64_t r_end, int64_t L, double* U, int64_t ldu,
                    int32_t* labels, double* top2, void* stream);

/* ---- dynamic basis size (adaptive.py:72-185) ------------------------ */
/* f_out[t*K + k] = seed_fit(q_s[:, :steps[t]], u_k, bound) for every
 * scheduled prefix steps[t] <= max_step <= M and label k, where
 * q_s[i, j] = V[s_i, col(j)] (col_map nullable) and u_k = [lab == k] d_sqrt[s].
 * One Householder QR of q_s, then per step (in parallel) a one-sided Jacobi
 * SVD of R[:m, :m], the 1e-13 sigma_0 cutoff and the ridge bisection. */
size_t swb_seed_fit_workspace_bytes(int64_t S, int64_t M, int64_t K, int64_t n_steps);
int swb_seed_fit_schedule(const double* V, int64_t ldv, const int32_t* col_map,
                          const int64_t* seed_idx, const int32_t* seed_lab, int64_t S,
                          const double* d_sqrt, int64_t M, int64_t K, const int32_t* steps,
                          int64_t n_steps, int32_t max_step, double bound, double* f_out,
                          void* workspace, size_t workspace_bytes, void* stream);

/* P^_masked (fastrw.py:395-397): out[r] = priors[r] * d_sqrt[r] for rows
 * [row_begin, row_end) (out row 0 = row_begin), seed rows zeroed. */
int swb_prior_hat(const double* priors, int64_t ldp, int64_t row_begin, int64_t row_end,
                  int64_t L, const double* d_sqrt, const int64_t* seed_idx, int64_t S,
                  double* out, int64_t ldo, void* stream);
/* swb_gemm_tn (symmetric, P = X^T Y over rows) whose diagonal tiles also
 * emit the INT8 rotation's A digit planes of X into oz_workspace (sized by
 * swb_oz_gemm_nn_workspace_bytes_full(rows, M, M2), zero-filled by the caller
 * once), with row scales from row_amax (swb_oz_gemm_planes_ex of the rotation
 * that produced X): bit-identical to swb_oz_split_rows, which the rotation
 * then skips. */
int swb_gemm_tn_sym_emit(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t rows, int64_t M,
                         double* out, int64_t ldo, void* workspace, size_t workspace_bytes,
                         const unsigned long long* row_amax, int64_t M2, void* oz_workspace,
                         size_t oz_workspace_bytes, void* stream);
/* Finalize + hard labels of a reconstruction computed elsewhere: uraw
 * (rows [r_begin, r_end), ld ldr) holds V'[x, :] coeff; then exactly the
 * tail of swb_reconstruct_label: u = (uraw + g_x*extra)/d_sqrt_x, clip >= 0,
 * dead row -> 1/L, normalise, label / top2, U optional (L > 8: in place,
 * U == uraw).  d_sqrt is globally indexed; uraw / U / labels / top2 by
 * (r - r_begin).  Used by update_and_solve, whose rotation GEMM emits
 * V (C coeff) in its padding columns (swb_oz_gemm_planes_split). */
int swb_finalize_label(int64_t r_begin, int64_t r_end, int64_t L, const double* uraw, int64_t ldr,
                       const double* extra, double dnorm, const double* d_sqrt, double* U, int64_t ldu,
                       int32_t* labels, double* top2, void* stream);
/* hard_labels of an existing field (images.py:128-130). */
int swb_argmax_rows(const double* U, int64_t ldu, int64_t N, int64_t L, int32_t* labels,
                    double* top2, void* stream);

/* FP64 tensor-core peak probe: launches back-to-back DMMA.8x8x4 work on
 * every SM; *flops_out = flops of the launch (host value) for the caller to
 * divide by its event-timed duration.  sink: device double (never written
 * in practice). */
int swb_fp64_peak_probe(int iters, double* sink, double* flops_out, void* stream);

/* ---- registration data term (registration.py:95-129) ------------------ */
/* priors[x*ldp + k] = softmax_k(-(s_k(x)/sigma)^2), s_k = edge-clamped mean
 * |F - M shifted by disp_k| over the (2r+1)^d patch, sigma = max(mean_x
 * min_k s_k, 1e-8) (device double *sigma_out).  disp: K x 3 int32 (x, y, z). */
size_t swb_similarity_priors_workspace_bytes(int64_t N, int64_t K);
int swb_similarity_priors(const double* fixed, const double* moving, int64_t nx, int64_t ny, int64_t nz,
                          int32_t ndim, const int32_t* disp, int64_t K, int32_t patch_radius,
                          double* priors, int64_t ldp, double* sigma_out, void* workspace,
                          size_t workspace_bytes, void* stream);

/* ---- .rwpk pack ingest (fastrw.py:228-325) ----------------------------- */
/* Streaming XXH64 on the host (state: swb_xxh64_state_bytes() bytes). */
size_t swb_xxh64_state_bytes(void);
void swb_xxh64_init(void* state, uint64_t seed);
void swb_xxh64_update(void* state, const void* data, size_t len);
uint64_t swb_xxh64_digest(const void* state);
/* f32 column-major N x m eigenvector block (as stored in a pack) ->
 * row-major f64 device basis (ld >= m). */
int swb_f32_colmajor_to_f64_rowmajor(const float* src, int64_t n, int64_t m, double* dst, int64_t ld,
                                     void* stream);
/* same for an f64 column-major block (in-memory reference packs, Fortran V);
 * dst may point at a column offset of the basis (dst + c0, ld = ldv) so a
 * pack streams into the device basis block by block */
int swb_f64_colmajor_to_f64_rowmajor(const double* src, int64_t n, int64_t m, double* dst, int64_t ld,
                                     void* stream);
/* and back (save_pack): first m columns (through col_map if given). */
int swb_f64_rowmajor_to_f32_colmajor(const double* src, int64_t n, int64_t ld, int64_t m,
                                     const int32_t* col_map, float* dst, void* stream);

/* ---- offline eigensolver column kernels (fastrw.py:180-221,
 *      linalg.py:90-175); deterministic fixed-order reductions ------- */
size_t swb_column_workspace_bytes(int64_t k);
/* res2[j] = || Y[:, j] - theta[j] X[:, j] ||^2 over N rows */
int swb_ritz_residuals(const double* X, int64_t ldx, const double* Y, int64_t ldy, const double* theta,
                       int64_t N, int64_t k, double* res2, void* workspace, size_t workspace_bytes,
                       void* stream);
/* out[j] = a^T X[:, j]  (a == NULL: ||X[:, j]||^2) */
int swb_column_dots(const double* X, int64_t ldx, const double* a, int64_t N, int64_t k, double* out,
                    void* workspace, size_t workspace_bytes, void* stream);
/* out[j] = X[:, j]^T Y[:, j] */
int swb_column_products(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t N, int64_t k,
                        double* out, void* workspace, size_t workspace_bytes, void* stream);
/* X[:, j] = (X[:, j] - a * h[j]) * scale[j]   (a / scale optional) */
int swb_column_update(double* X, int64_t ldx, int64_t N, int64_t k, const double* a, const double* h,
                      const double* scale, void* stream);
/* flip columns so the largest-|.| entry (first on ties) is positive
 * (_canonical_signs, linalg.py:90-95) */
int swb_canonical_signs(double* X, int64_t ldx, int64_t N, int64_t k, void* workspace,
                        size_t workspace_bytes, void* stream);

/* ---- super-vertex aggregation (aggregation.py:89-216) ---------------- */
/* Greedy region growing (host buffers; sequential by definition):
 * priors N x L row-major (ldp), dims[ndim] x-fastest -> cluster_ids (N),
 * n_super. */
int swb_build_aggregation(const double* priors, int64_t ldp, int64_t L, const int64_t* dims, int32_t ndim,
                          int32_t max_cluster_radius, double similarity_tol, int32_t* cluster_ids,
                          int64_t* n_super);
/* delta[x] = 2 * #lattice neighbours of x in another cluster */
int swb_delta_weights(const swb_lattice* lat, const int32_t* cluster_ids, double* delta, void* stream);
/* out[c, :m] = sum_{x in c, ascending} (1/|c|) * (X[x, :m] * w[x])  (w optional);
 * order = voxels sorted by cluster (stable), offsets[n_super + 1] */
int swb_cluster_rows(const double* X, int64_t ldx, int64_t m, const double* w, const int64_t* order,
                     const int64_t* offsets, int64_t n_super, double* out, int64_t ldo, void* stream);
/* Y = A X for a CSR matrix A (nrows rows), CSR order */
int swb_csr_spmm(const int64_t* indptr, const int64_t* indices, const double* data, int64_t nrows,
                 const double* X, int64_t ldx, int64_t m, double* Y, int64_t ldy, void* stream);
/* raw lattice edge weights w[v * ndir + d] = max(exp(-beta |dI|), 1e-8)
 * (0 off-grid / cut) -- graphs.py:127-140 before normalisation */
int swb_edge_weights(const swb_lattice* lat, const double* intensities, double beta, const uint8_t* cut_mask,
                     double* w, void* stream);

/* ---- composite entry points (whole update / whole solve per call) ---- */
/* First-order update of SURVEY §7 for beta_old -> beta_new (and/or cut
 * masks): builds both graphs (graphs.py:127-159), the difference stencil,
 * the symmetric DMMA projection P, refresh eigenvalues + coefficients C and
 * the rotation V_out = V C (V_out distinct from V, same ldv; pad columns
 * zeroed).  Outputs: lambda_out / order_out (M), d_sqrt_out (N, new graph),
 * vtg_out (M, optional: V_out^T d_sqrt / ||d_sqrt||), dnorm_out (device
 * double, optional), degenerate_out (2 device ints, optional: nonzero ->
 * DegenerateGraph for the old / new graph, read after synchronising). */
size_t swb_update_workspace_bytes(const swb_lattice* lat, int64_t M);
int swb_update_first_order(const swb_lattice* lat, const double* image, double beta_old, double beta_new,
                           const uint8_t* cut_old, const uint8_t* cut_new, const double* V, int64_t ldv,
                           const double* lambda_old, int64_t M, double gap_guard, double* V_out,
                           double* lambda_out, int64_t* order_out, double* d_sqrt_out, double* vtg_out,
                           double* dnorm_out, int32_t* degenerate_out, void* workspace, size_t workspace_bytes,
                           void* stream);
/* Reduced-basis RW solve (fastrw.py:352-467 + solver.py:55-66 +
 * images.py:128-130) on a row-major basis V (ldv) with eigenvalues values
 * (M, ascending) and the graph's stencil coefficients (what, diag, d_sqrt):
 * gamma == 0 needs seeds and vtg (V^T d_sqrt / ||d_sqrt||, M); gamma > 0
 * needs priors (N x K, ld ldp).  Writes labels_out (N int32), top2_out and
 * U_out (optional for K <= 8, required with ldu even beyond).  Synchronous:
 * returns SWB_SINGULAR_SMALL_SYSTEM when rcond < 1e-14 (rcond_host gets it),
 * SWB_INVALID_PARAM when the seeds are not strictly ascending / in range. */
size_t swb_rw_solve_workspace_bytes(const swb_lattice* lat, int64_t M, int64_t m_use, int64_t S, int64_t K,
                                    int with_priors);
int swb_rw_solve(const swb_lattice* lat, const double* what, const double* diag, const double* d_sqrt,
                 const double* V, int64_t ldv, const double* values, const double* vtg, int64_t M, int64_t m_use,
                 const int64_t* seed_idx, const int32_t* seed_lab, int64_t S, int64_t K, double gamma,
                 const double* priors, int64_t ldp, int32_t* labels_out, double* top2_out, double* U_out,
                 int64_t ldu, double* rcond_host, void* workspace, size_t workspace_bytes, void* stream);

/* The first-order update (swb_update_first_order) and the gamma = 0 RW solve
 * on the updated basis (swb_rw_solve with m_use columns) in one call, with
 * one pass less over the basis (api.update_and_solve): the seed system is
 * solved before the rotation on the V' rows of the seeds' stencil
 * neighbourhoods formed as V[rows] C, and its coefficients ride as K extra
 * columns of C in the INT8 rotation (swb_oz_gemm_nn_split), whose products
 * V (C coeff) = V' coeff are finalized (swb_finalize_label) into labels_out /
 * top2_out / U_out (U_out optional for K <= 8).  V_out, lambda_out,
 * order_out, d_sqrt_out and vtg_out are swb_update_first_order's outputs.
 * Synchronous (two host reads): SWB_DEGENERATE_GRAPH, SWB_INVALID_PARAM for
 * unsorted / out-of-range seeds, SWB_SINGULAR_SMALL_SYSTEM (rcond_host). */
size_t swb_update_and_solve_workspace_bytes(const swb_lattice* lat, int64_t M, int64_t m_use, int64_t S, int64_t K,
                                            int64_t ldv);
int swb_update_and_solve(const swb_lattice* lat, const double* image, double beta_old, double beta_new,
                         const uint8_t* cut_old, const uint8_t* cut_new, const double* V, int64_t ldv,
                         const double* lambda_old, int64_t M, double gap_guard, double* V_out, double* lambda_out,
                         int64_t* order_out, double* d_sqrt_out, double* vtg_out, int64_t m_use,
                         const int64_t* seed_idx, const int32_t* seed_lab, int64_t S, int64_t K, int32_t* labels_out,
                         double* top2_out, double* U_out, int64_t ldu, double* rcond_host, void* workspace,
                         size_t workspace_bytes, void* stream);

/* Pieces of update_and_solve: the V rows of the seeds' stencil
 * neighbourhoods (S x R entries of swb_seed_rows' ell_idx, -1 -> the seed;
 * rows clamped into a buffer of global rows [row_base, row_base +
 * local_rows)) gathered into out (S R x ldv, pad columns zero) / scattered
 * back from src (columns < M); C_aug = [C | ccf | 0] (M x ldca). */
int swb_ell_rows_gather(const double* V, int64_t ldv, int64_t row_base, int64_t local_rows, const int64_t* ell_idx,
                        const int64_t* seed_idx, int64_t S, int64_t R, int64_t M, double* out, void* stream);
int swb_ell_rows_scatter(const double* src, int64_t ldv, int64_t row_base, int64_t local_rows, const int64_t* ell_idx,
                         const int64_t* seed_idx, int64_t S, int64_t R, int64_t M, double* V, void* stream);
int swb_build_caug(const double* C, int64_t ldp, const double* ccf, int64_t ldk, int64_t M, int64_t K, double* caug,
                   int64_t ldca, void* stream);

/* ---- small helpers used by the host layer --------------------------- */
/* out = sum_x v[x]^2 over n entries (deterministic). */
int swb_sumsq(const double* v, int64_t n, double* out, void* workspace,
              size_t workspace_bytes, void* stream);
/* dst[r, j] = src[r, col_map[j]] for j < m (column gather / permutation). */
int swb_gather_columns(const double* src, int64_t lds, int64_t rows, const int32_t* col_map,
                       int64_t m, double* dst, int64_t ldd, void* stream);

/* ---- NCCL communicator for the z-slab sharded path ----
 * One process per GPU.  Rank 0 makes a unique id, the host ships the 128
 * bytes to every rank (any channel), each rank calls swb_comm_init with its
 * device current.  NCCL is dlopen'ed on first use (the library links none);
 * failures return SWB_COMM_ERROR, text in swb_comm_last_error(). */
#define SWB_COMM_ID_BYTES 128
typedef struct swb_comm swb_comm;
const char* swb_comm_last_error(void);
int swb_comm_nccl_version(int* version);
int swb_comm_unique_id(uint8_t* id_out);
int swb_comm_init(const uint8_t* id, int nranks, int rank, swb_comm** out);
int swb_comm_destroy(swb_comm* comm);
int swb_comm_rank(const swb_comm* comm, int* rank, int* nranks);
/* recv = sum over ranks of send (count f64; in place when send == recv):
 * the update's (P, quad, norm2, V^T d, |d|^2) and the solve's (q_s, b_qn,
 * ...) partials.  Stream-ordered. */
int swb_comm_allreduce_f64(swb_comm* comm, const double* send, double* recv, int64_t count, void* stream);
/* One-plane halo exchange of a z-slab shard of V (row-major, ldv): the
 * buffer holds [lower halo plane if has_lo] [own_rows owned rows] [upper
 * halo plane if has_hi], a plane = unit_rows = nx*ny rows.  Sends the first
 * owned plane to rank-1 and the last to rank+1, receives the neighbours'
 * planes into the halos (one NCCL group).  Stream-ordered: run the interior
 * stencil on another stream to overlap it. */
int swb_comm_halo_exchange(swb_comm* comm, double* V, int64_t ldv, int64_t unit_rows, int64_t own_rows,
                           int has_lo, int has_hi, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPECWALK_B200_H */
