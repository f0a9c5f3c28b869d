// FP64 GEMM on the INT8 tcgen05 tensor cores (Ozaki scheme, split-integer
// form) for the rotation V' = V * C of the first-order update.
//
// sm_100a has no FP64 kind for tcgen05.mma; its FP64 tensor path is the
// warp-level DMMA (dgemm.cu, ~37 TFLOP/s measured).  The INT8 kind runs at
// 4.5 POPS dense, and an FP64 product can be assembled exactly from INT8
// products:
//
//   row r of A is scaled by 2^-e_r (e_r = frexp exponent of max_k |A[r,k]|),
//   so x = A[r,k] 2^-e_r is in (-1, 1); X = rint(x 2^54) (|X| <= 2^54) is
//   split into S = 7 balanced base-256 digits
//       X = d_0 2^48 + d_1 2^40 + ... + d_6 2^0,  d_1..d_6 in [-128, 127],
//   d_0 in [-65, 65] (all signed int8); the columns of B the same way with
//   exponents f_c.  Then
//       sum_k A[r,k] B[k,c] ~= 2^(e_r + f_c - 12) sum_g acc_g 2^(-8 g),
//       acc_g = sum_{i+j=g} sum_k d_i[r,k] d'_j[k,c]   (g = 0..6, 28 pairs)
//   with every acc_g an exact int32 (|acc_g| <= 7 * 128^2 * K < 2^31 for
//   K <= 512 here).  The dropped pairs (i + j > 6, zero-mean balanced digits)
//   and the rounding of X bound the error by ~2^-53 * K * max|A[r,:]| *
//   max|B[:,c]| in the worst case -- the FP64 GEMM error model with row /
//   column maxima in place of element magnitudes -- and by ~2^-53 *
//   sqrt(K) * ... for unbiased data.
//
// Layout: the slice kernels write the digits pre-tiled in the tcgen05
// no-swizzle K-major core-matrix layout, one contiguous block per
// (row block, K chunk) stage, so the GEMM's producer is two 1-D bulk copies
// (cp.async.bulk + mbarrier transaction count) per stage.  The GEMM is a
// persistent warp-specialised kernel: warp 0 copies, warp 1 allocates TMEM
// and one lane issues the 28 MMAs per K chunk (M = 128, N = 64, K = 32) into
// seven int32 TMEM accumulators (7 x 64 of the 512 columns), warps 2..5
// drain TMEM, combine the groups in FP64 (Horner in 2^-8) and store.
#include <mutex>

#include "swb_common.cuh"
#include "oz_digits.cuh"

namespace {

constexpr int OZ_G = 7;                 // product groups g = i + j <= 6
constexpr int OZ_BN = 64;               // columns per tile (MMA N)
#ifndef OZ_STAGES_CFG
#define OZ_STAGES_CFG 4
#endif
constexpr int OZ_STAGES = OZ_STAGES_CFG;
constexpr int OZ_B_SLICE = OZ_BN * OZ_KC;            // 2048 B: [kq 2][col 64][16 B]
constexpr int OZ_B_STAGE = OZ_S * OZ_B_SLICE;        // 14 KB
constexpr int OZ_STAGE = OZ_A_STAGE + OZ_B_STAGE;
constexpr int OZ_EPI_WARPS = 8;
constexpr int OZ_EPI_COLS = OZ_BN / 2;              // columns per epilogue thread (two rounds of 16)
constexpr int OZ_THREADS = (2 + OZ_EPI_WARPS) * 32;
constexpr size_t OZ_SMEM = size_t(OZ_STAGES) * OZ_STAGE + 1024;
constexpr int OZ_TMEM_COLS = 512;
constexpr int OZ_MAX_K = 512;

// Wide MMAs (OZ_WIDE = 1): the B stage holds the seven digit planes of a
// column block side by side in N ([kq 2][plane 7][col 64][16 B]), so the
// digits E_0 .. E_(6-i) that A digit i meets are ONE contiguous 64 (7 - i)-
// column operand, and the group accumulators sit at TMEM column 64 g in the
// same order: A digit i times B columns [64 (g0 - i), 64 (g0 - i + n)) lands
// exactly on groups g0 .. g0 + n - 1.  The 28 digit products of a K chunk
// become 10 MMAs of N = 64..256 (the same int32 sums, bit for bit), which
// read the A digit once per MMA instead of once per group: at N = 64 every
// MMA re-read 4 KB of A for 2 KB of B and the shared-memory port (128 B per
// cycle) capped the rate; now A is read 10 times per chunk, not 28.
// OZ_WIDE = 0 keeps the 28 N = 64 MMAs ([plane 7][kq 2][col 64][16 B]).
#ifndef OZ_WIDE
#define OZ_WIDE 1
#endif
#if OZ_WIDE
constexpr uint32_t OZ_B_LBO = OZ_S * OZ_BN * 16;    // K-adjacent core matrices: past all 7 planes
constexpr uint32_t OZ_B_PLANE = OZ_BN * 16;         // plane j's columns follow plane j-1's
// A ragged last column block with <= 32 live columns (K = 400: 16, plus the
// solve's extra columns in update_and_solve) runs as a narrow 128 x 32 tile:
// planes of 32 columns side by side ([kq 2][plane 7][col 32][16 B], 7 KB per
// stage), groups at TMEM column 32 g, one MMA per A digit (N = 32 (7 - i)):
// half the MMA work and two thirds of the shared-memory traffic of a full
// tile whose last 48 columns are padding.
constexpr int OZ_BN_N = 32;
constexpr uint32_t OZ_B_LBO_N = OZ_S * OZ_BN_N * 16;
constexpr uint32_t OZ_B_PLANE_N = OZ_BN_N * 16;
constexpr int OZ_B_STAGE_N = OZ_S * OZ_BN_N * OZ_KC;   // 7 KB
#else
constexpr uint32_t OZ_B_LBO = OZ_BN * 16;
constexpr uint32_t OZ_B_PLANE = OZ_B_SLICE;
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "OZ_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra OZ_DONE;\n\t"
      "bra OZ_WAIT;\n\t"
      "OZ_DONE:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// shared-memory matrix descriptor, no swizzle, K-major core matrices
// (8 rows x 16 B): lbo = byte stride between the K-adjacent core matrices,
// sbo = byte stride between 8-row groups
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;  // descriptor version (sm_100)
  return d;
}

// instruction descriptor: kind::i8, s32 accumulate, K-major A and B, M x N
__host__ __device__ constexpr uint32_t idesc_i8(int a_signed, int b_signed, int n = OZ_BN) {
  return (2u << 4) | (uint32_t(a_signed) << 7) | (uint32_t(b_signed) << 10) | (uint32_t(n >> 3) << 17) |
         (uint32_t(OZ_BM >> 4) << 24);
}

// The 28 digit products of one K chunk (A digit planes at a0 + i 4 KB, B
// planes at b0 + j OZ_B_PLANE) into the seven group accumulators at TMEM
// column 64 g.  acc = 0 only for a tile's first chunk: its digit-0 MMAs
// come first and cover every group once, so they overwrite and all later
// MMAs accumulate.
__device__ __forceinline__ void oz_issue_chunk(uint32_t tmem, uint32_t a0, uint32_t b0, bool first) {
#if OZ_WIDE
  // (i, g0, n): A digit i x B digits g0 - i .. g0 - i + n - 1 -> groups g0 .. g0 + n - 1 (N = 64 n <= 256)
  constexpr int seq[10][3] = {{0, 0, 4}, {0, 4, 3}, {1, 1, 3}, {1, 4, 3}, {2, 2, 2},
                              {2, 4, 3}, {3, 3, 4}, {4, 4, 3}, {5, 5, 2}, {6, 6, 1}};
#pragma unroll
  for (int q = 0; q < 10; ++q) {
    const int i = seq[q][0], g0 = seq[q][1], n = seq[q][2];
    tc_mma_i8(tmem + uint32_t(g0 * OZ_BN), smem_desc(a0 + i * OZ_A_SLICE, OZ_BM * 16, 128),
              smem_desc(b0 + (g0 - i) * OZ_B_PLANE, OZ_B_LBO, 128), idesc_i8(1, 1, n * OZ_BN),
              (first && i == 0) ? 0u : 1u);
  }
#else
  // A digit i outer, group g inner: consecutive MMAs accumulate into
  // different TMEM groups; group g's first MMA of a tile is (i = 0, j = g)
#pragma unroll
  for (int i = 0; i < OZ_S; ++i) {
    const uint64_t ad = smem_desc(a0 + i * OZ_A_SLICE, OZ_BM * 16, 128);
#pragma unroll
    for (int g = i; g < OZ_G; ++g)
      tc_mma_i8(tmem + uint32_t(g * OZ_BN), ad, smem_desc(b0 + (g - i) * OZ_B_PLANE, OZ_B_LBO, 128), idesc_i8(1, 1),
                (first && i == 0) ? 0u : 1u);
  }
#endif
}

#if OZ_WIDE
// the narrow last tile: A digit i x B digits 0 .. 6 - i -> groups i .. 6
__device__ __forceinline__ void oz_issue_chunk_narrow(uint32_t tmem, uint32_t a0, uint32_t b0, bool first) {
#pragma unroll
  for (int i = 0; i < OZ_S; ++i)
    tc_mma_i8(tmem + uint32_t(i * OZ_BN_N), smem_desc(a0 + i * OZ_A_SLICE, OZ_BM * 16, 128),
              smem_desc(b0, OZ_B_LBO_N, 128), idesc_i8(1, 1, (OZ_S - i) * OZ_BN_N), (first && i == 0) ? 0u : 1u);
}
#endif

// is column block cb of M2 columns a narrow (<= 32 live columns) last tile
// (OZ_NARROW = 0, variant builds: full 64-column tiles throughout)
#ifndef OZ_NARROW
#define OZ_NARROW 1
#endif
__host__ __device__ __forceinline__ bool oz_narrow(int64_t cb, int64_t n_cb, int64_t M2) {
  return OZ_WIDE && OZ_NARROW && cb == n_cb - 1 && M2 - cb * OZ_BN <= 32;
}

// A (rows x K, row-major, lda) -> row-scaled digits, tiled
// [row block][K chunk][slice][kq 2][row 128][16 B]; sa[r] = 2^(e_r - 28)
// (the 2^-12 of the digit scales and the 2^-16 of the epilogue's split sum).
// A block takes 16 consecutive rows (K <= 512): each warp reads 4 rows
// (coalesced, lane = 2 consecutive doubles of every 64-column segment),
// reduces the row maximum, and writes its digit vectors into a shared
// staging tile laid out like the global planes; the block then writes every
// (chunk, slice) plane segment of its 16 rows as one contiguous 256-byte run.
// Rows >= rows and k >= K are zero.
// 8 warps x 4 rows per block (32 rows: 512-B plane segments), 2 blocks per
// SM.  Per 1M x 400 rows alone: 1.23 ms (5.2 TB/s) vs 1.28 ms for 4 warps x
// 16 rows (the round-1 shape, sized so that one split block co-resided with
// a GEMM CTA; the wide-MMA GEMM's 168 registers leave no room for that, and
// under the step's power cap a co-running split costs its own time anyway).
#ifndef OZ_SLICE_WARPS_CFG
#define OZ_SLICE_WARPS_CFG 8
#define OZ_SLICE_ROWS_CFG 32
#define OZ_SLICE_MINB 2
#endif
constexpr int OZ_SLICE_WARPS = OZ_SLICE_WARPS_CFG;
constexpr int OZ_SLICE_ROWS = OZ_SLICE_ROWS_CFG;
constexpr int OZ_SLICE_MAXCH = 32;   // K <= 512
#ifndef OZ_SLICE_NARROW
#define OZ_SLICE_NARROW 1            // 0: always the K <= 512 instance (measurement knob)
#endif
#ifndef OZ_SLICE_MINB_NARROW
#define OZ_SLICE_MINB_NARROW 4
#endif
// middle instance (K <= 64 OZ_SLICE_MID_SEGS; c4: K = 400 -> seven segments, no dead eighth: digit split 18.2 -> 17.6 ms), 0: none
#ifndef OZ_SLICE_MID_SEGS
#define OZ_SLICE_MID_SEGS 7
#endif
#ifndef OZ_SLICE_MINB_MID
#define OZ_SLICE_MINB_MID 2
#endif
// staging: [chunk][slice][row 16] x 16 B plus one 16-B pad per chunk, so the
// four chunks a warp's digit store touches land in different banks (without
// the pad the chunk stride is 0 mod 32 words: a 4-way conflict on every
// store, and the co-running GEMM is bound by the same shared-memory port)
constexpr int OZ_SLICE_CH_STRIDE = OZ_S * OZ_SLICE_ROWS + 1;   // uint4 per chunk
constexpr size_t OZ_SLICE_SMEM = size_t(OZ_SLICE_MAXCH) * OZ_SLICE_CH_STRIDE * 16;
// NSEGMAX: 64-column segments a lane can hold (K <= 64 NSEGMAX).  The K <= 256
// instance keeps two row buffers of 4 segments instead of 8, so more blocks
// are resident and enough bytes are in flight for the narrow bases (c3:
// K = 150, c2: K = 200), whose rows are only 1.2-1.6 KB.
template <int NSEGMAX, int MINB>
__global__ void __launch_bounds__(OZ_SLICE_WARPS * 32, MINB) oz_slice_rows_kernel(const double* __restrict__ A,
                                                                            int64_t lda, int64_t rows, int64_t K,
                                                                            int64_t nkc, uint8_t* __restrict__ sl,
                                                                            double* __restrict__ sa) {
  extern __shared__ __align__(16) uint4 stg[];   // [chunk][slice][row 32] x 16 B
  uint32_t* stg32 = reinterpret_cast<uint32_t*>(stg);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row0 = int64_t(blockIdx.x) * OZ_SLICE_ROWS;
  const int nch = static_cast<int>(nkc * 2);
  const int nseg = (nch + 3) / 4;                // 64-element segments
  constexpr int RPW = OZ_SLICE_ROWS / OZ_SLICE_WARPS;   // rows per warp
  // coalesced: lane holds elements 64 g + 2 lane, +1 of every segment g;
  // the next row's loads are issued before this row's digits
  auto load_row = [&](int jj, double2 (&x)[NSEGMAX]) {
    const int64_t r = row0 + warp * RPW + jj;
    const bool live = r < rows;
    const double* row = A + (live ? r : 0) * lda;
    const bool vec = !(reinterpret_cast<uintptr_t>(row) & 15);
#pragma unroll
    for (int g = 0; g < NSEGMAX; ++g) {
      const int64_t k = int64_t(g) * 64 + 2 * lane;
      if (g < nseg && live && vec && k + 2 <= K) {
        x[g] = *reinterpret_cast<const double2*>(row + k);
      } else {
        x[g].x = (g < nseg && live && k < K) ? row[k] : 0.0;
        x[g].y = (g < nseg && live && k + 1 < K) ? row[k + 1] : 0.0;
      }
    }
  };
  double2 xn[NSEGMAX];
  load_row(0, xn);
  for (int j = 0; j < RPW; ++j) {
    const int lr = warp * RPW + j;
    const int64_t r = row0 + lr;
    double2 x[NSEGMAX];
#pragma unroll
    for (int g = 0; g < NSEGMAX; ++g) x[g] = xn[g];
    if (j + 1 < RPW) load_row(j + 1, xn);
    double amax = 0.0;
#pragma unroll
    for (int g = 0; g < NSEGMAX; ++g) amax = fmax(amax, fmax(fabs(x[g].x), fabs(x[g].y)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const int e = oz_exponent(amax);
    if (lane == 0) sa[r] = ldexp(1.0, e - 28);
    const double scale = ldexp(1.0, 54 - e);
#pragma unroll
    for (int g = 0; g < NSEGMAX; ++g) {
      if (g >= nseg) break;
      // Y = X + 0x808080808080: balanced digit s = byte (6 - s) of Y (^ 0x80 for s >= 1)
      const unsigned long long Y0 = static_cast<unsigned long long>(__double2ll_rn(x[g].x * scale)) + 0x808080808080ull;
      const unsigned long long Y1 = static_cast<unsigned long long>(__double2ll_rn(x[g].y * scale)) + 0x808080808080ull;
      const uint32_t lo0 = uint32_t(Y0), hi0 = uint32_t(Y0 >> 32), lo1 = uint32_t(Y1), hi1 = uint32_t(Y1 >> 32);
      const int ch = g * 4 + (lane >> 3);
#pragma unroll
      for (int s2 = 0; s2 < OZ_S; ++s2) {
        const int p = 6 - s2;
        const uint32_t sel = (p & 3) | (((p & 3) + 4) << 4);
        uint32_t h = p < 4 ? __byte_perm(lo0, lo1, sel) : __byte_perm(hi0, hi1, sel);
        h = (h & 0xFFFFu) ^ (s2 == 0 ? 0u : 0x8080u);
        const uint32_t nb = __shfl_down_sync(0xffffffffu, h, 1);
        if (!(lane & 1) && ch < nch)
          stg32[(ch * OZ_SLICE_CH_STRIDE + s2 * OZ_SLICE_ROWS + lr) * 4 + ((lane & 7) >> 1)] = h | (nb << 16);
      }
    }
  }
  __syncthreads();
  // plane segment (chunk ch, slice s2): rows row0..row0+31 -> 512 contiguous bytes
  const int64_t rb = row0 / OZ_BM, rr0 = row0 % OZ_BM;
  {
    const int lr = threadIdx.x % OZ_SLICE_ROWS;
    constexpr int SEG_STEP = OZ_SLICE_WARPS * 32 / OZ_SLICE_ROWS;
    uint8_t* base = sl + rb * nkc * OZ_A_STAGE + (rr0 + lr) * 16;
    for (int seg = threadIdx.x / OZ_SLICE_ROWS; seg < nch * OZ_S; seg += SEG_STEP) {
      const int ch = seg / OZ_S, s2 = seg - ch * OZ_S;
      *reinterpret_cast<uint4*>(base + (ch >> 1) * OZ_A_STAGE + s2 * OZ_A_SLICE + (ch & 1) * (OZ_BM * 16)) =
          stg[ch * OZ_SLICE_CH_STRIDE + s2 * OZ_SLICE_ROWS + lr];
    }
  }
}

// B (K x M2, row-major, ldb) -> column-scaled digits, tiled
// [col block][K chunk][slice][kq 2][col 64][16 B]; sb[c] = 2^f_c.
__global__ void __launch_bounds__(OZ_BN) oz_slice_cols_kernel(const double* __restrict__ B, int64_t ldb,
                                                              int64_t K, int64_t M2, int64_t nkc,
                                                              uint8_t* __restrict__ sl, double* __restrict__ sb) {
  const int64_t cb = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t c = cb * OZ_BN + tid;
  const bool live = c < M2;
  const bool nar = oz_narrow(cb, gridDim.x, M2);
  double amax = 0.0;
  if (live)
    for (int64_t k = 0; k < K; ++k) amax = fmax(amax, fabs(B[k * ldb + c]));
  const int f = oz_exponent(amax);
  const double scale = ldexp(1.0, 54 - f);
  sb[c] = ldexp(1.0, f);
  if (nar && tid >= OZ_BN_N) return;
  const int64_t nch = nkc * 2;
  for (int64_t ch = 0; ch < nch; ++ch) {
    double v[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int64_t k = ch * 16 + t;
      v[t] = (live && k < K) ? B[k * ldb + c] : 0.0;
    }
    uint4 d[OZ_S];
    oz_digits16(v, scale, d);
    const int64_t kc = ch >> 1, kq = ch & 1;
#if OZ_WIDE
    const uint32_t lbo = nar ? OZ_B_LBO_N : OZ_B_LBO, pl = nar ? OZ_B_PLANE_N : OZ_B_PLANE;
#else
    const uint32_t lbo = OZ_B_LBO, pl = OZ_B_PLANE;
#endif
    uint8_t* base = sl + (cb * nkc + kc) * OZ_B_STAGE + kq * lbo + tid * 16;
#pragma unroll
    for (int s = 0; s < OZ_S; ++s) *reinterpret_cast<uint4*>(base + s * pl) = d[s];
  }
}

// OZ_PROF (variant builds only, tools/oz_bench.py SWB_OZ_PROF=1): per-role
// clock64 sums, [role][wait0, wait1, total, count] for role 0 = producer
// (wait empty), 1 = MMA issuer (wait tile-empty | wait stage-full),
// 2 = epilogue (wait tile-full | tile-full -> TMEM released)
#ifndef OZ_PROF
#define OZ_PROF 0
#endif
#ifndef OZ_EPI2
#define OZ_EPI2 1
#endif
#if OZ_PROF
__device__ unsigned long long oz_prof[12];
#define OZ_T(x) const long long x = clock64()
#else
#define OZ_T(x)
#endif

// out[rows x M2] = sum_g ... (see header).  raw != nullptr: write the seven
// int32 group accumulators instead, raw[(g * rows_p + r) * np + c].
//
// TMEM columns [0, 7 BN): the seven group accumulators (the remaining 64
// columns cannot hold a second set, so TMEM is single-buffered).  The
// epilogue (8 warps, two per TMEM lane quarter, 32 columns each) pulls its
// accumulators into registers in two rounds and releases TMEM right after
// the last load, so the next tile's MMAs overlap the last round's combine
// and stores.  Operands come from shared memory (SS): at N = 64 the MMA
// rate is set by shared-memory bandwidth (6 KB of operands per 128x64x32
// MMA), measured 48 cycles per MMA in isolation (tools/tc_probe.cu).
__global__ void __launch_bounds__(OZ_THREADS, 1)
oz_gemm_kernel(const uint8_t* __restrict__ asl, const double* __restrict__ sa, const uint8_t* __restrict__ bsl,
               const double* __restrict__ sb, int64_t rows, int64_t M2, int64_t nkc, int64_t n_rb, int64_t n_cb,
               double* __restrict__ out, int64_t ldo, int32_t* __restrict__ raw, int64_t ncol_main,
               double* __restrict__ out2, int64_t ldo2, unsigned long long* __restrict__ row_amax) {
  extern __shared__ __align__(1024) uint8_t oz_smem[];
  uint8_t* stages = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_smem) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) uint64_t full_bar[OZ_STAGES], empty_bar[OZ_STAGES], tfull_bar, tempty_bar;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = n_rb * n_cb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    mbar_init(smem_u32(&tfull_bar), 1);
    mbar_init(smem_u32(&tempty_bar), OZ_EPI_WARPS * 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(OZ_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ---------------- producer: two bulk copies per stage ----------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t rb = t / n_cb, cb = t % n_cb;
        for (int64_t kc = 0; kc < nkc; ++kc) {
          mbar_wait(smem_u32(&empty_bar[s]), ph ^ 1);
          const uint32_t fb = smem_u32(&full_bar[s]);
#if OZ_WIDE
          const uint32_t bbytes = oz_narrow(cb, n_cb, M2) ? OZ_B_STAGE_N : OZ_B_STAGE;
#else
          const uint32_t bbytes = OZ_B_STAGE;
#endif
          mbar_expect_tx(fb, OZ_A_STAGE + bbytes);
          const uint32_t dst = smem_u32(stages + size_t(s) * OZ_STAGE);
          bulk_g2s(dst, asl + (rb * nkc + kc) * OZ_A_STAGE, OZ_A_STAGE, fb);
          bulk_g2s(dst + OZ_A_STAGE, bsl + (cb * nkc + kc) * OZ_B_STAGE, bbytes, fb);
          if (++s == OZ_STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int s = 0;
    uint32_t ph = 0, tph = 0;
#if OZ_PROF
    long long w_te = 0, w_full = 0;
    OZ_T(t_begin);
#endif
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const bool nar = oz_narrow(t % n_cb, n_cb, M2);
      OZ_T(t0);
      mbar_wait(smem_u32(&tempty_bar), tph ^ 1);
#if OZ_PROF
      w_te += clock64() - t0;
#endif
      tc_fence_after();
      for (int64_t kc = 0; kc < nkc; ++kc) {
        OZ_T(t1);
        mbar_wait(smem_u32(&full_bar[s]), ph);
#if OZ_PROF
        w_full += clock64() - t1;
#endif
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a0 = smem_u32(stages + size_t(s) * OZ_STAGE);
#if OZ_WIDE
          if (nar) oz_issue_chunk_narrow(tmem, a0, a0 + OZ_A_STAGE, kc == 0);
          else
#endif
            oz_issue_chunk(tmem, a0, a0 + OZ_A_STAGE, kc == 0);
          tc_commit(smem_u32(&empty_bar[s]));          // frees the stage when these finish
          if (kc + 1 == nkc) tc_commit(smem_u32(&tfull_bar));
        }
        __syncwarp();
        if (++s == OZ_STAGES) { s = 0; ph ^= 1; }
      }
      tph ^= 1;
    }
#if OZ_PROF
    if (lane == 0) {
      atomicAdd(&oz_prof[4], (unsigned long long)w_te);
      atomicAdd(&oz_prof[5], (unsigned long long)w_full);
      atomicAdd(&oz_prof[6], (unsigned long long)(clock64() - t_begin));
      atomicAdd(&oz_prof[7], 1ull);
    }
#endif
  } else {
    // ---------------- epilogue: warps 2..9, two per TMEM lane quarter ----------------
    const int ew = warp - 2;                        // 0..7
    const int quarter = warp & 3;                   // TMEM lane quarter this warp may access
    const int c0 = (ew >> 2) * OZ_EPI_COLS;         // 32-column half
    const uint32_t tsrc = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(c0);
    uint32_t tph = 0;
#if OZ_PROF
    long long w_tf = 0, w_drain = 0, t_rel = 0;
    OZ_T(t_begin);
#endif
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int64_t rb = t / n_cb, cb = t % n_cb;
      const int64_t r = rb * OZ_BM + quarter * 32 + lane;
      const int64_t gc0 = cb * OZ_BN + c0;
      const double srow = r < rows ? sa[r] : 0.0;
      OZ_T(t0);
      mbar_wait(smem_u32(&tfull_bar), tph);
#if OZ_PROF
      const long long t_got = clock64();
      w_tf += t_got - t0;
#endif
      tc_fence_after();
      tph ^= 1;
      // narrow last tile: groups at TMEM column 32 g, the c0 = 32 warps idle
      const bool nar = oz_narrow(cb, n_cb, M2);
      const uint32_t gs = nar ? 32u : uint32_t(OZ_BN);
      if (raw) {
        const int64_t rows_p = n_rb * OZ_BM, np = n_cb * OZ_BN;
        for (int h = 0; h < OZ_EPI_COLS; h += 16)
          for (int g = 0; g < OZ_G; ++g) {
            int32_t v[16] = {};
            if (!(nar && c0)) {
              tmem_ld16(tsrc + uint32_t(g * gs + h), v);
              tmem_wait_ld();
            }
            for (int q = 0; q < 16; ++q) raw[(g * rows_p + r) * np + gc0 + h + q] = v[q];
          }
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty_bar));
        continue;
      }
      if (nar) {
        // narrow tile: the two warps of a lane quarter take 16 columns each
        // (one TMEM round: 7 groups x 16 columns), released after one wait
        const int hf = ew >> 2;
        int32_t v[OZ_G][16];
#pragma unroll
        for (int g = 0; g < OZ_G; ++g)
          tmem_ld16(tmem + (uint32_t(quarter * 32) << 16) + uint32_t(g * OZ_BN_N + 16 * hf), v[g]);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty_bar));
        if (r >= rows) continue;
        const int64_t gcn = cb * OZ_BN + 16 * hf;
        double amax = 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const long long H = (static_cast<long long>(v[0][q]) << 16) + (static_cast<long long>(v[1][q]) << 8) +
                              static_cast<long long>(v[2][q]);
          const long long L = (static_cast<long long>(v[3][q]) << 24) + (static_cast<long long>(v[4][q]) << 16) +
                              (static_cast<long long>(v[5][q]) << 8) + static_cast<long long>(v[6][q]);
          const int64_t c = gcn + q;
          if (c < M2) {
            const double y = fma(static_cast<double>(L), 0x1p-32, static_cast<double>(H)) * srow * sb[c];
            if (c < ncol_main) {
              out[r * ldo + c] = y;
              amax = fmax(amax, fabs(y));
            } else {
              out2[r * ldo2 + (c - ncol_main)] = y;
            }
          }
        }
        if (row_amax) atomicMax(row_amax + r, static_cast<unsigned long long>(__double_as_longlong(amax)));
        continue;
      }
      // both 16-column rounds are combined in registers before any store, so
      // TMEM is released right after the second round's loads
      double o[2][16];
#if OZ_EPI2
      // two TMEM waits per tile (not four): round 1's loads are issued in two
      // batches around round 0's combine, so at most ~144 accumulator /
      // partial registers are live (10 warps: <= 168 registers per thread)
      {
        double o0[16];
        int32_t w[3][16];
        {
          int32_t v[OZ_G][16];
#pragma unroll
          for (int g = 0; g < OZ_G; ++g) tmem_ld16(tsrc + uint32_t(g * gs), v[g]);
          tmem_wait_ld();
          long long H0[16];
#pragma unroll
          for (int q = 0; q < 16; ++q)
            H0[q] = (static_cast<long long>(v[0][q]) << 16) + (static_cast<long long>(v[1][q]) << 8) +
                    static_cast<long long>(v[2][q]);
#pragma unroll
          for (int g = 0; g < 3; ++g) tmem_ld16(tsrc + uint32_t(g * gs + 16), w[g]);
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const long long L = (static_cast<long long>(v[3][q]) << 24) + (static_cast<long long>(v[4][q]) << 16) +
                                (static_cast<long long>(v[5][q]) << 8) + static_cast<long long>(v[6][q]);
            o0[q] = fma(static_cast<double>(L), 0x1p-32, static_cast<double>(H0[q])) * srow;
          }
        }
        int32_t x[4][16];
#pragma unroll
        for (int g = 0; g < 4; ++g) tmem_ld16(tsrc + uint32_t((g + 3) * gs + 16), x[g]);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(smem_u32(&tempty_bar));         // the next tile's MMAs may start
#if OZ_PROF
        w_drain += clock64() - t_got;
#endif
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          o[0][q] = o0[q];
          const long long H = (static_cast<long long>(w[0][q]) << 16) + (static_cast<long long>(w[1][q]) << 8) +
                              static_cast<long long>(w[2][q]);
          const long long L = (static_cast<long long>(x[0][q]) << 24) + (static_cast<long long>(x[1][q]) << 16) +
                              (static_cast<long long>(x[2][q]) << 8) + static_cast<long long>(x[3][q]);
          o[1][q] = fma(static_cast<double>(L), 0x1p-32, static_cast<double>(H)) * srow;
        }
      }
#else
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int h = hh * 16;
        // sum_g acc_g 2^-8g = 2^-16 (H + 2^-32 L), H and L exact in int64
        long long H[16];
        {
          int32_t v[3][16];
#pragma unroll
          for (int g = 0; g < 3; ++g) tmem_ld16(tsrc + uint32_t(g * gs + h), v[g]);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 16; ++q)
            H[q] = (static_cast<long long>(v[0][q]) << 16) + (static_cast<long long>(v[1][q]) << 8) +
                   static_cast<long long>(v[2][q]);
        }
        int32_t v[4][16];
#pragma unroll
        for (int g = 0; g < 4; ++g) tmem_ld16(tsrc + uint32_t((g + 3) * gs + h), v[g]);
        tmem_wait_ld();
        if (hh == 1) {                              // all of this thread's TMEM is in registers
          tc_fence_before();
          mbar_arrive(smem_u32(&tempty_bar));       // the next tile's MMAs may start
#if OZ_PROF
          w_drain += clock64() - t_got;
#endif
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const long long L = (static_cast<long long>(v[0][q]) << 24) + (static_cast<long long>(v[1][q]) << 16) +
                              (static_cast<long long>(v[2][q]) << 8) + static_cast<long long>(v[3][q]);
          o[hh][q] = fma(static_cast<double>(L), 0x1p-32, static_cast<double>(H[q])) * srow;
        }
      }
#endif
      if (r >= rows) continue;
      double* orow = out + r * ldo + gc0;
      double amax = 0.0;   // max |out[r, c]| over this thread's columns c < ncol_main
      if (gc0 + OZ_EPI_COLS <= ncol_main) {
#pragma unroll
        for (int q = 0; q < OZ_EPI_COLS; q += 2) {
          const double2 sc = *reinterpret_cast<const double2*>(sb + gc0 + q);
          const double2 y = make_double2(o[q >> 4][q & 15] * sc.x, o[q >> 4][(q & 15) + 1] * sc.y);
          *reinterpret_cast<double2*>(orow + q) = y;
          amax = fmax(amax, fmax(fabs(y.x), fabs(y.y)));
        }
      } else {
        // the ragged last column tile: columns [ncol_main, M2) (extra B
        // columns riding in the tile's padding) go to out2
#pragma unroll
        for (int q = 0; q < OZ_EPI_COLS; ++q) {
          const int64_t c = gc0 + q;
          const double y = o[q >> 4][q & 15] * sb[c];
          if (c < ncol_main) {
            orow[q] = y;
            amax = fmax(amax, fabs(y));
          } else if (c < M2) {
            out2[r * ldo2 + (c - ncol_main)] = y;
          }
        }
      }
      // the row maxima of the product: the next rotation's row scales, so a
      // producer holding these rows can emit their digit planes (no split)
      if (row_amax) atomicMax(row_amax + r, static_cast<unsigned long long>(__double_as_longlong(amax)));
    }
#if OZ_PROF
    (void)t_rel;
    if (lane == 0) {
      atomicAdd(&oz_prof[8], (unsigned long long)w_tf);
      atomicAdd(&oz_prof[9], (unsigned long long)w_drain);
      atomicAdd(&oz_prof[10], (unsigned long long)(clock64() - t_begin));
      atomicAdd(&oz_prof[11], 1ull);
    }
#endif
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(OZ_TMEM_COLS) : "memory");
  }
}

struct OzLayout {
  int64_t chunk_rows, nkc, n_cb, nbuf;
  size_t a_sl, sa, b_sl, sb, total;
};

OzLayout oz_layout(int64_t rows, int64_t K, int64_t M2) {
  OzLayout o{};
  o.nkc = (K + OZ_KC - 1) / OZ_KC;
  o.n_cb = (M2 + OZ_BN - 1) / OZ_BN;
  const int64_t rows_p = (rows + OZ_BM - 1) / OZ_BM * OZ_BM;
  o.chunk_rows = rows_p < (int64_t(1) << 20) ? rows_p : (int64_t(1) << 20);
  if (o.chunk_rows < OZ_BM) o.chunk_rows = OZ_BM;
  const int64_t crb = o.chunk_rows / OZ_BM;
  o.a_sl = swb_align_up(size_t(crb * o.nkc) * OZ_A_STAGE, 256);
  o.sa = swb_align_up(sizeof(double) * size_t(o.chunk_rows), 256);
  o.b_sl = swb_align_up(size_t(o.n_cb * o.nkc) * OZ_B_STAGE, 256);
  o.sb = swb_align_up(sizeof(double) * size_t(o.n_cb * OZ_BN), 256);
  o.nbuf = rows_p > o.chunk_rows ? 2 : 1;   // two chunks' A planes: split i+1 overlaps GEMM i
  o.total = o.nbuf * (o.a_sl + o.sa) + o.b_sl + o.sb;
  return o;
}

struct OzPtrs {
  uint8_t* a_sl;
  double* sa;
  uint8_t* b_sl;
  double* sb;
};

// layout: B planes | C scales | A planes / row scales of buffer 0 [| buffer 1]
OzPtrs oz_ptrs(const OzLayout& o, void* ws, int buf) {
  char* p = static_cast<char*>(ws);
  char* a = p + o.b_sl + o.sb + size_t(buf) * (o.a_sl + o.sa);
  return {reinterpret_cast<uint8_t*>(a), reinterpret_cast<double*>(a + o.a_sl), reinterpret_cast<uint8_t*>(p),
          reinterpret_cast<double*>(p + o.b_sl)};
}

int oz_set_attrs() {
  static unsigned long long attr = 0;
  if (swb_first_on_device(&attr)) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(oz_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(OZ_SMEM)));
    SWB_CUDA_TRY(cudaFuncSetAttribute(oz_slice_rows_kernel<OZ_SLICE_MAXCH / 4, OZ_SLICE_MINB>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(OZ_SLICE_SMEM)));
    SWB_CUDA_TRY(cudaFuncSetAttribute(oz_slice_rows_kernel<4, OZ_SLICE_MINB_NARROW>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(OZ_SLICE_SMEM / 2)));
#if OZ_SLICE_MID_SEGS
    SWB_CUDA_TRY(cudaFuncSetAttribute(oz_slice_rows_kernel<OZ_SLICE_MID_SEGS, OZ_SLICE_MINB_MID>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(OZ_SLICE_SMEM)));
#endif
  }
  return SWB_OK;
}

int oz_check(int64_t rows, int64_t K, int64_t M2, void* ws, size_t ws_bytes, OzLayout* o) {
  if (rows < 0 || K <= 0 || M2 <= 0 || K > OZ_MAX_K || !ws) return SWB_INVALID_PARAM;
  *o = oz_layout(rows > 0 ? rows : 1, K, M2);
  if (ws_bytes < o->total) return SWB_WORKSPACE_TOO_SMALL;
  // a workspace sized by swb_oz_gemm_nn_workspace_bytes_full holds one A-plane
  // buffer per row chunk (planes emitted ahead of the GEMMs)
  const int64_t per = int64_t(o->a_sl + o->sa);
  const int64_t fit = (int64_t(ws_bytes) - int64_t(o->b_sl + o->sb)) / per;
  if (fit > o->nbuf) o->nbuf = fit;
  return oz_set_attrs();
}

}  // namespace

// Split B (K x M2) into its column-scaled digit planes (workspace B region).
extern "C" int swb_oz_split_cols(const double* B, int64_t ldb, int64_t rows, int64_t K, int64_t M2, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  OzLayout o;
  int rc = oz_check(rows, K, M2, workspace, workspace_bytes, &o);
  if (rc) return rc;
  if (!B || ldb < M2) return SWB_INVALID_PARAM;
  const OzPtrs q = oz_ptrs(o, workspace, 0);
  oz_slice_cols_kernel<<<static_cast<unsigned>(o.n_cb), OZ_BN, 0, swb_stream(stream)>>>(B, ldb, K, M2, o.nkc,
                                                                                          q.b_sl, q.sb);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

// Split nr <= swb_oz_chunk_rows() rows of A into their row-scaled digit
// planes (workspace A buffer `buf`, 0 or 1; 1 exists when rows > one chunk).
extern "C" int swb_oz_split_rows(const double* A, int64_t lda, int64_t nr, int64_t rows, int64_t K, int64_t M2,
                                 int buf, void* workspace, size_t workspace_bytes, void* stream) {
  OzLayout o;
  int rc = oz_check(rows, K, M2, workspace, workspace_bytes, &o);
  if (rc) return rc;
  if (!A || lda < K || nr < 0 || nr > o.chunk_rows || buf < 0 || buf >= o.nbuf) return SWB_INVALID_PARAM;
  if (nr == 0) return SWB_OK;
  const OzPtrs q = oz_ptrs(o, workspace, buf);
  const int64_t nrp = (nr + OZ_BM - 1) / OZ_BM * OZ_BM;
  // staging for this K only (2 nkc 16-column halves), not the K <= 512 maximum
  const size_t split_smem = size_t(2 * o.nkc) * OZ_SLICE_CH_STRIDE * 16;
  if (K <= 256 && OZ_SLICE_NARROW)
    oz_slice_rows_kernel<4, OZ_SLICE_MINB_NARROW><<<static_cast<unsigned>(nrp / OZ_SLICE_ROWS), OZ_SLICE_WARPS * 32,
                                                    split_smem, swb_stream(stream)>>>(A, lda, nr, K, o.nkc, q.a_sl, q.sa);
#if OZ_SLICE_MID_SEGS
  else if (K <= 64 * OZ_SLICE_MID_SEGS)
    oz_slice_rows_kernel<OZ_SLICE_MID_SEGS, OZ_SLICE_MINB_MID><<<static_cast<unsigned>(nrp / OZ_SLICE_ROWS),
                                                                 OZ_SLICE_WARPS * 32, split_smem, swb_stream(stream)>>>(
        A, lda, nr, K, o.nkc, q.a_sl, q.sa);
#endif
  else
    oz_slice_rows_kernel<OZ_SLICE_MAXCH / 4, OZ_SLICE_MINB><<<static_cast<unsigned>(nrp / OZ_SLICE_ROWS),
                                                               OZ_SLICE_WARPS * 32, split_smem, swb_stream(stream)>>>(
        A, lda, nr, K, o.nkc, q.a_sl, q.sa);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

// out[nr x M2] from the digit planes in the workspace (raw: diagnostics);
// with ncol_main < M2 the columns [ncol_main, M2) go to out2 instead.
int swb_oz_planes_gemm(int64_t nr, int64_t rows, int64_t K, int64_t M2, int buf, double* out, int64_t ldo,
                       int32_t* raw, void* workspace, size_t workspace_bytes, cudaStream_t st,
                       int64_t ncol_main = -1, double* out2 = nullptr, int64_t ldo2 = 0,
                       unsigned long long* row_amax = nullptr) {
  OzLayout o;
  int rc = oz_check(rows, K, M2, workspace, workspace_bytes, &o);
  if (rc) return rc;
  if (ncol_main < 0) ncol_main = M2;
  if ((!out && !raw) || nr < 0 || nr > o.chunk_rows || buf < 0 || buf >= o.nbuf) return SWB_INVALID_PARAM;
  if (ncol_main > M2 || (ncol_main < M2 && (!out2 || ldo2 < M2 - ncol_main))) return SWB_INVALID_PARAM;
  // 32-column epilogue segments below ncol_main use 16-B stores
  if (out && (ldo < ncol_main || (ldo & 1) || (reinterpret_cast<uintptr_t>(out) & 15))) return SWB_INVALID_PARAM;
  if (nr == 0) return SWB_OK;
  const OzPtrs q = oz_ptrs(o, workspace, buf);
  const int64_t n_rb = (nr + OZ_BM - 1) / OZ_BM;
  const int64_t tiles = n_rb * o.n_cb;
  const int64_t grid_cap = swb_sm_count();
  const int64_t grid = tiles < grid_cap ? tiles : grid_cap;
  oz_gemm_kernel<<<static_cast<unsigned>(grid), OZ_THREADS, OZ_SMEM, st>>>(q.a_sl, q.sa, q.b_sl, q.sb, nr, M2, o.nkc,
                                                                           n_rb, o.n_cb, out, ldo, raw, ncol_main,
                                                                           out2, ldo2, row_amax);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" int swb_oz_gemm_planes(int64_t nr, int64_t rows, int64_t K, int64_t M2, int buf, double* out,
                                  int64_t ldo, void* workspace, size_t workspace_bytes, void* stream) {
  return swb_oz_planes_gemm(nr, rows, K, M2, buf, out, ldo, nullptr, workspace, workspace_bytes,
                            swb_stream(stream));
}

extern "C" int swb_oz_gemm_planes_split(int64_t nr, int64_t rows, int64_t K, int64_t M2, int buf, double* out,
                                        int64_t ldo, int64_t ncol_main, double* out2, int64_t ldo2, void* workspace,
                                        size_t workspace_bytes, void* stream) {
  if (ncol_main < 0) return SWB_INVALID_PARAM;
  return swb_oz_planes_gemm(nr, rows, K, M2, buf, out, ldo, nullptr, workspace, workspace_bytes,
                            swb_stream(stream), ncol_main, out2, ldo2);
}

// The same, also recording row_amax[r] = max_c<ncol_main |out[r, c]| (as the
// bits of a non-negative double; atomicMax, so row_amax must start at 0 --
// the chunk's rows are indexed from out_chunk's first row)
extern "C" int swb_oz_gemm_planes_ex(int64_t nr, int64_t rows, int64_t K, int64_t M2, int buf, double* out,
                                     int64_t ldo, int64_t ncol_main, double* out2, int64_t ldo2,
                                     unsigned long long* row_amax, void* workspace, size_t workspace_bytes,
                                     void* stream) {
  if (ncol_main < 0) return SWB_INVALID_PARAM;
  return swb_oz_planes_gemm(nr, rows, K, M2, buf, out, ldo, nullptr, workspace, workspace_bytes,
                            swb_stream(stream), ncol_main, out2, ldo2, row_amax);
}

#if OZ_PROF
extern "C" int swb_oz_prof_read(unsigned long long* out) {
  SWB_CUDA_TRY(cudaDeviceSynchronize());
  SWB_CUDA_TRY(cudaMemcpyFromSymbol(out, oz_prof, sizeof(oz_prof)));
  return SWB_OK;
}
#endif

extern "C" size_t swb_oz_gemm_nn_workspace_bytes(int64_t rows, int64_t K, int64_t M2) {
  if (rows <= 0 || K <= 0 || M2 <= 0) return 0;
  return oz_layout(rows, K, M2).total;
}

// one A-plane buffer per row chunk: all of A's planes resident at once
extern "C" size_t swb_oz_gemm_nn_workspace_bytes_full(int64_t rows, int64_t K, int64_t M2) {
  if (rows <= 0 || K <= 0 || M2 <= 0) return 0;
  const OzLayout o = oz_layout(rows, K, M2);
  const int64_t rows_p = (rows + OZ_BM - 1) / OZ_BM * OZ_BM;
  const int64_t nch = (rows_p + o.chunk_rows - 1) / o.chunk_rows;
  return o.b_sl + o.sb + size_t(nch) * (o.a_sl + o.sa);
}

// plane geometry for producers that write A planes themselves:
// info = {chunk_rows, nkc, offset of buffer 0's planes, bytes of a buffer's
// planes (its row scales follow), stride between buffers}
extern "C" int swb_oz_layout_info(int64_t rows, int64_t K, int64_t M2, int64_t* info) {
  if (rows <= 0 || K <= 0 || M2 <= 0 || K > OZ_MAX_K || !info) return SWB_INVALID_PARAM;
  const OzLayout o = oz_layout(rows, K, M2);
  info[0] = o.chunk_rows;
  info[1] = o.nkc;
  info[2] = int64_t(o.b_sl + o.sb);
  info[3] = int64_t(o.a_sl);
  info[4] = int64_t(o.a_sl + o.sa);
  return SWB_OK;
}

extern "C" int64_t swb_oz_chunk_rows(int64_t rows, int64_t K, int64_t M2) {
  if (rows <= 0 || K <= 0 || M2 <= 0) return 0;
  return oz_layout(rows, K, M2).chunk_rows;
}

// out[rows x M2] = A[rows x K] * B[K x M2] in FP64 via INT8 tensor cores:
// B's planes once, then per row chunk the chunk's A planes and the GEMM.
// The split of chunk i+1 runs on a side stream into the other A buffer while
// the GEMM of chunk i runs (one split block fits beside a GEMM CTA on every
// SM: 96 + 160 registers x threads, 47 + 173 KB shared memory), so only the
// first chunk's split is exposed.
extern "C" int swb_oz_gemm_nn_split(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows,
                                    int64_t K, int64_t M2, int64_t ncol_main, double* out, int64_t ldo, double* out2,
                                    int64_t ldo2, void* workspace, size_t workspace_bytes, void* stream);

extern "C" int swb_oz_gemm_nn(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows, int64_t K,
                              int64_t M2, double* out, int64_t ldo, void* workspace, size_t workspace_bytes,
                              void* stream) {
  return swb_oz_gemm_nn_split(A, lda, B, ldb, rows, K, M2, M2, out, ldo, nullptr, 0, workspace, workspace_bytes,
                              stream);
}

// The same with the product's columns [ncol_main, M2) written to out2 (ld
// ldo2) instead of out: update_and_solve's extra columns C coeff.
extern "C" int swb_oz_gemm_nn_split(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows,
                                    int64_t K, int64_t M2, int64_t ncol_main, double* out, int64_t ldo, double* out2,
                                    int64_t ldo2, void* workspace, size_t workspace_bytes, void* stream) {
  if (rows == 0) return SWB_OK;
  if (!A || !out || ncol_main < 0 || ncol_main > M2) return SWB_INVALID_PARAM;
  auto gemm = [&](int64_t nr, int buf, int64_t r0) {
    return swb_oz_planes_gemm(nr, rows, K, M2, buf, out + r0 * ldo, ldo, nullptr, workspace, workspace_bytes,
                              swb_stream(stream), ncol_main, out2 ? out2 + r0 * ldo2 : nullptr, ldo2);
  };
  int rc;
  if ((rc = swb_oz_split_cols(B, ldb, rows, K, M2, workspace, workspace_bytes, stream))) return rc;
  const int64_t chunk = swb_oz_chunk_rows(rows, K, M2);
  const int64_t nch = (rows + chunk - 1) / chunk;
#ifndef OZ_OVERLAP
#define OZ_OVERLAP 1
#endif
  if (nch == 1 || !OZ_OVERLAP) {   // OZ_OVERLAP = 0 (variant builds): split and GEMM in turn
    for (int64_t i = 0; i < nch; ++i) {
      const int64_t r0 = i * chunk, nr = rows - r0 < chunk ? rows - r0 : chunk;
      if ((rc = swb_oz_split_rows(A + r0 * lda, lda, nr, rows, K, M2, 0, workspace, workspace_bytes, stream)))
        return rc;
      if ((rc = gemm(nr, 0, r0))) return rc;
    }
    return SWB_OK;
  }
  // side stream + events per device; the mutex makes the enqueue of one
  // call's chunk loop atomic, so concurrent callers (different streams) share
  // the side stream in order and never see each other's event records
  struct Aux {
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_in, ev_split[2], ev_gemm[2];
  };
  static Aux tab[64];
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  Aux& X = tab[swb_device()];
  if (!X.aux) {
    SWB_CUDA_TRY(cudaStreamCreateWithFlags(&X.aux, cudaStreamNonBlocking));
    SWB_CUDA_TRY(cudaEventCreateWithFlags(&X.ev_in, cudaEventDisableTiming));
    for (int b = 0; b < 2; ++b) {
      SWB_CUDA_TRY(cudaEventCreateWithFlags(&X.ev_split[b], cudaEventDisableTiming));
      SWB_CUDA_TRY(cudaEventCreateWithFlags(&X.ev_gemm[b], cudaEventDisableTiming));
    }
  }
  cudaStream_t aux = X.aux;
  cudaEvent_t& ev_in = X.ev_in;
  cudaEvent_t* ev_split = X.ev_split;
  cudaEvent_t* ev_gemm = X.ev_gemm;
  cudaStream_t st = swb_stream(stream);
  SWB_CUDA_TRY(cudaEventRecord(ev_in, st));            // A, B's planes ready
  SWB_CUDA_TRY(cudaStreamWaitEvent(aux, ev_in, 0));
  auto split = [&](int64_t i) -> int {
    const int64_t r0 = i * chunk, nr = rows - r0 < chunk ? rows - r0 : chunk;
    if (i >= 2) SWB_CUDA_TRY(cudaStreamWaitEvent(aux, ev_gemm[i & 1], 0));   // buffer free
    int e = swb_oz_split_rows(A + r0 * lda, lda, nr, rows, K, M2, int(i & 1), workspace, workspace_bytes, aux);
    if (e) return e;
    SWB_CUDA_TRY(cudaEventRecord(ev_split[i & 1], aux));
    return SWB_OK;
  };
  if ((rc = split(0))) return rc;
  for (int64_t i = 0; i < nch; ++i) {
    if (i + 1 < nch && (rc = split(i + 1))) return rc;
    const int64_t r0 = i * chunk, nr = rows - r0 < chunk ? rows - r0 : chunk;
    SWB_CUDA_TRY(cudaStreamWaitEvent(st, ev_split[i & 1], 0));
    if ((rc = gemm(nr, int(i & 1), r0))) return rc;
    SWB_CUDA_TRY(cudaEventRecord(ev_gemm[i & 1], st));
  }
  return SWB_OK;
}

// diagnostics: the seven int32 group accumulators of rows [0, min(rows,
// chunk)) as raw[(g * rows_p + r) * np + c] (rows_p, np padded to 128 / 64)
extern "C" int swb_oz_gemm_nn_raw(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t rows,
                                  int64_t K, int64_t M2, int32_t* raw, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  if (rows <= 0 || !raw) return SWB_INVALID_PARAM;
  int rc;
  if ((rc = swb_oz_split_cols(B, ldb, rows, K, M2, workspace, workspace_bytes, stream))) return rc;
  const int64_t nr = rows < swb_oz_chunk_rows(rows, K, M2) ? rows : swb_oz_chunk_rows(rows, K, M2);
  if ((rc = swb_oz_split_rows(A, lda, nr, rows, K, M2, 0, workspace, workspace_bytes, stream))) return rc;
  return swb_oz_planes_gemm(nr, rows, K, M2, 0, nullptr, 0, raw, workspace, workspace_bytes, swb_stream(stream));
}

// ---------------------------------------------------------------------------
// INT8 tensor-core peak probe (measurement only): back-to-back
// tcgen05.mma.kind::i8 M = 128, N = 256, K = 32 from shared memory on every
// SM (the shape that reaches the full rate); bench.py times it for the live
// INT8 roofline.  ops_out = 2 * MACs issued.
// ---------------------------------------------------------------------------
namespace {
__device__ __forceinline__ uint32_t probe_hash(uint32_t seed, uint32_t i) {
  uint32_t x = seed * 0x9E3779B9u ^ (i + blockIdx.x * 0x85EBCA6Bu);
  x ^= x >> 16; x *= 0x7FEB352Du; x ^= x >> 15; x *= 0x846CA68Bu; x ^= x >> 16;
  return x;
}

__global__ void __launch_bounds__(128, 1) int8_probe_kernel(int iters, uint32_t seed) {
  extern __shared__ __align__(1024) uint8_t pr_smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  // operands: zeros (seed 0: the burst figure) or pseudo-random bytes (the
  // data-dependent switching power of real operands)
  for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(pr_smem)[i] =
        seed ? make_uint4(probe_hash(seed, 4 * i), probe_hash(seed, 4 * i + 1), probe_hash(seed, 4 * i + 2),
                          probe_hash(seed, 4 * i + 3))
             : make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(pr_smem), b0 = a0 + 16384;
    constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(256 >> 3) << 17) | (8u << 24);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        tc_mma_i8(tm, smem_desc(a0 + (k & 3) * 4096, OZ_BM * 16, 128), smem_desc(b0 + (k & 1) * 8192, 256 * 16, 128),
                  idesc, 1u);
    tc_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
  }
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm) : "memory");
}
}  // namespace

// The rotation GEMM's own MMA pattern in isolation: M 128, N 64, K 32 from
// shared memory into seven rotating TMEM accumulators (7 x 64 columns), i.e.
// the ceiling of the 28-digit-product scheme, whose seven resident group
// accumulators cap N at 64 (bench.py reports the GEMM against it too).
namespace {
__global__ void __launch_bounds__(128, 1) int8_probe_n64_kernel(int iters, uint32_t seed) {
  extern __shared__ __align__(1024) uint8_t pr_smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  // operands: zeros (seed 0: the burst figure) or pseudo-random bytes (the
  // data-dependent switching power of real operands)
  for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(pr_smem)[i] =
        seed ? make_uint4(probe_hash(seed, 4 * i), probe_hash(seed, 4 * i + 1), probe_hash(seed, 4 * i + 2),
                          probe_hash(seed, 4 * i + 3))
             : make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(pr_smem), b0 = a0 + 28672;
    for (int it = 0; it < iters; ++it) oz_issue_chunk(tm, a0, b0, false);
    tc_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
  }
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}
}  // namespace

extern "C" int swb_int8_scheme_probe(int iters, double* ops_out, void* stream) {
  return swb_int8_probe_ex(1, iters, 0, ops_out, stream);
}

extern "C" int swb_int8_peak_probe(int iters, double* ops_out, void* stream) {
  return swb_int8_probe_ex(0, iters, 0, ops_out, stream);
}

static int int8_scheme_probe_impl(int iters, uint32_t seed, double* ops_out, void* stream) {
  if (iters <= 0 || !ops_out) return SWB_INVALID_PARAM;
  static unsigned long long attr = 0;
  if (swb_first_on_device(&attr)) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(int8_probe_n64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
  }
  const int sms = swb_sm_count();
  int8_probe_n64_kernel<<<sms, 128, 48 * 1024, swb_stream(stream)>>>(iters, seed);
  SWB_CHECK_LAUNCH();
  *ops_out = 2.0 * double(sms) * iters * (OZ_S * (OZ_S + 1) / 2) * double(OZ_BM) * OZ_BN * OZ_KC;
  return SWB_OK;
}

static int int8_peak_probe_impl(int iters, uint32_t seed, double* ops_out, void* stream) {
  if (iters <= 0 || !ops_out) return SWB_INVALID_PARAM;
  static unsigned long long attr = 0;
  if (swb_first_on_device(&attr)) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(int8_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
  }
  const int sms = swb_sm_count();
  int8_probe_kernel<<<sms, 128, 48 * 1024, swb_stream(stream)>>>(iters, seed);
  SWB_CHECK_LAUNCH();
  *ops_out = 2.0 * double(sms) * iters * 8 * 128.0 * 256.0 * 32.0;
  return SWB_OK;
}

extern "C" int swb_int8_probe_ex(int pattern, int iters, unsigned int seed, double* ops_out, void* stream) {
  if (pattern == 0) return int8_peak_probe_impl(iters, seed, ops_out, stream);
  if (pattern == 1) return int8_scheme_probe_impl(iters, seed, ops_out, stream);
  return SWB_INVALID_PARAM;
}
