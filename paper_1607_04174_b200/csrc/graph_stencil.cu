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

// one thread per voxel, its forward edges in turn; 32-bit index splits when
// the lattice allows (a 64-bit division by a runtime divisor is ~100
// instructions, and the per-edge version paid five of them)
template <typename IT>
__device__ __forceinline__ void voxel_xyz(const LatticeDev& L, int64_t v, int64_t& x, int64_t& y, int64_t& z) {
  const IT vv = static_cast<IT>(v), nx = static_cast<IT>(L.nx), ny = static_cast<IT>(L.ny);
  const IT q = vv / nx;
  x = static_cast<int64_t>(vv - q * nx);
  const IT q2 = q / ny;
  y = static_cast<int64_t>(q - q2 * ny);
  z = static_cast<int64_t>(q2);
}

__global__ void edge_weight_kernel(const StencilGeom g, const double* __restrict__ I, double beta, int weight_mode,
                                   const uint8_t* __restrict__ cut, double* __restrict__ w, int64_t N) {
  const int nd = g.lat.ndir;
  const bool small = N < (int64_t(1) << 31);
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < N; v += int64_t(gridDim.x) * blockDim.x) {
    int64_t x, y, z;
    if (small) voxel_xyz<uint32_t>(g.lat, v, x, y, z);
    else voxel_xyz<int64_t>(g.lat, v, x, y, z);
    const double iv = I[v];
#pragma unroll 4
    for (int d = 0; d < nd; ++d) {
      const int64_t e = v * nd + d;
      const int64_t x2 = x + g.lat.dx[d], y2 = y + g.lat.dy[d], z2 = z + g.lat.dz[d];
      double out = 0.0;
      if (in_grid(g.lat, x2, y2, z2) && !(cut && cut[e])) {
        const int64_t u = x2 + g.lat.nx * (y2 + g.lat.ny * z2);
        const double diff = __dadd_rn(iv, -I[u]);
        const double arg = weight_mode == 0 ? fabs(diff) : __dmul_rn(diff, diff);
        out = fmax(exp(__dmul_rn(-beta, arg)), W_MIN);  // graphs.py:136
      }
      w[e] = out;
    }
  }
}

// degrees in increasing neighbour-index order (scipy csr row sum), d_sqrt,
// diag = (inv*d)*inv with inv = 1/d_sqrt (graphs.py:154-158)
__global__ void degree_kernel(const StencilGeom g, const double* __restrict__ w, double* __restrict__ d_sqrt,
                              double* __restrict__ diag, int32_t* __restrict__ degenerate, int64_t N) {
  const int nd = g.lat.ndir;
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < N;
       v += int64_t(gridDim.x) * blockDim.x) {
    int64_t x, y, z;
    if (N < (int64_t(1) << 31)) voxel_xyz<uint32_t>(g.lat, v, x, y, z);
    else voxel_xyz<int64_t>(g.lat, v, x, y, z);
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
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < N; v += int64_t(gridDim.x) * blockDim.x) {
    const double iv = 1.0 / d_sqrt[v];
#pragma unroll 4
    for (int d = 0; d < nd; ++d) {
      const int64_t e = v * nd + d;
      const double we = w[e];
      if (we == 0.0) continue;
      const int64_t u = v + g.lat.dx[d] + g.lat.nx * (g.lat.dy[d] + g.lat.ny * int64_t(g.lat.dz[d]));
      const double iu = 1.0 / d_sqrt[u];
      const double a = __dmul_rn(__dmul_rn(iv, we), iu);
      const double b = __dmul_rn(__dmul_rn(iu, we), iv);
      w[e] = __dmul_rn(__dadd_rn(a, b), 0.5);
    }
  }
}

// --- stencil passes --------------------------------------------------------

// cp.async with a precomputed shared-space address
__device__ __forceinline__ void cp_async16_s(uint32_t s, const void* gmem, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" :: "r"(s), "l"(gmem), "r"(pred ? 16 : 0));
}
__device__ __forceinline__ void cp_async8_s(uint32_t s, const void* gmem, bool pred) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" :: "r"(s), "l"(gmem), "r"(pred ? 8 : 0));
}

constexpr int ST_WARPS = 8;
// SWB_ST_EXACT=1 (default): L^'v in the reference's CSR order with separate
// multiply / add (refresh eigenvalues track scipy to ~1e-16); 0: FMAs
#ifndef SWB_ST_EXACT
#define SWB_ST_EXACT 1
#endif
#ifndef SWB_ST_CTAS
#define SWB_ST_CTAS 2
#endif
#ifndef SWB_ST_PREF
#define SWB_ST_PREF 5
#endif
constexpr int ST_CTAS_PER_SM = SWB_ST_CTAS;
// rows per barrier step: two independent rows per step halve the barriers and
// give each warp two dependency chains to interleave
#ifndef SWB_ST_ROWS
#define SWB_ST_ROWS 2
#endif
constexpr int ST_ROWS = SWB_ST_ROWS;
static_assert(ST_ROWS == 1 || ST_ROWS == 2, "one or two rows per step");
// x-lines per warp: 1 = a warp covers one line x 64 columns; 2 = each half-warp
// one line x 32 columns (32-column blocks: K = 400 wastes 16 of 416 columns
// instead of 48 of 448, and the CTA's 16 lines share a smaller halo)
#ifndef SWB_ST_LPW
#define SWB_ST_LPW 2
#endif
constexpr int ST_LPW = SWB_ST_LPW;
static_assert(ST_LPW == 1 || ST_LPW == 2, "one or two lines per warp");
constexpr int ST_CBW = 64 / ST_LPW;   // columns per line (column block width)

// Compile-time neighbour tables, sorted by flat offset (the reference CSR
// column order): kind 0 = diagonal, 1 = forward edge `dir` of this voxel,
// 2 = backward edge `dir` (stored at the neighbour).
struct NbC { int dx, dy, dz, dir, kind; };

__host__ __device__ constexpr int nb_count(int conn) { return conn == 4 ? 5 : (conn == 8 ? 9 : 7); }
__host__ __device__ constexpr int nb_ndir(int conn) { return conn == 4 ? 2 : (conn == 8 ? 4 : 3); }
__host__ __device__ constexpr NbC nb_entry(int conn, int i) {
  // 4-conn: -y -x diag +x +y        dirs {+x, +y}
  // 8-conn: (-1,-1) -y (+1,-1) -x diag +x (-1,+1) +y (+1,+1)
  //         dirs {+x, +y, (+1,+1), (-1,+1)}
  // 6-conn: -z -y -x diag +x +y +z  dirs {+x, +y, +z}
  return conn == 4
             ? (i == 0 ? NbC{0, -1, 0, 1, 2} : i == 1 ? NbC{-1, 0, 0, 0, 2} : i == 2 ? NbC{0, 0, 0, -1, 0}
                : i == 3 ? NbC{1, 0, 0, 0, 1} : NbC{0, 1, 0, 1, 1})
         : conn == 8
             ? (i == 0 ? NbC{-1, -1, 0, 2, 2} : i == 1 ? NbC{0, -1, 0, 1, 2} : i == 2 ? NbC{1, -1, 0, 3, 2}
                : i == 3 ? NbC{-1, 0, 0, 0, 2} : i == 4 ? NbC{0, 0, 0, -1, 0} : i == 5 ? NbC{1, 0, 0, 0, 1}
                : i == 6 ? NbC{-1, 1, 0, 3, 1} : i == 7 ? NbC{0, 1, 0, 1, 1} : NbC{1, 1, 0, 2, 1})
             : (i == 0 ? NbC{0, 0, -1, 2, 2} : i == 1 ? NbC{0, -1, 0, 1, 2} : i == 2 ? NbC{-1, 0, 0, 0, 2}
                : i == 3 ? NbC{0, 0, 0, -1, 0} : i == 4 ? NbC{1, 0, 0, 0, 1} : i == 5 ? NbC{0, 1, 0, 1, 1}
                : NbC{0, 0, 1, 2, 1});
}

// One warp: one x-line (nx consecutive voxel rows) of one 64-column block
// (lane = 2 adjacent columns, 16-byte loads).  Per line the warp sets up one
// row pointer per stencil entry (off-grid lines point at the centre row with
// a zero coefficient) and then walks x with pointer increments only; the
// first / last voxel of a line clamp their +-x neighbours.  Per-column
// partial sums live in registers and are flushed to slots[warp][col][3]
// whenever the warp moves to another column block.
// Coefficient element of the stencil pass: the new L^ entry, or for the
// difference pass the (new, old) pair interleaved by pair_coeffs_kernel so
// one 16-byte load serves both.
template <bool DELTA> struct CoefT { using T = double; };
template <> struct CoefT<true> { using T = double2; };

// (new, new - old) pairs: pw[r*ND + d] = {what_new, what_new - what_old}, pd[r] likewise for the diagonal
__global__ void pair_coeffs_kernel(const double* __restrict__ wn, const double* __restrict__ wo,
                                   const double* __restrict__ dn, const double* __restrict__ dold, int nd_dir,
                                   int64_t r0, int64_t r1, double2* __restrict__ pw, double2* __restrict__ pd) {
  // rows [r0, r1) only: a range pass needs its own rows and their y-1 / z-1 sources
  const int64_t nr = r1 - r0, nw = nr * nd_dir;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nw + nr; i += int64_t(gridDim.x) * blockDim.x) {
    if (i < nw) {
      const int64_t e = r0 * nd_dir + i;
      pw[e] = make_double2(wn[e], wn[e] - wo[e]);
    } else {
      const int64_t r = r0 + (i - nw);
      pd[r] = make_double2(dn[r], dn[r] - dold[r]);
    }
  }
}


// ---------------------------------------------------------------------------
// Stencil pass v5: CTA-shared ring.  A CTA's 8 warps own a block of
// ZB x YB x-lines (3-D: 4 z x 2*LPW y; 2-D: 8*LPW y) of one CBW-column block;
// warp w takes the LPW lines (zi, yi) = (w / (YB/LPW), (w % (YB/LPW))*LPW + h),
// h = lane / (CBW/2) -- a warp's lines are y-adjacent, so with the linear slot
// grid below half-warp h's operands sit h slots past half-warp 0's.  Each ring stage holds, for voxel
// row x, every V line the block needs exactly once -- the 8 centre lines plus
// the one-line halo around the block (no corners) -- together with each
// centre line's coefficients (forward + diag, and the forward coefficients
// of its y-1 / z-1 source rows) and d_sqrt.  Lines shared by sibling warps
// (their +-y / +-z neighbours) are therefore fetched from L2 once instead of
// once per warp; +-x comes from the adjacent stages as before.  One CTA
// barrier per row; RING = PREF + 3 so the stage being refilled is never one
// a warp can still read.
// ---------------------------------------------------------------------------
template <int CONN, bool DELTA>
struct Ring5 {
  static constexpr bool D3 = CONN == 6;
  static constexpr int ND = nb_ndir(CONN);
  static constexpr int LPW = ST_LPW, CBW = ST_CBW, HL = CBW / 2;     // lines per warp, columns, lanes per line
  static constexpr int ZB = D3 ? 4 : 1;
  static constexpr int YB = D3 ? 2 * LPW : 8 * LPW;
  static constexpr int WY = YB / LPW;                                  // warps along y
  static constexpr int NL = ZB * YB;                                   // centre lines (= warps x LPW)
  // extended grid (ZB+2) x (YB+2) without corners (3-D); 2-D: 1 x (YB+2).
  // LPW = 1: compact slots; LPW = 2: the full linear grid (4 corner slots
  // never filled) so that slot(z, y + 1) = slot(z, y) + 1 everywhere
  static constexpr bool LIN = LPW > 1;
  static constexpr int NSU = D3 ? NL + 2 * ZB + 2 * YB : YB + 2;       // V line slots in use
  static constexpr int NS = D3 && LIN ? (ZB + 2) * (YB + 2) : NSU;     // V line slots
  static constexpr int CW = DELTA ? 2 : 1;
  static constexpr int NCL = D3 ? 3 : 2;                               // coefficient rows per line
  static constexpr int COEF = (ND + 1) + ND * (NCL - 1);
  static constexpr int LCD = (COEF * CW + 1 + 1) / 2 * 2;              // doubles per line (+ d_sqrt), 16-B aligned
  static constexpr int V_DBL = NS * CBW;
  static constexpr int C_DBL = (NL * LCD + 1) / 2 * 2;
  static constexpr int STAGE_DBL = V_DBL + C_DBL;
  static constexpr int PREF = SWB_ST_PREF;
  static constexpr int RING = PREF + ST_ROWS + 1;   // rows x-1 .. x+PREF+ST_ROWS-1 live at once
  // slot of extended line (zi, yi), zi in [-1, ZB], yi in [-1, YB]; -1 = unused corner
  __host__ __device__ static constexpr int slot(int zi, int yi) {
    return !D3 ? (yi + 1)
           : LIN ? (zi + 1) * (YB + 2) + (yi + 1)
                 : (zi >= 0 && zi < ZB && yi >= 0 && yi < YB) ? zi * YB + yi
                 : (zi >= 0 && zi < ZB && yi == -1) ? NL + zi
                 : (zi >= 0 && zi < ZB && yi == YB) ? NL + ZB + zi
                 : (yi >= 0 && yi < YB && zi == -1) ? NL + 2 * ZB + yi
                 : (yi >= 0 && yi < YB && zi == ZB) ? NL + 2 * ZB + YB + yi
                 : -1;
  }
  // slot of the u-th line in use (copy order) -> extended (zi, yi)
  __host__ __device__ static void used_line(int u, int& ez, int& ey) {
    if (!D3) { ez = 0; ey = u - 1; return; }
    if (LIN) {
      const int s = u < YB ? u + 1 : u < YB + ZB * (YB + 2) ? u + 2 : u + 3;   // skip the corners
      ez = s / (YB + 2) - 1;
      ey = s % (YB + 2) - 1;
      return;
    }
    if (u < NL) { ez = u / YB; ey = u % YB; }
    else if (u < NL + ZB) { ez = u - NL; ey = -1; }
    else if (u < NL + 2 * ZB) { ez = u - NL - ZB; ey = YB; }
    else if (u < NL + 2 * ZB + YB) { ey = u - NL - 2 * ZB; ez = -1; }
    else { ey = u - NL - 2 * ZB - YB; ez = ZB; }
  }
};

// Apply mode of the plain pass (no DELTA, W given): W = a * (L^ v) + b * v + g * Z
// (Z optional) -- one step of a three-term polynomial recurrence in L^.
struct ApplyArgs {
  const double* Z;
  int64_t ldz;
  double a, b, g;
};

// One row of one warp's centre line: (L^' v, dL v) for the lane's two
// columns, the Rayleigh / norm / d-projection partial sums and the W store.
// Register window of a warp's own line along x: the centre value of the
// previous / current row and the previous row's +x coefficient, so the +-x
// neighbours and the -x backward coefficient come from registers (5 shared
// V loads per row instead of 7).
// W is written once and not read by this kernel: SWB_ST_WCS=1 (default) stores it
// with the streaming (evict-first) policy so it does not displace the V halo
// lines neighbouring CTAs are about to read from L2
#ifndef SWB_ST_WCS
#define SWB_ST_WCS 1
#endif
__device__ __forceinline__ void st_w(double* p, double2 v) {
#if SWB_ST_WCS
  __stcs(reinterpret_cast<double2*>(p), v);
#else
  *reinterpret_cast<double2*>(p) = v;
#endif
}

struct RowWin {
  double2 prev, cur, f0;
};

// `lane` here is the thread's V offset inside its half-warp's line slot
// (h * CBW + 2 * li doubles) and `coff` its coefficient offset (h * LCD).
template <int CONN, bool DELTA, int WARP>
__device__ __forceinline__ void row_compute(const double* sc, const double* sm1, const double* sp1, int lane,
                                            int coff, bool active, double2& q, double2& s2, double2& sd,
                                            double* wrow, const ApplyArgs& ap, const double* zrow, RowWin& win,
                                            bool first) {
  using Rg = Ring5<CONN, DELTA>;
  constexpr int ND = Rg::ND, CW = Rg::CW, LCD = Rg::LCD, NB = nb_count(CONN), CBW = Rg::CBW;
  constexpr int ZI = WARP / Rg::WY, YI = (WARP % Rg::WY) * Rg::LPW;   // half-warp 0's line
  constexpr int CBASE = Rg::V_DBL + (ZI * Rg::YB + YI) * LCD;
  constexpr int OWN = Rg::slot(ZI, YI) * CBW;
  const double* scl = sc + lane;
  const double* sml = sm1 + lane;
  const double* spl = sp1 + lane;
  sc += coff;
  sm1 += coff;
  sp1 += coff;
  if (first) {
    win.prev = make_double2(0.0, 0.0);
    win.cur = *reinterpret_cast<const double2*>(scl + OWN);
    win.f0 = make_double2(0.0, 0.0);
  }
  const double2 c = win.cur;
  const double2 nxt = *reinterpret_cast<const double2*>(spl + OWN);
  const double d = sc[CBASE + Rg::COEF * CW];
  double lx = 0.0, ly = 0.0, dx = 0.0, dy = 0.0;
  double2 f0 = make_double2(0.0, 0.0);
#pragma unroll
  for (int e = 0; e < NB; ++e) {
    const NbC t = nb_entry(CONN, e);
    const bool own_x = t.dy == 0 && t.dz == 0;
    double2 val;
    if (own_x) {
      val = t.dx < 0 ? win.prev : t.dx > 0 ? nxt : c;
    } else {
      const double* vl = t.dx < 0 ? sml : t.dx > 0 ? spl : scl;
      val = *reinterpret_cast<const double2*>(vl + Rg::slot(ZI + t.dz, YI + t.dy) * CBW);
    }
    const double* vs = t.dx < 0 ? sm1 : t.dx > 0 ? sp1 : sc;
    const int slot = t.kind == 0 ? ND : t.kind == 1 ? t.dir
                     : (t.dz < 0 ? 2 * ND + 1 + t.dir : t.dy < 0 ? ND + 1 + t.dir : t.dir);
    double cn, g = 0.0;
    if (t.kind == 2 && own_x) {          // -x: the previous row's +x forward pair
      cn = win.f0.x;
      g = win.f0.y;
    } else {
      const double* cp = (t.kind == 2 ? vs : sc) + CBASE + slot * CW;
      if (DELTA) {
        const double2 pr = *reinterpret_cast<const double2*>(cp);  // (new, new - old) in one 16-B load
        cn = pr.x;
        g = pr.y;
      } else {
        cn = cp[0];
      }
      if (t.kind == 1 && t.dir == 0) f0 = make_double2(cn, g);
    }
    // L^' v in the reference CSR order (exact products and sums); dL v with FMAs
    if (t.kind == 0) {
#if SWB_ST_EXACT
      lx = __dadd_rn(lx, __dmul_rn(cn, val.x));
      ly = __dadd_rn(ly, __dmul_rn(cn, val.y));
#else
      lx = fma(cn, val.x, lx);
      ly = fma(cn, val.y, ly);
#endif
      if (DELTA) { dx = fma(g, val.x, dx); dy = fma(g, val.y, dy); }
    } else {
#if SWB_ST_EXACT
      lx = __dadd_rn(lx, __dmul_rn(-cn, val.x));
      ly = __dadd_rn(ly, __dmul_rn(-cn, val.y));
#else
      lx = fma(-cn, val.x, lx);
      ly = fma(-cn, val.y, ly);
#endif
      if (DELTA) { dx = fma(-g, val.x, dx); dy = fma(-g, val.y, dy); }
    }
  }
  win.prev = c;
  win.cur = nxt;
  win.f0 = f0;
  if (active) {
    q.x = fma(c.x, lx, q.x);
    q.y = fma(c.y, ly, q.y);
    s2.x = fma(c.x, c.x, s2.x);
    s2.y = fma(c.y, c.y, s2.y);
    sd.x = fma(c.x, d, sd.x);
    sd.y = fma(c.y, d, sd.y);
    if (DELTA) {
      st_w(wrow, make_double2(dx, dy));
    } else if (wrow) {
      double ox = fma(ap.a, lx, ap.b * c.x), oy = fma(ap.a, ly, ap.b * c.y);
      if (zrow) {
        const double2 z = *reinterpret_cast<const double2*>(zrow);
        ox = fma(ap.g, z.x, ox);
        oy = fma(ap.g, z.y, oy);
      }
      st_w(wrow, make_double2(ox, oy));
    }
  }
}

// warp-uniform binary dispatch to the compile-time line position
template <int CONN, bool DELTA, int LO, int HI>
__device__ __forceinline__ void row_dispatch(int warp, const double* sc, const double* sm1, const double* sp1, int lane,
                                             int coff, bool active, double2& q, double2& s2, double2& sd, double* wrow,
                                             const ApplyArgs& ap, const double* zrow, RowWin& win, bool first) {
  if constexpr (HI - LO == 1) {
    row_compute<CONN, DELTA, LO>(sc, sm1, sp1, lane, coff, active, q, s2, sd, wrow, ap, zrow, win, first);
  } else {
    constexpr int MID = (LO + HI) / 2;
    if (warp < MID)
      row_dispatch<CONN, DELTA, LO, MID>(warp, sc, sm1, sp1, lane, coff, active, q, s2, sd, wrow, ap, zrow, win,
                                         first);
    else
      row_dispatch<CONN, DELTA, MID, HI>(warp, sc, sm1, sp1, lane, coff, active, q, s2, sd, wrow, ap, zrow, win,
                                         first);
  }
}

// two consecutive rows (x over stages s0 | s1 | s2, x+1 over s1 | s2 | s3) in
// one straight-line leaf; the second row is inert (active2 false, zero
// stages) past the end of an odd line
template <int CONN, bool DELTA, int LO, int HI>
__device__ __forceinline__ void row_dispatch2(int warp, const double* s0, const double* s1, const double* s2p,
                                              const double* s3, int lane, int coff, bool active, bool active2,
                                              double2& q,
                                              double2& s2, double2& sd, double* wrow, int64_t ldw,
                                              const ApplyArgs& ap, const double* zrow, RowWin& win, bool first) {
  if constexpr (HI - LO == 1) {
    row_compute<CONN, DELTA, LO>(s1, s0, s2p, lane, coff, active, q, s2, sd, wrow, ap, zrow, win, first);
    row_compute<CONN, DELTA, LO>(s2p, s1, s3, lane, coff, active2, q, s2, sd, wrow ? wrow + ldw : wrow, ap,
                                 zrow ? zrow + ap.ldz : zrow,
                                 win, false);
  } else {
    constexpr int MID = (LO + HI) / 2;
    if (warp < MID)
      row_dispatch2<CONN, DELTA, LO, MID>(warp, s0, s1, s2p, s3, lane, coff, active, active2, q, s2, sd, wrow, ldw,
                                          ap, zrow, win, first);
    else
      row_dispatch2<CONN, DELTA, MID, HI>(warp, s0, s1, s2p, s3, lane, coff, active, active2, q, s2, sd, wrow, ldw,
                                          ap, zrow, win, first);
  }
}

// add a warp's per-column partial sums into its slots (the LPW lines of a warp
// cover the same columns: fold half-warp 1 into half-warp 0 first); warp-uniform
template <int LPW, int HL>
__device__ __forceinline__ void flush_slots(double* sl, int h, double2 q, double2 s2, double2 sd) {
  if constexpr (LPW == 2) {
    constexpr unsigned FULL = 0xffffffffu;
    q.x += __shfl_down_sync(FULL, q.x, HL);
    q.y += __shfl_down_sync(FULL, q.y, HL);
    s2.x += __shfl_down_sync(FULL, s2.x, HL);
    s2.y += __shfl_down_sync(FULL, s2.y, HL);
    sd.x += __shfl_down_sync(FULL, sd.x, HL);
    sd.y += __shfl_down_sync(FULL, sd.y, HL);
  }
  if (h == 0) {
    sl[0] += q.x; sl[1] += s2.x; sl[2] += sd.x; sl[3] += q.y; sl[4] += s2.y; sl[5] += sd.y;
  }
}

template <int CONN, bool DELTA>
__global__ void __launch_bounds__(ST_WARPS * 32, ST_CTAS_PER_SM)
stencil5_kernel(const StencilGeom g, const double* __restrict__ V, int64_t ldv, int64_t row_base, int64_t blk_begin,
                int64_t blk_end, int64_t M, int n_cb, const double* __restrict__ cwhat, const double* __restrict__ cdiag,
                const double* __restrict__ d_sqrt, double* __restrict__ W, int64_t ldw, int64_t w_row0,
                double* __restrict__ slots, int64_t slot_ld, const ApplyArgs ap) {
  using Rg = Ring5<CONN, DELTA>;
  constexpr int ND = Rg::ND, CW = Rg::CW, RING = Rg::RING, PREF = Rg::PREF, SD = Rg::STAGE_DBL;
  constexpr int ZB = Rg::ZB, YB = Rg::YB, NL = Rg::NL, LCD = Rg::LCD, CBW = Rg::CBW, HL = Rg::HL;
  static_assert(NL == ST_WARPS * Rg::LPW, "LPW centre lines per warp");
  extern __shared__ __align__(16) double ring[];
  double* zst = ring + RING * SD;  // zero stage for x-1 < 0 / x+1 >= nx
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  constexpr uint32_t STAGE_BYTES = 8u * SD;
  for (int i = threadIdx.x; i < SD; i += blockDim.x) zst[i] = 0.0;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int h = lane / HL, li = lane % HL;          // half-warp (line) and lane within it
  const int zi = warp / Rg::WY, yi = (warp % Rg::WY) * Rg::LPW + h;
  const int voff = h * CBW + 2 * li, coff = h * LCD;
  const int64_t gwarp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nx = g.lat.nx, ny = g.lat.ny, nz = g.lat.nz;
  const int64_t plane = nx * ny;
  const int nxi = static_cast<int>(nx);
  // items: (column block, block along the slowest axis, block along y) -- y fastest
  const int64_t n_slow = Rg::D3 ? (blk_end - blk_begin + ZB - 1) / ZB : 1;
  const int64_t n_yb = Rg::D3 ? (ny + YB - 1) / YB : (blk_end - blk_begin + YB - 1) / YB;
  const int64_t per_cb = n_slow * n_yb;
  const int64_t n_items = int64_t(n_cb) * per_cb;

  // copy assignment of this thread (fixed per kernel): V chunks j = tid + i*256
  constexpr int VCH = Rg::NSU * HL;                  // 16-byte chunks per stage (HL per line)
  constexpr int VPT = (VCH + ST_WARPS * 32 - 1) / (ST_WARPS * 32);
  constexpr int CSL = NL * (Rg::COEF + 1);           // coefficient / d_sqrt slots per stage
  __syncthreads();

  double2 q = make_double2(0.0, 0.0), s2 = q, sd = q;
  int cur_cb = -1;
  // static round-robin, y fastest (a global work counter with z-fastest
  // bands raised the L2 hit rate 28% -> 53% but ran 11% slower, and made the
  // per-warp Rayleigh partial sums run-to-run nondeterministic)
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int cb = static_cast<int>(it / per_cb);
    const int64_t rem = it % per_cb;
    const int64_t zb = rem / n_yb, yb = rem % n_yb;
    const int64_t z0 = Rg::D3 ? blk_begin + zb * ZB : 0;
    const int64_t y0 = Rg::D3 ? yb * YB : blk_begin + yb * YB;
    const int64_t z_end = Rg::D3 ? blk_end : 1;
    const int64_t y_end = Rg::D3 ? ny : blk_end;
    // my centre line
    const int64_t my_z = z0 + zi, my_y = y0 + yi;
    const bool line_live = (Rg::D3 ? my_z < z_end : true) && my_y < y_end;
    if (cb != cur_cb) {
      if (cur_cb >= 0) {
        flush_slots<Rg::LPW, HL>(slots + gwarp * slot_ld * 3 + (int64_t(cur_cb) * CBW + 2 * li) * 3, h, q, s2, sd);
      }
      q = make_double2(0.0, 0.0); s2 = q; sd = q;
      cur_cb = cb;
    }
    const int64_t col0 = int64_t(cb) * CBW;
    // per-thread copy sources for this item: V chunks
    const double* vsrc[VPT];
    int vdst[VPT];
    bool vok[VPT];
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int j = threadIdx.x + i * ST_WARPS * 32;
      vok[i] = false; vsrc[i] = V; vdst[i] = 0;
      if (j < VCH) {
        const int u = j / HL, ch = j % HL;
        int ez = 0, ey = 0;
        Rg::used_line(u, ez, ey);
        const int s = Rg::slot(ez, ey);
        const int64_t lz = z0 + ez, ly = y0 + ey;
        const int64_t col = col0 + 2 * ch;
        const bool ok = lz >= 0 && lz < nz && ly >= 0 && ly < ny && col < M &&
                        (Rg::D3 ? true : ly < ny);
        vok[i] = ok;
        vsrc[i] = ok ? V + ((lz * ny + ly) * nx - row_base) * ldv + col : V;
        vdst[i] = s * CBW + 2 * ch;
      }
    }
    // coefficient slot: line l = cs / (COEF+1), k = cs % (COEF+1) (k == COEF -> d_sqrt)
    const double* csrc = d_sqrt;
    int64_t cstride = 0;
    int cdst = 0, cbytes = 0;
    bool cok = false;
    if (threadIdx.x < CSL) {
      const int l = threadIdx.x / (Rg::COEF + 1), k = threadIdx.x % (Rg::COEF + 1);
      const int lzi = l / YB, lyi = l % YB;
      const int64_t lz = z0 + lzi, ly = y0 + lyi;
      const bool live = (lz < nz) && (ly < ny);
      const int64_t r0 = (lz * ny + ly) * nx;
      cdst = Rg::V_DBL + l * LCD + (k < Rg::COEF ? k * CW : Rg::COEF * CW);
      if (!live) {
        cok = false; csrc = d_sqrt; cstride = 0; cbytes = 8 * CW;
      } else if (k < ND) {
        csrc = cwhat + (r0 * ND + k) * CW; cstride = ND * CW; cbytes = 8 * CW; cok = true;
      } else if (k == ND) {
        csrc = cdiag + r0 * CW; cstride = CW; cbytes = 8 * CW; cok = true;
      } else if (k < 2 * ND + 1) {
        cok = ly > 0;
        csrc = cwhat + ((r0 - (cok ? nx : 0)) * ND + (k - ND - 1)) * CW; cstride = ND * CW; cbytes = 8 * CW;
      } else if (k < Rg::COEF) {
        cok = lz > 0;
        csrc = cwhat + ((r0 - (cok ? plane : 0)) * ND + (k - 2 * ND - 1)) * CW; cstride = ND * CW; cbytes = 8 * CW;
      } else {
        csrc = d_sqrt + r0; cstride = 1; cbytes = 8; cok = true;
      }
    }
    // shared-space byte addresses of this thread's copy destinations in stage 0
    uint32_t vdst_s[VPT];
#pragma unroll
    for (int i = 0; i < VPT; ++i) vdst_s[i] = ring_s + 8u * uint32_t(vdst[i]);
    const uint32_t cdst_s = ring_s + 8u * uint32_t(cdst);
    uint32_t pst_off = 0;  // byte offset of the stage being filled
    int xp = 0;
    // per-chunk row steps (0 for masked chunks), fixed for the item
    int64_t vinc[VPT];
#pragma unroll
    for (int i = 0; i < VPT; ++i) vinc[i] = vok[i] ? ldv : 0;
    const int64_t cinc = cok ? cstride : 0;
    const bool last_chunk = threadIdx.x + (VPT - 1) * ST_WARPS * 32 < VCH;
    const bool has_coef = threadIdx.x < CSL;
    auto prefetch = [&]() {
      if (xp < nxi) {
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
          if (i + 1 < VPT || last_chunk) {
            cp_async16_s(vdst_s[i] + pst_off, vsrc[i], vok[i]);
            vsrc[i] += vinc[i];  // next row (pointer increments only)
          }
        }
        if (has_coef) {
          if (cbytes == 16) cp_async16_s(cdst_s + pst_off, csrc, cok);
          else cp_async8_s(cdst_s + pst_off, csrc, cok);
          csrc += cinc;
        }
        ++xp;
        pst_off = pst_off + STAGE_BYTES == RING * STAGE_BYTES ? 0u : pst_off + STAGE_BYTES;
      }
      cp_async_commit();
    };
#pragma unroll
    for (int i = 0; i < PREF; ++i) prefetch();

    const bool active = line_live && (col0 + 2 * li < M);
    const int64_t my_r0 = (my_z * ny + my_y) * nx;
    double* wrow = (W && line_live) ? W + (my_r0 - w_row0) * ldw + col0 + 2 * li : nullptr;
    const double* zrow = (!DELTA && ap.Z && line_live) ? ap.Z + (my_r0 - w_row0) * ap.ldz + col0 + 2 * li : nullptr;
    const double* sc = ring;
    RowWin win;
    if constexpr (ST_ROWS == 2) {
      auto nxt = [&](const double* p) { return p + SD == ring + RING * SD ? ring : p + SD; };
      const double* sm1 = zst;
      for (int x = 0; x < nxi; x += 2) {
        cp_async_wait<PREF - 3>();   // rows <= x+2 have landed (this thread's copies)
        __syncthreads();             // ... every thread's; rows x-2, x-1 finished everywhere
        prefetch();                  // rows x+PREF, x+PREF+1 -> stages of rows x-3, x-2
        prefetch();
        const double* sp = nxt(sc);
        const double* sp2 = nxt(sp);
        const double* s2s = x + 1 < nxi ? sp : zst;
        const double* s3s = x + 2 < nxi ? sp2 : zst;
        if (line_live) {
          row_dispatch2<CONN, DELTA, 0, ST_WARPS>(warp, sm1, sc, s2s, s3s, voff, coff, active, active && x + 1 < nxi, q,
                                                  s2, sd, wrow, ldw, ap, zrow, win, x == 0);
          if (wrow) wrow += 2 * ldw;
          if (zrow) zrow += 2 * ap.ldz;
        }
        sm1 = sp;
        sc = sp2;
      }
    } else
    for (int x = 0; x < nxi; ++x) {
      cp_async_wait<PREF - 2>();   // rows <= x+1 have landed (this thread's copies)
      __syncthreads();             // ... every thread's; compute(x-1) finished everywhere
      prefetch();                  // row x+PREF -> stage (x+PREF) % RING == stage of row x-2
      const double* sp = sc + SD == ring + RING * SD ? ring : sc + SD;
      const double* sm1 = x > 0 ? (sc == ring ? ring + (RING - 1) * SD : sc - SD) : zst;
      const double* sp1 = x + 1 < nxi ? sp : zst;
      if (line_live) {
        // the warp's line position is a compile-time constant in each
        // instantiation, so every shared operand is an immediate offset
        row_dispatch<CONN, DELTA, 0, ST_WARPS>(warp, sc, sm1, sp1, voff, coff, active, q, s2, sd, wrow, ap, zrow, win,
                                               x == 0);
        if (wrow) wrow += ldw;
        if (zrow) zrow += ap.ldz;
      }
      sc = sp;
    }
    cp_async_wait<0>();
    __syncthreads();
  }
  if (cur_cb >= 0)
    flush_slots<Rg::LPW, HL>(slots + gwarp * slot_ld * 3 + (int64_t(cur_cb) * CBW + 2 * li) * 3, h, q, s2, sd);
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

template <int CONN, bool DELTA>
int launch_stencil5(const StencilGeom& g, const double* V, int64_t ldv, int64_t row_base, int64_t blk_begin,
                    int64_t blk_end, int64_t M, int n_cb, const double* cw, const double* cd, const double* d_sqrt,
                    double* W, int64_t ldw, int64_t w_row0, double* slots, int64_t slot_ld, int64_t grid,
                    const ApplyArgs& ap, cudaStream_t st) {
  using Rg = Ring5<CONN, DELTA>;
  const size_t smem = sizeof(double) * size_t(Rg::RING + 1) * Rg::STAGE_DBL;
  auto kern = stencil5_kernel<CONN, DELTA>;
  static unsigned long long attr = 0;
  if (swb_first_on_device(&attr)) {
    SWB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  }
  kern<<<static_cast<unsigned>(grid), ST_WARPS * 32, smem, st>>>(g, V, ldv, row_base, blk_begin, blk_end, M, n_cb, cw,
                                                                 cd, d_sqrt, W, ldw, w_row0, slots, slot_ld, ap);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

// workspace layout: slots | zeros (nx*ND + 1 coefficient elements) | pairs (DELTA)
struct StencilWs {
  size_t slots, zeros, pairs, total;
};

StencilWs stencil_ws_layout(const LatticeDev& L, int64_t M) {
  StencilWs w{};
  const int64_t n_cb = (M + ST_CBW - 1) / ST_CBW;
  const int64_t N = L.nx * L.ny * L.nz;
  w.slots = swb_align_up(sizeof(double) * size_t(stencil_grid() * ST_WARPS) * size_t(n_cb * ST_CBW) * 3, 256);
  w.zeros = swb_align_up(sizeof(double2) * size_t(L.nx * L.ndir + 1), 256);
  w.pairs = swb_align_up(sizeof(double2) * size_t(N * (L.ndir + 1)), 256);
  w.total = w.slots + w.zeros + w.pairs;
  return w;
}

template <bool DELTA>
int run_stencil(const swb_lattice* lat, const double* V, int64_t ldv, int64_t row_base,
                int64_t r_begin, int64_t r_end, int64_t M, const double* what_new,
                const double* diag_new, const double* what_old, const double* diag_old,
                const double* d_sqrt, double* W, int64_t ldw, double* quad, double* norm2, double* vtd,
                void* ws, size_t ws_bytes, void* stream, const ApplyArgs& ap = ApplyArgs{nullptr, 0, 1.0, 0.0, 0.0}) {
  using T = typename CoefT<DELTA>::T;
  cudaStream_t st = swb_stream(stream);
  StencilGeom g;
  int rc = make_geom(lat, &g);
  if (rc) return rc;
  const LatticeDev& L = g.lat;
  if (!V || M <= 0 || ldv < M || r_begin < row_base || r_end < r_begin) return SWB_INVALID_PARAM;
  if (r_begin % L.nx || r_end % L.nx) return SWB_INVALID_PARAM;  // whole x-lines
  const int64_t N = L.nx * L.ny * L.nz;
  if (r_end > N) return SWB_INVALID_PARAM;
  if (ldv & 1) return SWB_INVALID_PARAM;                              // 16-byte row access
  if ((reinterpret_cast<uintptr_t>(V) | reinterpret_cast<uintptr_t>(W)) & 15) return SWB_INVALID_PARAM;
  if (W && (ldw & 1)) return SWB_INVALID_PARAM;
  const StencilWs lay = stencil_ws_layout(L, M);
  if (!ws || ws_bytes < lay.total) return SWB_WORKSPACE_TOO_SMALL;
  const int n_cb = static_cast<int>((M + ST_CBW - 1) / ST_CBW);
  const int64_t slot_ld = int64_t(n_cb) * ST_CBW;
  const int64_t grid = stencil_grid();
  const int64_t n_warps = grid * ST_WARPS;
  char* base = static_cast<char*>(ws);
  double* slots = reinterpret_cast<double*>(base);
  T* zeros = reinterpret_cast<T*>(base + lay.slots);
  SWB_CUDA_TRY(cudaMemsetAsync(slots, 0, lay.slots + lay.zeros, st));
  const T* cwhat;
  const T* cdiag;
  if (DELTA) {
    double2* pw = reinterpret_cast<double2*>(base + lay.slots + lay.zeros);
    double2* pd = pw + N * L.ndir;
    const int64_t back = L.conn == 6 ? L.nx * L.ny : L.nx;   // y-1 / z-1 source rows of the range
    const int64_t p0 = std::max<int64_t>(0, r_begin - back), p1 = r_end;
    pair_coeffs_kernel<<<swb_sm_count() * 8, 256, 0, st>>>(what_new, what_old, diag_new, diag_old, L.ndir, p0, p1, pw,
                                                           pd);
    SWB_CHECK_LAUNCH();
    cwhat = reinterpret_cast<const T*>(pw);
    cdiag = reinterpret_cast<const T*>(pd);
  } else {
    cwhat = reinterpret_cast<const T*>(what_new);
    cdiag = reinterpret_cast<const T*>(diag_new);
  }
  const int64_t n_lines = (r_end - r_begin) / L.nx;
  if (n_lines > 0) {
    (void)zeros;
    const double* cw = reinterpret_cast<const double*>(cwhat);
    const double* cd = reinterpret_cast<const double*>(cdiag);
    int rc2 = SWB_OK;
    // 3-D: blocks along z (whole planes); 2-D: along y (whole lines)
    const int64_t unit = L.conn == 6 ? L.nx * L.ny : L.nx;
    if (r_begin % unit || r_end % unit) return SWB_INVALID_PARAM;
    const int64_t b0 = r_begin / unit, b1 = r_end / unit;
    if (L.conn == 4) rc2 = launch_stencil5<4, DELTA>(g, V, ldv, row_base, b0, b1, M, n_cb, cw, cd, d_sqrt, W, ldw, r_begin, slots, slot_ld, grid, ap, st);
    else if (L.conn == 8) rc2 = launch_stencil5<8, DELTA>(g, V, ldv, row_base, b0, b1, M, n_cb, cw, cd, d_sqrt, W, ldw, r_begin, slots, slot_ld, grid, ap, st);
    else rc2 = launch_stencil5<6, DELTA>(g, V, ldv, row_base, b0, b1, M, n_cb, cw, cd, d_sqrt, W, ldw, r_begin, slots, slot_ld, grid, ap, st);
    if (rc2) return rc2;
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

extern "C" int swb_edge_weights(const swb_lattice* lat, const double* intensities, double beta,
                                const uint8_t* cut_mask, double* w, void* stream) {
  if (!(beta >= 0.0) || !intensities || !w) return SWB_INVALID_PARAM;
  StencilGeom g;
  int rc = make_geom(lat, &g);
  if (rc) return rc;
  const int64_t N = g.lat.nx * g.lat.ny * g.lat.nz;
  edge_weight_kernel<<<swb_sm_count() * 8, 256, 0, swb_stream(stream)>>>(g, intensities, beta, lat->weight_mode,
                                                                         cut_mask, w, N);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

extern "C" size_t swb_stencil_workspace_bytes(const swb_lattice* lat, int64_t M) {
  LatticeDev L;
  if (swb_make_lattice(lat, &L) || M <= 0) return 0;
  return stencil_ws_layout(L, M).total;
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

extern "C" int swb_stencil_apply(const swb_lattice* lat, const double* V, int64_t ldv, int64_t row_base,
                                 int64_t r_begin, int64_t r_end, int64_t M, const double* what, const double* diag,
                                 const double* d_sqrt, double a, double b, const double* Z, int64_t ldz, double g,
                                 double* out, int64_t ldo, double* quad, double* norm2, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  if (!what || !diag || !d_sqrt || !out || ldo < M || (ldo & 1)) return SWB_INVALID_PARAM;
  if (Z && (ldz < M || (ldz & 1) || (reinterpret_cast<uintptr_t>(Z) & 15))) return SWB_INVALID_PARAM;
  const ApplyArgs ap{Z, ldz, a, b, g};
  return run_stencil<false>(lat, V, ldv, row_base, r_begin, r_end, M, what, diag, nullptr, nullptr, d_sqrt, out, ldo,
                            quad, norm2, nullptr, workspace, workspace_bytes, stream, ap);
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
