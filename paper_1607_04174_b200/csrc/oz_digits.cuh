// The rotation's INT8 digit planes (ozaki.cu): digit geometry and the
// row-scaled digit split shared by the split kernel and by producers that
// emit the A planes from rows they already hold (the projection's diagonal
// tiles, dgemm.cu).
#pragma once
#include <cstdint>

namespace {

constexpr int OZ_S = 7;                 // digits per operand
constexpr int OZ_BM = 128;              // rows per tile (MMA M)
constexpr int OZ_KC = 32;               // bytes (= int8 K) per stage / per MMA
constexpr int OZ_A_SLICE = OZ_BM * OZ_KC;            // 4096 B: [kq 2][row 128][16 B]
constexpr int OZ_A_STAGE = OZ_S * OZ_A_SLICE;        // 28 KB

__device__ __forceinline__ int oz_exponent(double amax) {
  if (!(amax > 0.0)) return 0;
  int e;
  frexp(amax, &e);          // amax = m 2^e, m in [0.5, 1)
  return e < -960 ? -960 : e;
}

// 16 consecutive values -> 7 balanced digit vectors of 16 bytes.
// With Y = X + 0x808080808080, the balanced digits are the bytes of Y:
// d_s = byte (6 - s) of Y minus 128 (= byte ^ 0x80) for s = 1..6, and
// d_0 = byte 6 of Y (the signed top, |d_0| <= 65).  Byte gathers are PRMTs.
__device__ __forceinline__ void oz_digits16(const double (&v)[16], double scale, uint4 (&out)[OZ_S]) {
  uint32_t lo[16], hi[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) {
    const unsigned long long Y =
        static_cast<unsigned long long>(__double2ll_rn(v[t] * scale)) + 0x808080808080ull;
    lo[t] = static_cast<uint32_t>(Y);
    hi[t] = static_cast<uint32_t>(Y >> 32);
  }
#pragma unroll
  for (int s = 0; s < OZ_S; ++s) {
    const int p = 6 - s;                     // byte of Y
    const uint32_t sel = (p & 3) | (((p & 3) + 4) << 4);
    const uint32_t flip = s == 0 ? 0u : 0x80808080u;
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t* src = p < 4 ? lo : hi;
      const uint32_t a = __byte_perm(src[4 * q], src[4 * q + 1], sel);
      const uint32_t b = __byte_perm(src[4 * q + 2], src[4 * q + 3], sel);
      w[q] = __byte_perm(a, b, 0x5410) ^ flip;
    }
    out[s] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

}  // namespace
