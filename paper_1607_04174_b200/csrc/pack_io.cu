// .rwpk pack ingest (reference fastrw.py:228-325):
//   * xxh64 over the header + payload on the host (native C++, streaming; the
//     reference hashes in pure Python at ~16 MB/s)
//   * the f32 column-major eigenvector block -> f64 row-major device basis
//     (one transpose kernel through shared memory)
#include "swb_common.cuh"

namespace {
constexpr uint64_t P1 = 0x9E3779B185EBCA87ULL, P2 = 0xC2B2AE3D27D4EB4FULL, P3 = 0x165667B19E3779F9ULL,
                   P4 = 0x85EBCA77C2B2AE63ULL, P5 = 0x27D4EB2F165667C5ULL;
inline uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
inline uint64_t round64(uint64_t acc, uint64_t lane) { return rotl(acc + lane * P2, 31) * P1; }
inline uint64_t rd64(const unsigned char* p) { uint64_t v; __builtin_memcpy(&v, p, 8); return v; }
inline uint32_t rd32(const unsigned char* p) { uint32_t v; __builtin_memcpy(&v, p, 4); return v; }

struct Xxh64State {
  uint64_t v[4];
  uint64_t seed, length;
  unsigned char buf[32];
  int nbuf;
};

// transpose src (m x n f32, row j = eigenvector column j) -> dst (n x ld f64)
__global__ void f32cm_to_f64rm_kernel(const float* __restrict__ src, int64_t n, int64_t m, double* __restrict__ dst,
                                      int64_t ld) {
  __shared__ float tile[32][33];
  const int64_t j0 = int64_t(blockIdx.y) * 32, r0 = int64_t(blockIdx.x) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t j = j0 + k, r = r0 + threadIdx.x;
    if (j < m && r < n) tile[k][threadIdx.x] = src[j * n + r];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, j = j0 + threadIdx.x;
    if (r < n && j < m) dst[r * ld + j] = static_cast<double>(tile[threadIdx.x][k]);
  }
}
}  // namespace

extern "C" size_t swb_xxh64_state_bytes(void) { return sizeof(Xxh64State); }

extern "C" void swb_xxh64_init(void* state, uint64_t seed) {
  Xxh64State* s = static_cast<Xxh64State*>(state);
  s->seed = seed;
  s->v[0] = seed + P1 + P2;
  s->v[1] = seed + P2;
  s->v[2] = seed;
  s->v[3] = seed - P1;
  s->length = 0;
  s->nbuf = 0;
}

extern "C" void swb_xxh64_update(void* state, const void* data, size_t len) {
  Xxh64State* s = static_cast<Xxh64State*>(state);
  const unsigned char* p = static_cast<const unsigned char*>(data);
  s->length += len;
  if (s->nbuf) {
    while (len && s->nbuf < 32) { s->buf[s->nbuf++] = *p++; --len; }
    if (s->nbuf == 32) {
      for (int i = 0; i < 4; ++i) s->v[i] = round64(s->v[i], rd64(s->buf + 8 * i));
      s->nbuf = 0;
    }
  }
  uint64_t v0 = s->v[0], v1 = s->v[1], v2 = s->v[2], v3 = s->v[3];
  while (len >= 32) {
    v0 = round64(v0, rd64(p)); v1 = round64(v1, rd64(p + 8));
    v2 = round64(v2, rd64(p + 16)); v3 = round64(v3, rd64(p + 24));
    p += 32; len -= 32;
  }
  s->v[0] = v0; s->v[1] = v1; s->v[2] = v2; s->v[3] = v3;
  while (len) { s->buf[s->nbuf++] = *p++; --len; }
}

extern "C" uint64_t swb_xxh64_digest(const void* state) {
  const Xxh64State* s = static_cast<const Xxh64State*>(state);
  uint64_t h;
  if (s->length >= 32) {
    h = rotl(s->v[0], 1) + rotl(s->v[1], 7) + rotl(s->v[2], 12) + rotl(s->v[3], 18);
    for (int i = 0; i < 4; ++i) h = (h ^ round64(0, s->v[i])) * P1 + P4;
  } else {
    h = s->seed + P5;
  }
  h += s->length;
  const unsigned char* p = s->buf;
  int n = s->nbuf;
  while (n >= 8) { h ^= round64(0, rd64(p)); h = rotl(h, 27) * P1 + P4; p += 8; n -= 8; }
  if (n >= 4) { h ^= uint64_t(rd32(p)) * P1; h = rotl(h, 23) * P2 + P3; p += 4; n -= 4; }
  while (n > 0) { h ^= uint64_t(*p) * P5; h = rotl(h, 11) * P1; ++p; --n; }
  h ^= h >> 33; h *= P2; h ^= h >> 29; h *= P3; h ^= h >> 32;
  return h;
}

extern "C" int swb_f32_colmajor_to_f64_rowmajor(const float* src, int64_t n, int64_t m, double* dst, int64_t ld,
                                                void* stream) {
  if (!src || !dst || n < 0 || m < 0 || ld < m) return SWB_INVALID_PARAM;
  if (n == 0 || m == 0) return SWB_OK;
  dim3 tb(32, 8), tg(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((m + 31) / 32));
  if (tg.y > 65535) return SWB_INVALID_PARAM;
  f32cm_to_f64rm_kernel<<<tg, tb, 0, swb_stream(stream)>>>(src, n, m, dst, ld);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

namespace {
// transpose src (m x n f64 column-major block) -> dst (n x ld f64 row-major)
__global__ void f64cm_to_f64rm_kernel(const double* __restrict__ src, int64_t n, int64_t m, double* __restrict__ dst,
                                      int64_t ld) {
  __shared__ double tile[32][33];
  const int64_t j0 = int64_t(blockIdx.y) * 32, r0 = int64_t(blockIdx.x) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t j = j0 + k, r = r0 + threadIdx.x;
    if (j < m && r < n) tile[k][threadIdx.x] = src[j * n + r];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, j = j0 + threadIdx.x;
    if (r < n && j < m) dst[r * ld + j] = tile[threadIdx.x][k];
  }
}
}  // namespace

extern "C" int swb_f64_colmajor_to_f64_rowmajor(const double* src, int64_t n, int64_t m, double* dst, int64_t ld,
                                                void* stream) {
  if (!src || !dst || n < 0 || m < 0 || ld < m) return SWB_INVALID_PARAM;
  if (n == 0 || m == 0) return SWB_OK;
  dim3 tb(32, 8), tg(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((m + 31) / 32));
  if (tg.y > 65535) return SWB_INVALID_PARAM;
  f64cm_to_f64rm_kernel<<<tg, tb, 0, swb_stream(stream)>>>(src, n, m, dst, ld);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}

namespace {
// inverse: row-major f64 device basis (n x ld, first m columns, optional
// column map) -> f32 column-major block (m x n rows of n floats)
__global__ void f64rm_to_f32cm_kernel(const double* __restrict__ src, int64_t n, int64_t ld, int64_t m,
                                      const int32_t* __restrict__ col_map, float* __restrict__ dst) {
  __shared__ float tile[32][33];
  const int64_t r0 = int64_t(blockIdx.x) * 32, j0 = int64_t(blockIdx.y) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, j = j0 + threadIdx.x;
    if (r < n && j < m) tile[k][threadIdx.x] = static_cast<float>(src[r * ld + (col_map ? col_map[j] : j)]);
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t j = j0 + k, r = r0 + threadIdx.x;
    if (j < m && r < n) dst[j * n + r] = tile[threadIdx.x][k];
  }
}
}  // namespace

extern "C" int swb_f64_rowmajor_to_f32_colmajor(const double* src, int64_t n, int64_t ld, int64_t m,
                                                const int32_t* col_map, float* dst, void* stream) {
  if (!src || !dst || n < 0 || m < 0 || ld < m) return SWB_INVALID_PARAM;
  if (n == 0 || m == 0) return SWB_OK;
  dim3 tb(32, 8), tg(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((m + 31) / 32));
  if (tg.y > 65535) return SWB_INVALID_PARAM;
  f64rm_to_f32cm_kernel<<<tg, tb, 0, swb_stream(stream)>>>(src, n, ld, m, col_map, dst);
  SWB_CHECK_LAUNCH();
  return SWB_OK;
}
