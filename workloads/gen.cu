// gen.cu -- device twin of the C5 input generator in workloads/__init__.py.
//
// INPUT GENERATION ONLY (test / bench infrastructure): none of the method's
// arithmetic lives here (no coder, no comparison, no sort of the method).  The
// recipe is the counter-based one documented in workloads/__init__.py (reading
// R14 in DESIGN.md); every value of global position i is a function of
// (seed, stream, counter), so one rank can produce block [base, base + n) of
// one global dataset.  tests/test_gpu_workloads.py checks the bytes against the
// numpy twin.  The prefix sort (positions [0, N/10) in ascending order) is
// input preparation done by the Python driver with torch.sort on the keys
// written by c5_prefix_keys.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t splitmix64_h(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Streams {
  uint64_t s[4];
};

inline Streams make_streams(uint64_t seed) {
  Streams S;
  for (int i = 0; i < 4; ++i) S.s[i] = splitmix64_h(seed * 0x100000001B3ull + (uint64_t)i);
  return S;
}

__device__ __forceinline__ uint64_t hi_mul(uint64_t h, uint64_t m) { return ((h >> 32) * m) >> 32; }

constexpr uint32_t kDupThresh = 42949673u;  // ceil(0.01 * 2^32)
constexpr int kSrcTries = 64;

__device__ __forceinline__ bool is_target(const Streams &S, uint64_t pos) {
  return (splitmix64(pos + S.s[1]) >> 32) < kDupThresh;
}

__device__ __forceinline__ int64_t c5_len(const Streams &S, uint64_t ident) {
  return 8 + (int64_t)hi_mul(splitmix64(ident + S.s[0]), 17);
}

__device__ __forceinline__ uint8_t c5_char(const Streams &S, uint64_t ident, uint32_t k) {
  const char *alnum = "0123456789ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz";
  return (uint8_t)alnum[hi_mul(splitmix64((ident << 5) + k + S.s[3]), 62)];
}

__global__ void k_ident(Streams S, uint64_t N, uint64_t base, uint64_t n, int64_t *ident) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t pos = base + i;
    uint64_t id = pos;
    if (is_target(S, pos)) {
      for (int a = 0; a < kSrcTries; ++a) {
        const uint64_t j = hi_mul(splitmix64(pos * 64 + (uint64_t)a + S.s[2]), N);
        if (!is_target(S, j)) {
          id = j;
          break;
        }
      }
    }
    ident[i] = (int64_t)id;
  }
}

__global__ void k_len(Streams S, const int64_t *ident, uint64_t n, int64_t *lens) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    lens[i] = c5_len(S, (uint64_t)ident[i]);
}

// big-endian, NUL-padded 24-byte key of each string as three words (every
// byte < 0x80, so the words compare the same signed or unsigned)
__global__ void k_keys(Streams S, const int64_t *ident, uint64_t n, int64_t *w0, int64_t *w1, int64_t *w2) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t id = (uint64_t)ident[i];
    const int64_t L = c5_len(S, id);
    uint64_t w[3] = {0, 0, 0};
    for (int k = 0; k < 24; ++k) {
      const uint64_t c = k < L ? c5_char(S, id, (uint32_t)k) : 0u;
      w[k >> 3] |= c << (8 * (7 - (k & 7)));
    }
    w0[i] = (int64_t)w[0];
    w1[i] = (int64_t)w[1];
    w2[i] = (int64_t)w[2];
  }
}

__global__ void k_fill(Streams S, const int64_t *ident, const int64_t *off, uint64_t n, uint8_t *units) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t id = (uint64_t)ident[i];
    const int64_t o = off[i], L = off[i + 1] - o;
    for (int64_t k = 0; k < L; ++k) units[o + k] = c5_char(S, id, (uint32_t)k);
  }
}

inline unsigned grid_for(uint64_t n) {
  uint64_t b = (n + 255) / 256;
  return (unsigned)(b > 65536 ? 65536 : (b ? b : 1));
}

}  // namespace

extern "C" {

int gen_c5_ident(uint64_t seed, uint64_t N, uint64_t base, uint64_t n, int64_t *ident, void *stream) {
  if (n) k_ident<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(make_streams(seed), N, base, n, ident);
  return (int)cudaGetLastError();
}

int gen_c5_len(uint64_t seed, const int64_t *ident, uint64_t n, int64_t *lens, void *stream) {
  if (n) k_len<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(make_streams(seed), ident, n, lens);
  return (int)cudaGetLastError();
}

int gen_c5_keys(uint64_t seed, const int64_t *ident, uint64_t n, int64_t *w0, int64_t *w1, int64_t *w2,
                void *stream) {
  if (n) k_keys<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(make_streams(seed), ident, n, w0, w1, w2);
  return (int)cudaGetLastError();
}

int gen_c5_fill(uint64_t seed, const int64_t *ident, const int64_t *off, uint64_t n, uint8_t *units,
                void *stream) {
  if (n) k_fill<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(make_streams(seed), ident, off, n, units);
  return (int)cudaGetLastError();
}

}  // extern "C"
