// verify.cu -- GPU linear verifier of a sort result (TEST / BENCH INFRASTRUCTURE).
//
// Independent of the product (shares no code with paper_2012_00866_b200/csrc):
// it checks a claimed sort result against the DEFINITION of the order the
// method must reach (Alg. 1's final Arrays.sort; SURVEY.md 8(c)
// "Sort result: uniqueness"): under the strict total order (code units compared
// unsigned position by position, a proper prefix first, then the original
// index) the sorted arrangement is unique, so a result equals the oracle's iff
//   (i)   perm is a bijection onto the input indices,
//   (ii)  every adjacent pair of the output is strictly increasing, and
//   (iii) output string i is the input string perm[i] (units and length).
// Used in-bench on every timed output (the CPU oracle's verify is too slow at
// 2^30 strings) and pinned against oracle.verify by tests/test_gpu_checker.py.
// Sharded outputs use (ii) per shard plus order-independent (gidx, string)
// hash sums of inputs and outputs, compared after an all-reduce.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

// unit k of a string (w = 1: uint8, w = 2: uint16)
__device__ __forceinline__ uint32_t unit_at(const uint8_t *u, int w, int64_t k) {
  return w == 1 ? (uint32_t)u[k] : (uint32_t)reinterpret_cast<const uint16_t *>(u)[k];
}

// <0, 0, >0: plain lexicographic comparison of a[0..la), b[0..lb) (no index)
__device__ int cmp_str(const uint8_t *units, int w, int64_t oa, int64_t la, int64_t ob, int64_t lb) {
  const int64_t m = la < lb ? la : lb;
  for (int64_t k = 0; k < m; ++k) {
    const uint32_t x = unit_at(units, w, oa + k), y = unit_at(units, w, ob + k);
    if (x != y) return x < y ? -1 : 1;
  }
  return la < lb ? -1 : (la > lb ? 1 : 0);
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 33)) * 0xFF51AFD7ED558CCDull;
  x = (x ^ (x >> 33)) * 0xC4CEB9FE1A85EC53ull;
  return x ^ (x >> 33);
}

__device__ uint64_t hash_string(const uint8_t *units, int w, int64_t o, int64_t L, uint64_t gidx) {
  uint64_t h = mix64(gidx * 0x9E3779B97F4A7C15ull + (uint64_t)L + 1);
  for (int64_t k = 0; k < L; ++k) h = mix64(h ^ ((uint64_t)unit_at(units, w, o + k) + 0x100ull * (uint64_t)(k + 1)));
  return h;
}

// (ii) on the output: bad[0] += pairs (i, i+1) not strictly increasing
__global__ void k_pairs(const uint8_t *su, int w, const int64_t *so, const uint32_t *perm, uint64_t n,
                        unsigned long long *bad) {
  unsigned long long cnt = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t oa = so[i], ob = so[i + 1], oc = so[i + 2];
    int c = cmp_str(su, w, oa, ob - oa, ob, oc - ob);
    if (c > 0 || (c == 0 && perm[i] >= perm[i + 1])) ++cnt;
  }
  if (cnt) atomicAdd(bad, cnt);
}

// (i) + (iii) single GPU: bad[1] += indices out of range or repeated (bitmap),
// bad[2] += outputs whose string differs from input string perm[i];
// bad[3] += sorted_offsets not starting at 0 / not ending at the total
__global__ void k_content(const uint8_t *units, const int64_t *off, uint64_t n_in, const uint8_t *su,
                          const int64_t *so, const uint32_t *perm, uint64_t n, int w, uint32_t *bitmap,
                          unsigned long long *bad) {
  unsigned long long b1 = 0, b2 = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = perm[i];
    if (p >= n_in) { ++b1; ++b2; continue; }
    const uint32_t old = atomicOr(&bitmap[p >> 5], 1u << (p & 31));
    if (old & (1u << (p & 31))) ++b1;
    const int64_t o = off[p], L = off[p + 1] - o, d = so[i], Ld = so[i + 1] - d;
    if (L != Ld) { ++b2; continue; }
    for (int64_t k = 0; k < L; ++k)
      if (unit_at(units, w, o + k) != unit_at(su, w, d + k)) { ++b2; break; }
  }
  if (b1) atomicAdd(bad + 1, b1);
  if (b2) atomicAdd(bad + 2, b2);
  if (blockIdx.x == 0 && threadIdx.x == 0 && so[0] != 0) atomicAdd(bad + 3, 1ull);
}

// order-independent sums of H(gidx, string): inputs (gidx = gbase + i) and
// outputs (gidx = perm[i]); equal multisets give equal sums
__global__ void k_hash(const uint8_t *units, const int64_t *off, const uint32_t *perm, uint64_t gbase, uint64_t n,
                       int w, unsigned long long *sum) {
  unsigned long long h = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = perm ? (uint64_t)perm[i] : gbase + i;
    h += hash_string(units, w, off[i], off[i + 1] - off[i], g);
  }
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xFFFFFFFFu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(sum, h);
}

inline unsigned grid_for(uint64_t n) {
  uint64_t b = (n + 255) / 256;
  return (unsigned)(b > 8192 ? 8192 : (b ? b : 1));
}

}  // namespace

extern "C" {

int check_pairs(const void *su, int w, const int64_t *so, const uint32_t *perm, uint64_t n,
                unsigned long long *bad, void *stream) {
  if (n > 1) k_pairs<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((const uint8_t *)su, w, so, perm, n, bad);
  return (int)cudaGetLastError();
}

int check_content(const void *units, const int64_t *off, uint64_t n_in, const void *su, const int64_t *so,
                  const uint32_t *perm, uint64_t n, int w, uint32_t *bitmap, unsigned long long *bad, void *stream) {
  if (n)
    k_content<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((const uint8_t *)units, off, n_in, (const uint8_t *)su,
                                                              so, perm, n, w, bitmap, bad);
  return (int)cudaGetLastError();
}

int check_hash(const void *units, const int64_t *off, const uint32_t *perm, uint64_t gbase, uint64_t n, int w,
               unsigned long long *sum, void *stream) {
  if (n) k_hash<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((const uint8_t *)units, off, perm, gbase, n, w, sum);
  return (int)cudaGetLastError();
}

}  // extern "C"
