// rand_probe.cu -- lab microbenchmark (not product): throughput of random
// 16-byte reads over buffers of growing size (TLB reach vs working set), with
// and without a dependent first hop (index -> offset -> data, like the gather).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/rand_probe tools/rand_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x = (x ^ (x >> 33)) * 0xFF51AFD7ED558CCDull;
  return x ^ (x >> 29);
}

// independent random reads: each thread ITEMS reads of 16 B at random 16-B slots
template <int ITEMS>
__global__ void k_rand(const uint4 *buf, uint64_t slots, uint64_t n, unsigned long long *sink) {
  uint64_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x * ITEMS + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x * ITEMS) {
    uint4 v[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) v[k] = __ldg(buf + mix(i + k * blockDim.x) % slots);
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) acc += v[k].x ^ v[k].w;
  }
  if (acc == 42) atomicAdd(sink, acc);
}

// dependent: idx[i] (sequential) -> off = tab[idx] (random 8 B) -> data at off (random 16 B)
template <int ITEMS>
__global__ void k_chain(const uint32_t *idx, const uint64_t *tab, const uint4 *buf, uint64_t n,
                        unsigned long long *sink) {
  uint64_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x * ITEMS + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x * ITEMS) {
    uint64_t o[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) o[k] = tab[idx[i + k * blockDim.x]];
    uint4 v[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) v[k] = __ldg(buf + o[k]);
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) acc += v[k].x ^ v[k].w;
  }
  if (acc == 42) atomicAdd(sink, acc);
}

// random reads of W consecutive uint4 (16*W bytes, aligned to 16*W)
template <int ITEMS, int W>
__global__ void k_randw(const uint4 *buf, uint64_t blocks, uint64_t n, unsigned long long *sink) {
  uint64_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x * ITEMS + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x * ITEMS) {
    uint4 v[ITEMS][W];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint4 *p = buf + (mix(i + k * blockDim.x) % blocks) * W;
#pragma unroll
      for (int w = 0; w < W; ++w) v[k][w] = __ldg(p + w);
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k)
#pragma unroll
      for (int w = 0; w < W; ++w) acc += v[k][w].x ^ v[k][w].w;
  }
  if (acc == 42) atomicAdd(sink, acc);
}
// random 4-byte / 16-byte writes
template <int W>
__global__ void k_rwrite(uint4 *buf, uint64_t slots, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s = mix(i) % slots;
    if (W == 0) reinterpret_cast<uint32_t *>(buf)[s * 4 + (i & 3)] = (uint32_t)i;
    else buf[s] = make_uint4((uint32_t)i, 1, 2, 3);
  }
}

__global__ void k_init_idx(uint32_t *idx, uint64_t n, uint64_t m) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    idx[i] = (uint32_t)(mix(i * 7 + 3) % m);
}
__global__ void k_init_tab(uint64_t *tab, uint64_t m, uint64_t slots) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    tab[i] = mix(i * 13 + 1) % slots;
}

int main() {
  const uint64_t n = 1ull << 28;  // reads per launch
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  uint32_t *idx;
  cudaMalloc(&idx, n * 4 + 64 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (double gb : {0.125, 0.5, 2.0, 8.0, 16.0, 32.0}) {
    const uint64_t bytes = (uint64_t)(gb * (1ull << 30));
    const uint64_t slots = bytes / 16;
    uint4 *buf;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) { printf("alloc fail %.1f\n", gb); break; }
    cudaMemset(buf, 1, bytes);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      k_rand<8><<<148 * 8, 256>>>(buf, slots, n, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    // chain: table of m = slots/2 entries (8 B each, its own buffer of m*8 B)
    const uint64_t m = slots / 2 < (1ull << 31) ? slots / 2 : (1ull << 31);
    uint64_t *tab;
    float ms2 = -1;
    if (cudaMalloc(&tab, m * 8) == cudaSuccess) {
      k_init_idx<<<4096, 256>>>(idx, n + 16384, m);
      k_init_tab<<<4096, 256>>>(tab, m, slots);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k_chain<8><<<148 * 8, 256>>>(idx, tab, buf, n, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      cudaEventElapsedTime(&ms2, a, b);
      cudaFree(tab);
    }
    float m32, m64, m128, w4, w16;
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); k_randw<8, 2><<<148 * 8, 256>>>(buf, slots / 2, n, sink); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&m32, a, b);
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); k_randw<4, 4><<<148 * 8, 256>>>(buf, slots / 4, n, sink); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&m64, a, b);
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); k_randw<2, 8><<<148 * 8, 256>>>(buf, slots / 8, n, sink); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&m128, a, b);
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); k_rwrite<0><<<148 * 8, 256>>>(buf, slots, n); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&w4, a, b);
    for (int rep = 0; rep < 2; ++rep) { cudaEventRecord(a); k_rwrite<1><<<148 * 8, 256>>>(buf, slots, n); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&w16, a, b);
    printf("   random aligned 32B %.1f G/s, 64B %.1f G/s, 128B %.1f G/s | random writes 4B %.1f G/s, 16B %.1f G/s\n",
           n / (m32 * 1e6), n / (m64 * 1e6), n / (m128 * 1e6), n / (w4 * 1e6), n / (w16 * 1e6));
    printf("buf %6.2f GB: random 16B reads %.1f G/s (%.0f GB/s of 32B sectors) | chain idx->8B->16B %.1f G/s "
           "(table %.2f GB)\n",
           gb, n / (ms * 1e6), n * 32.0 / (ms * 1e6), ms2 > 0 ? n / (ms2 * 1e6) : -1.0, m * 8 / 1e9);
    cudaFree(buf);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
