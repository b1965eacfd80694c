// rand_probe3.cu -- lab microbenchmark (not product): random 16-B reads whose
// addresses stay inside a "bucket" of B records that advances with the
// position (what a gather sees when its sources were first partitioned by the
// top key bits): does bucket-local randomness run at L2 instead of DRAM rates?
// Optional sequential 32-B writes per position model the gather's output stream.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/rand_probe3 tools/rand_probe3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x = (x ^ (x >> 33)) * 0xFF51AFD7ED558CCDull;
  x = (x ^ (x >> 29)) * 0xC4CEB9FE1A85EC53ull;
  return x ^ (x >> 32);
}

// positions are processed in order (tile t = 1024 positions by one CTA, tiles by atomic counter)
template <bool WRITE>
__global__ void __launch_bounds__(256) k_probe(const uint4 *rec, uint64_t n, uint64_t bucket, uint4 *out,
                                              unsigned int *ctr, unsigned long long *sink) {
  __shared__ unsigned int s_t;
  uint64_t acc = 0;
  for (;;) {
    if (threadIdx.x == 0) s_t = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint64_t t = s_t;
    __syncthreads();
    if (t * 1024 >= n) break;
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t p = t * 1024 + k * 256 + threadIdx.x;
      const uint64_t b0 = (p / bucket) * bucket;
      v[k] = rec[b0 + mix(p) % bucket];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      acc += v[k].x ^ v[k].w;
      if (WRITE) {
        const uint64_t p = t * 1024 + k * 256 + threadIdx.x;
        out[2 * p] = v[k];
        out[2 * p + 1] = v[k];
      }
    }
  }
  if (acc == 42) atomicAdd(sink, acc);
}

int main() {
  const uint64_t n = 1ull << 30;
  uint4 *rec, *out;
  cudaMalloc(&rec, n * 16);
  cudaMalloc(&out, n * 32);
  cudaMemset(rec, 1, n * 16);
  unsigned int *ctr;
  unsigned long long *sink;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t buckets[] = {1ull << 30, 1ull << 26, 1ull << 24, 1ull << 23, 1ull << 22, 1ull << 21, 1ull << 20, 1ull << 18, 1ull << 16};
  for (int w = 0; w < 2; ++w) {
    for (uint64_t bk : buckets) {
      float ms = 0;
      for (int r = 0; r < 2; ++r) {
        cudaMemset(ctr, 0, 4);
        cudaEventRecord(a);
        if (w) k_probe<true><<<148 * 8, 256>>>(rec, n, bk, out, ctr, sink);
        else k_probe<false><<<148 * 8, 256>>>(rec, n, bk, out, ctr, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      cudaEventElapsedTime(&ms, a, b);
      printf("%s bucket %10llu records (%7.1f MB): %7.2f ms  %6.1f G reads/s  (%s)\n", w ? "read+write32" : "read only   ",
             (unsigned long long)bk, bk * 16 / 1e6, ms, n / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
