// rand_probe2.cu -- lab microbenchmark (not product): is random-read throughput
// bound by the SM side (L1 wavefronts: distinct lines per warp instruction) or
// by DRAM?  Random 32 B / 128 B blocks over a 16 GB buffer, read (a) one block
// per lane, (b) one block per group of lanes (coalesced inside the block),
// (c) by cp.async.bulk into shared memory (one bulk op per block, mbarrier).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/rand_probe2 tools/rand_probe2.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x = (x ^ (x >> 33)) * 0xFF51AFD7ED558CCDull;
  return x ^ (x >> 29);
}

// G lanes cooperate on one block of G*16 bytes; each lane loads ITEMS blocks' parts
template <int G, int ITEMS>
__global__ void k_group(const uint4 *buf, uint64_t blocks, uint64_t nblocks_total, unsigned long long *sink) {
  const uint32_t lane = threadIdx.x & 31, sub = lane % G, grp = lane / G;
  constexpr int GPW = 32 / G;  // blocks per warp instruction
  uint64_t acc = 0;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t b0 = warp * GPW * ITEMS; b0 < nblocks_total; b0 += nwarps * GPW * ITEMS) {
    uint4 v[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint64_t id = b0 + k * GPW + grp;
      v[k] = __ldg(buf + (mix(id) % blocks) * G + sub);
    }
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) acc += v[k].x ^ v[k].w;
  }
  if (acc == 42) atomicAdd(sink, acc);
}

// bulk copies: each thread issues ITEMS bulk copies of BYTES into smem, one mbarrier per warp
template <int BYTES, int ITEMS>
__global__ void k_bulk(const uint8_t *buf, uint64_t blocks, uint64_t nblocks_total, unsigned long long *sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[32];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t *my = sm + (size_t)threadIdx.x * BYTES * ITEMS;
  const uint32_t bar_addr = (uint32_t)__cvta_generic_to_shared(&bar[w]);
  if (lane == 0) asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(bar_addr), "r"(1));
  __syncwarp();
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  uint32_t phase = 0;
  uint64_t acc = 0;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b0 = tid * ITEMS; b0 < nblocks_total; b0 += nth * ITEMS) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar_addr), "r"(32 * BYTES * ITEMS)
                   : "memory");
    __syncwarp();
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
      const uint8_t *src = buf + (mix(b0 + k) % blocks) * BYTES;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(my + k * BYTES);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "l"(src), "r"(BYTES), "r"(bar_addr)
                   : "memory");
    }
    // wait
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(bar_addr), "r"(phase)
          : "memory");
    }
    phase ^= 1;
    acc += my[0] ^ my[BYTES * ITEMS - 1];
    __syncwarp();
  }
  if (acc == 42) atomicAdd(sink, acc);
}

int main(int argc, char **argv) {
  if (argc > 1) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[1]));
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("cudaLimitMaxL2FetchGranularity set %s -> %zu\n", cudaGetErrorString(e), v);
  } else {
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("cudaLimitMaxL2FetchGranularity default %zu\n", v);
  }
  const uint64_t bytes = 16ull << 30;
  uint8_t *buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t nb = 1ull << 27;
  auto run = [&](const char *name, auto launch, uint64_t count, int blockbytes) {
    float ms = 0;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("%-44s %7.1f G blocks/s  %7.0f GB/s  (%s)\n", name, count / (ms * 1e6), count * (double)blockbytes / (ms * 1e6),
           cudaGetErrorString(cudaGetLastError()));
  };
  const uint4 *b4 = (const uint4 *)buf;
  run("32B per lane-pair (G=2, 16 blocks/instr)", [&] { k_group<2, 8><<<148 * 8, 256>>>(b4, bytes / 32, nb, sink); }, nb, 32);
  run("16B per lane (G=1)", [&] { k_group<1, 8><<<148 * 8, 256>>>(b4, bytes / 16, nb, sink); }, nb, 16);
  run("64B per 4 lanes (G=4)", [&] { k_group<4, 8><<<148 * 8, 256>>>(b4, bytes / 64, nb, sink); }, nb, 64);
  run("128B per 8 lanes (G=8)", [&] { k_group<8, 8><<<148 * 8, 256>>>(b4, bytes / 128, nb, sink); }, nb, 128);
  run("256B per 16 lanes (G=16)", [&] { k_group<16, 8><<<148 * 8, 256>>>(b4, bytes / 256, nb, sink); }, nb, 256);
  cudaFuncSetAttribute(k_bulk<32, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 32 * 8);
  run("bulk 32B x8 per thread", [&] { k_bulk<32, 8><<<148 * 4, 256, 256 * 32 * 8>>>(buf, bytes / 32, nb, sink); }, nb, 32);
  cudaFuncSetAttribute(k_bulk<64, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 64 * 4);
  run("bulk 64B x4 per thread", [&] { k_bulk<64, 4><<<148 * 4, 256, 256 * 64 * 4>>>(buf, bytes / 64, nb, sink); }, nb, 64);
  cudaFuncSetAttribute(k_bulk<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 128 * 2);
  run("bulk 128B x2 per thread", [&] { k_bulk<128, 2><<<148 * 4, 256, 256 * 128 * 2>>>(buf, bytes / 128, nb, sink); }, nb, 128);
  return 0;
}
