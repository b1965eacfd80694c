// radix.cu -- A2: stable onesweep LSD radix sort of (64-bit key, 32-bit payload).
//
// Role in the paper: step 2 of Alg. 1, "Sort array longs ... in such a way that
// when elements i, j of longs are exchanged, then elements i, j of xs are also
// exchanged".  Introsort's comparisons are replaced
// by an 8-bit-digit LSD radix sort whose payload is the string index, so the
// co-swap is the payload scatter.  Being stable, it leaves equal codes in index
// order (R7), which the fix-up (A5) relies on.
//
// Per pass (one launch): a tile of 4096 keys (256 threads x 16, warp-striped so
// every load/store instruction is a coalesced 256-B access) is ranked in shared
// memory with warp-level match (__match_any_sync) + popc ranking into per-warp
// digit counters; the tile's digit counts are published to a per-(tile, digit)
// decoupled look-back array; the global digit base comes from the histograms the
// encoder fused into A1 (exclusive-scanned by k_hist_scan).  Keys are then
// exchanged through shared memory into digit order and written out as runs of
// consecutive addresses.  Tile ids come from an atomic counter, so every
// predecessor a tile waits on is already resident (forward progress).
#include "husky_internal.cuh"
#include "kernels.cuh"

namespace husky {

// Exclusive scan of hist[d][0..255] -> digit_start[d]; trivial_mask bit d when
// one digit value holds all n keys (that pass is the identity and is skipped).
__global__ void __launch_bounds__(256) k_hist_scan(uint64_t n, DevState *st) {
  __shared__ uint32_t wt[9];
  const int d = blockIdx.x;
  uint32_t v = st->hist[d][threadIdx.x];
  uint32_t total;
  uint32_t ex = block_exclusive_scan<uint32_t, 256>(v, &total, wt);
  st->digit_start[d][threadIdx.x] = ex;
  if ((uint64_t)v == n) atomicOr(&st->trivial_mask, 1u << d);
}

void launch_hist_scan(uint64_t n, DevState *st, cudaStream_t s) {
  Scope sc_(ST_HIST_SCAN, s, n);
  k_hist_scan<<<8, 256, 0, s>>>(n, st);
}

constexpr int kRadixWarps = kRadixThreads / 32;
#ifndef RADIX_LB_W
#define RADIX_LB_W 16
#endif

#ifdef HUSKY_TIMING
// per-tile phase timestamps of the last onesweep launch (instrumented builds only)
constexpr int kTimingTiles = 8192;
__device__ unsigned long long g_tile_times[kTimingTiles][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define HT(tile, i) \
  do { if (threadIdx.x == 0 && (tile) < kTimingTiles) g_tile_times[tile][i] = gtimer(); } while (0)
#else
#define HT(tile, i) do { } while (0)
#endif
constexpr int kExchangeBytes = kRadixTile * (8 + 4) + kRadixWarps * 256 * 4;

template <bool SYNTH_VALS>
__global__ void __launch_bounds__(kRadixThreads, kRadixMinBlocks)
    k_onesweep(const uint64_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
               uint64_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out, uint64_t n, int shift,
               const uint32_t *__restrict__ digit_start, unsigned long long *lb, uint32_t *tile_counter,
               uint32_t epoch, uint64_t lb_stride) {
  extern __shared__ __align__(16) uint8_t smem[];
  // key/value exchange buffer, then per-warp digit counters [warps][256]
  uint64_t *xk = reinterpret_cast<uint64_t *>(smem);
  uint32_t *xv = reinterpret_cast<uint32_t *>(smem + kRadixTile * 8);
  uint32_t *cnt = reinterpret_cast<uint32_t *>(smem + kRadixTile * 12);
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_local_start[256];
  __shared__ uint32_t s_gbase[256];
  __shared__ uint32_t s_wt[kRadixWarps + 1];

  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < kRadixWarps * 256; i += kRadixThreads) cnt[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t tile_base = (uint64_t)tile * kRadixTile;
  HT(tile, 0);

  // ---- load (warp-striped: element = tile_base + warp*512 + r*32 + lane)
  uint64_t k[kRadixItems];
  uint32_t v[kRadixItems];
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    uint64_t idx = tile_base + warp * (kRadixItems * 32) + r * 32 + lane;
    if (idx < n) {
      k[r] = __ldg(keys_in + idx);
      v[r] = SYNTH_VALS ? (uint32_t)idx : __ldg(vals_in + idx);
    } else {
      k[r] = ~0ull;  // ranks last in digit 255; never stored
      v[r] = 0;
    }
  }

  // ---- warp-level match ranking into per-warp counters (stable: (r, lane) order)
  uint32_t *wc = cnt + warp * 256;
  uint32_t rank[kRadixItems];
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    uint32_t d = (uint32_t)(k[r] >> shift) & 0xFF;
    uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    if (r == 0) HT(tile, 1);
    uint32_t pre = wc[d];
    rank[r] = pre + __popc(peers & lanemask_lt());
    __syncwarp();
    if (lane == 31 - __clz(peers)) wc[d] = pre + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  HT(tile, 2);

  // ---- per digit (thread tid = digit): warp prefixes, tile count; the tile's
  // counts are published (aggregate) before anything else so successors can
  // consume them without waiting for this tile's own look-back.
  // threads 0..255 own one digit each (the CTA may have more threads)
  const bool is_dg = tid < 256;
  const uint32_t dg = tid & 255;
  uint32_t tot = 0;
  if (is_dg) {
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      uint32_t c = cnt[w * 256 + dg];
      cnt[w * 256 + dg] = tot;
      tot += c;
    }
  }
  uint64_t tile_end = tile_base + kRadixTile;
  if (is_dg && dg == 255 && tile_end > n) tot -= (uint32_t)(tile_end - n);  // padding keys
  unsigned long long *my_flag = lb + (uint64_t)tile * 256 + dg;
  (void)lb_stride;
  if (is_dg) {
    if (tile == 0) st_relaxed_u64(my_flag, make_flag(kFlagInc, epoch, (unsigned long long)digit_start[dg] + tot));
    else st_relaxed_u64(my_flag, make_flag(kFlagAgg, epoch, tot));
  }
  uint32_t block_total;
  uint32_t local_start = block_exclusive_scan<uint32_t, kRadixThreads>(tot, &block_total, s_wt);
  if (is_dg) s_local_start[dg] = local_start;
  __syncthreads();
  HT(tile, 3);

  // ---- exchange through shared memory into tile-local digit order (frees the
  // key/value registers before the look-back)
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    uint32_t d = (uint32_t)(k[r] >> shift) & 0xFF;
    uint32_t pos = s_local_start[d] + wc[d] + rank[r];
    xk[pos] = k[r];
    xv[pos] = v[r];
  }

  // ---- decoupled look-back, RADIX_LB_W predecessor tiles per round trip
  if (is_dg) {
#ifdef HUSKY_TIMING
    uint32_t lbst[2] = {0, 0};
    unsigned long long excl = tile == 0 ? (unsigned long long)digit_start[dg]
                                        : lookback_window<RADIX_LB_W>(lb + dg, tile, 256, epoch, lbst);
    if (tid == 0 && tile < kTimingTiles) g_tile_times[tile][7] = lbst[0] | ((unsigned long long)lbst[1] << 32);
#else
    unsigned long long excl = tile == 0 ? (unsigned long long)digit_start[dg]
                                        : lookback_window<RADIX_LB_W>(lb + dg, tile, 256, epoch);
#endif
    if (tile != 0) st_relaxed_u64(my_flag, make_flag(kFlagInc, epoch, excl + tot));
    if (tid == 0) HT(tile, 4);  // thread 0's own look-back done
    s_gbase[dg] = (uint32_t)excl - local_start;  // modular; global = gbase + local position
  }
  __syncthreads();
  HT(tile, 5);

  // ---- scatter: consecutive local positions of a digit -> consecutive addresses
  uint32_t n_valid = (uint32_t)((n - tile_base) < (uint64_t)kRadixTile ? (n - tile_base) : kRadixTile);
#pragma unroll 4
  for (uint32_t i = tid; i < n_valid; i += kRadixThreads) {
    uint64_t key = xk[i];
    uint32_t d = (uint32_t)(key >> shift) & 0xFF;
    uint32_t g = s_gbase[d] + i;
    keys_out[g] = key;
    vals_out[g] = xv[i];
  }
  HT(tile, 6);
}

// instrumented builds: copy the per-tile phase timestamps of the last pass
extern "C" int husky_debug_tile_times(unsigned long long *out, int max_tiles) {
#ifdef HUSKY_TIMING
  int k = max_tiles < kTimingTiles ? max_tiles : kTimingTiles;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_tile_times, (size_t)k * 8 * sizeof(unsigned long long));
  return k;
#else
  (void)out;
  (void)max_tiles;
  return 0;
#endif
}

void launch_onesweep(const uint64_t *keys_in, const uint32_t *vals_in, uint64_t *keys_out,
                     uint32_t *vals_out, uint64_t n, int digit, DevState *st,
                     unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, cudaStream_t s) {
  if (n == 0) return;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_onesweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kExchangeBytes);
    cudaFuncSetAttribute(k_onesweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kExchangeBytes);
    configured = true;
  }
  Scope sc_(ST_RADIX, s, n);
  dim3 g((unsigned)radix_tiles(n)), b(kRadixThreads);
  const uint32_t *ds = st->digit_start[digit];
  const uint64_t stride = radix_lb_stride(n);
  if (vals_in == nullptr)
    k_onesweep<true><<<g, b, kExchangeBytes, s>>>(keys_in, nullptr, keys_out, vals_out, n, 8 * digit, ds, lb,
                                                  tile_counter, epoch, stride);
  else
    k_onesweep<false><<<g, b, kExchangeBytes, s>>>(keys_in, vals_in, keys_out, vals_out, n, 8 * digit, ds, lb,
                                                   tile_counter, epoch, stride);
}

__global__ void k_iota(uint32_t *perm, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    perm[i] = (uint32_t)i;
}

void launch_iota(uint32_t *perm, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  Scope sc_(ST_RADIX, s, 0);
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_iota<<<(unsigned)blocks, 256, 0, s>>>(perm, n);
}

}  // namespace husky
