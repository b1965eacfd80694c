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
constexpr int kExchangeBytes = kRadixTile * (8 + 4) + kRadixWarps * 256 * 4;

template <bool SYNTH_VALS>
__global__ void __launch_bounds__(kRadixThreads, kRadixMinBlocks)
    k_onesweep(const uint64_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
               uint64_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out, uint64_t n, int shift,
               const uint32_t *__restrict__ digit_start, unsigned long long *lb, uint32_t *tile_counter,
               uint32_t epoch) {
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
    uint32_t pre = wc[d];
    rank[r] = pre + __popc(peers & lanemask_lt());
    __syncwarp();
    if (lane == 31 - __clz(peers)) wc[d] = pre + __popc(peers);
    __syncwarp();
  }
  __syncthreads();

  // ---- per digit (thread tid = digit): warp prefixes, tile count; the tile's
  // counts are published (aggregate) before anything else so successors can
  // consume them without waiting for this tile's own look-back.
  const uint32_t dg = tid;
  uint32_t tot = 0;
#pragma unroll
  for (int w = 0; w < kRadixWarps; ++w) {
    uint32_t c = cnt[w * 256 + dg];
    cnt[w * 256 + dg] = tot;
    tot += c;
  }
  uint64_t tile_end = tile_base + kRadixTile;
  if (dg == 255 && tile_end > n) tot -= (uint32_t)(tile_end - n);  // padding keys
  unsigned long long *my_flag = lb + (uint64_t)tile * 256 + dg;
  if (tile == 0) st_relaxed_u64(my_flag, make_flag(kFlagInc, epoch, (unsigned long long)digit_start[dg] + tot));
  else st_relaxed_u64(my_flag, make_flag(kFlagAgg, epoch, tot));
  uint32_t block_total;
  uint32_t local_start = block_exclusive_scan<uint32_t, kRadixThreads>(tot, &block_total, s_wt);
  s_local_start[dg] = local_start;
  __syncthreads();

  // ---- exchange through shared memory into tile-local digit order (frees the
  // key/value registers before the look-back)
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    uint32_t d = (uint32_t)(k[r] >> shift) & 0xFF;
    uint32_t pos = s_local_start[d] + wc[d] + rank[r];
    xk[pos] = k[r];
    xv[pos] = v[r];
  }

  // ---- windowed decoupled look-back (8 predecessor tiles per round trip)
  unsigned long long excl = tile == 0 ? (unsigned long long)digit_start[dg]
                                      : lookback_window<8>(lb + dg, tile, 256, epoch);
  if (tile != 0) st_relaxed_u64(my_flag, make_flag(kFlagInc, epoch, excl + tot));
  s_gbase[dg] = (uint32_t)excl - local_start;  // modular; global = gbase + local position
  __syncthreads();

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
  if (vals_in == nullptr)
    k_onesweep<true><<<g, b, kExchangeBytes, s>>>(keys_in, nullptr, keys_out, vals_out, n, 8 * digit, ds, lb,
                                                  tile_counter, epoch);
  else
    k_onesweep<false><<<g, b, kExchangeBytes, s>>>(keys_in, vals_in, keys_out, vals_out, n, 8 * digit, ds, lb,
                                                   tile_counter, epoch);
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
