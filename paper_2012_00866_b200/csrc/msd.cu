// msd.cu -- A2 key sort of (code, index), MSD-hybrid variant (opt-in with
// HUSKY_KEYSORT=msd; the default is the 8-pass LSD onesweep of radix.cu, which
// measured faster: DESIGN.md section 6.2).
//
// Role in the paper: step 2 of Alg. 1, "Sort array longs ... in such a way that
// when elements i, j of longs are exchanged, then elements i, j of xs are also
// exchanged".  The result is identical to the LSD
// sort: the unique (code, index) order (every pass below is stable, and the
// level-0 payload is in index order), so equal codes come out in index order
// (R7).
//
// Why MSD on B200: an LSD radix of 63-bit codes moves every key 8 times
// (8 x 24 B/key).  Here a bucket is partitioned only while it holds more than
// kMsdSmall keys; buckets are then finished in shared memory.  Uniform keys
// (C1, C3, C5) take 2 (1e7) or 3 (2^30) partition passes plus the local sort;
// heavy duplicates (C2) leave the partition as soon as their bucket is all-equal.
//
//   level 0   segment [0, n), digit = top varying byte of all codes (A1 fuses
//             the OR / NOT-AND of the codes, so this is exact)
//   level L   k_msd_hist    per segment: histogram of its digit + OR / NOT-AND
//             k_msd_plan    per segment: if its top varying byte is below the
//                           digit (speculated as parent digit - 1), re-queue it;
//                           else scan -> bucket starts; buckets > kMsdSmall keys
//                           continue (next list, other scratch buffer), buckets of
//                           2..kMsdSmall keys register with the local-sort window
//                           of their start, all-equal segments finish
//             k_msd_partition  onesweep tile (kRadixTile keys, warp match ranking,
//                           decoupled look-back per (tile, digit) that stops at
//                           the segment's first tile) scattering each bucket to
//                           the scratch buffer (continuing) or the home buffer
//   local     k_msd_local   window j sorts the span of the buckets that start in
//                           [j*W, (j+1)*W) (<= kMsdLocalCap keys) in shared memory:
//                           stable LSD over the bytes that vary inside the span.
//                           A span holds whole buckets only, so sorting it is
//                           sorting each of them (buckets are key ranges in order).
#include <algorithm>
#include <cstdio>

#include "husky_internal.cuh"
#include "kernels.cuh"
#include "host_common.h"

namespace husky {

constexpr int kMsdWarps = kRadixThreads / 32;
constexpr int kMsdXBytes = kRadixTile * (8 + 4) + kMsdWarps * 256 * 4;  // exchange + per-warp counters
constexpr int kHistThreads = 256, kHistItems = kRadixTile / kHistThreads;

__device__ __forceinline__ uint32_t top_byte(unsigned long long vm) { return (63u - (uint32_t)__clzll(vm)) >> 3; }

// 64-bit OR over the warp (two 32-bit reductions)
__device__ __forceinline__ unsigned long long warp_or64(unsigned long long x) {
  uint32_t lo = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)x), hi = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)(x >> 32));
  return ((unsigned long long)hi << 32) | lo;
}

// --------------------------------------------------------------- level 0
__global__ void k_msd_level0(DevState *st, MsdBufs B, uint32_t n) {
  const unsigned long long vm = st->key_or & st->key_nand;  // bits that differ between codes
  MsdSeg s;
  s.start = 0;
  s.len = vm ? n : 0;
  s.digit = vm ? top_byte(vm) : 0;
  s.tile0 = 0;
  s.buf = 0;
  s.flags = 0;
  B.segs[0][0] = s;
  st->msd_count[0] = vm ? 1u : 0u;
  st->msd_count[1] = 0;
  st->msd_all_equal = vm == 0;
  st->sorted_keys = (unsigned long long)(vm ? B.kh : B.k[0]);
}

// tile0 of every segment of `list` = exclusive prefix of their tile counts (one CTA)
__global__ void __launch_bounds__(1024) k_msd_tiles(DevState *st, MsdBufs B, int list) {
  __shared__ uint32_t wt[33];
  const uint32_t cnt = st->msd_count[list];
  MsdSeg *segs = B.segs[list];
  uint32_t running = 0;
  for (uint32_t c = 0; c < cnt; c += 1024) {
    const uint32_t i = c + threadIdx.x;
    const uint32_t t = i < cnt ? (uint32_t)((segs[i].len + (uint64_t)kRadixTile - 1) / kRadixTile) : 0u;
    uint32_t total;
    const uint32_t ex = block_exclusive_scan<uint32_t, 1024>(t, &total, wt);
    if (i < cnt) segs[i].tile0 = running + ex;
    running += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) st->msd_tiles[list] = running;
}

// tile -> segment map of `list` (a warp per segment)
__global__ void k_msd_tilemap(const DevState *st, MsdBufs B, int list) {
  const uint32_t cnt = st->msd_count[list];
  const uint32_t lane = lane_id();
  const uint32_t wstride = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t si = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; si < cnt; si += wstride) {
    const MsdSeg s = B.segs[list][si];
    const uint32_t nt = (uint32_t)((s.len + (uint64_t)kRadixTile - 1) / kRadixTile);
    for (uint32_t t = lane; t < nt; t += 32) B.tile_seg[list][s.tile0 + t] = si;
  }
}

__global__ void k_msd_seg_init(const DevState *st, MsdBufs B, int list) {
  const uint32_t cnt = st->msd_count[list];
  for (uint32_t s = blockIdx.x; s < cnt; s += gridDim.x) {
    B.hist[(uint64_t)s * 256 + threadIdx.x] = 0;
    if (threadIdx.x == 0) {
      B.seg_or[s] = 0;
      B.seg_nand[s] = 0;
    }
  }
}

// --------------------------------------------------------------- histogram
// Per tile of a segment: counts of the segment's digit (warp-private counters,
// match-aggregated) and the OR / NOT-AND of its keys.
__global__ void __launch_bounds__(kHistThreads) k_msd_hist(const DevState *st, MsdBufs B, int list) {
  __shared__ uint32_t wc[kHistThreads / 32][256];
  __shared__ unsigned long long s_or[kHistThreads / 32], s_nand[kHistThreads / 32];
  const uint32_t tile = blockIdx.x;
  if (tile >= st->msd_tiles[list]) return;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint32_t si = B.tile_seg[list][tile];
  const MsdSeg sg = B.segs[list][si];
  const uint64_t *keys = B.k[sg.buf];
  const uint64_t beg = sg.start + (uint64_t)(tile - sg.tile0) * kRadixTile;
  const uint64_t end = min(beg + (uint64_t)kRadixTile, (uint64_t)sg.start + sg.len);
  const int shift = 8 * (int)sg.digit;
  for (int i = tid; i < (kHistThreads / 32) * 256; i += kHistThreads) (&wc[0][0])[i] = 0;
  uint64_t k[kHistItems];
#pragma unroll
  for (int r = 0; r < kHistItems; ++r) {
    const uint64_t idx = beg + r * kHistThreads + tid;
    k[r] = idx < end ? __ldg(keys + idx) : 0ull;
  }
  __syncthreads();
  unsigned long long o = 0, na = 0;
  uint32_t *my = wc[warp];
#pragma unroll
  for (int r = 0; r < kHistItems; ++r) {
    const bool valid = beg + r * kHistThreads + tid < end;
    const uint32_t d = valid ? (uint32_t)(k[r] >> shift) & 0xFF : 256u;
    if (valid) {
      o |= k[r];
      na |= ~k[r];
    }
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    if (valid && lane == 31 - __clz(peers)) my[d] += __popc(peers);
    __syncwarp();
  }
  o = warp_or64(o);
  na = warp_or64(na);
  if (lane == 0) {
    s_or[warp] = o;
    s_nand[warp] = na;
  }
  __syncthreads();
  uint32_t c = 0;
#pragma unroll
  for (int w = 0; w < kHistThreads / 32; ++w) c += wc[w][tid];
  if (c) atomicAdd(&B.hist[(uint64_t)si * 256 + tid], c);
  if (tid == 0) {
    unsigned long long a = 0, b = 0;
#pragma unroll
    for (int w = 0; w < kHistThreads / 32; ++w) {
      a |= s_or[w];
      b |= s_nand[w];
    }
    atomicOr(&B.seg_or[si], a);
    atomicOr(&B.seg_nand[si], b);
  }
}

// --------------------------------------------------------------- plan
__global__ void __launch_bounds__(256) k_msd_plan(DevState *st, MsdBufs B, int list) {
  __shared__ uint32_t wt[9];
  const uint32_t si = blockIdx.x;
  if (si >= st->msd_count[list]) return;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  MsdSeg *segp = &B.segs[list][si];
  const MsdSeg sg = *segp;
  const int nxt = list ^ 1;
  const unsigned long long vm = B.seg_or[si] & B.seg_nand[si];
  if (vm != 0 && top_byte(vm) != sg.digit) {
    // the speculated digit is shared by all keys of the segment: re-queue it on
    // its real top varying byte (no data movement; same buffer)
    if (tid == 0) {
      const uint32_t j = atomicAdd(&st->msd_count[nxt], 1u);
      MsdSeg ns = sg;
      ns.digit = top_byte(vm);
      ns.flags = 0;
      B.segs[nxt][j] = ns;
      segp->flags = 0;
    }
    return;
  }
  // all-equal segment, or digit 0 (every bucket then holds equal keys): one
  // more pass moves it home and nothing continues
  const bool all_final = vm == 0 || sg.digit == 0;
  const uint32_t c = B.hist[(uint64_t)si * 256 + tid];
  uint32_t total;
  const uint32_t ex = block_exclusive_scan<uint32_t, 256>(c, &total, wt);
  const uint32_t start = sg.start + ex;
  B.hist[(uint64_t)si * 256 + tid] = start;
  const bool cont = !all_final && c > kMsdSmall;
  const uint32_t bits = __ballot_sync(0xFFFFFFFFu, cont);
  if (lane == 0) B.cont[(uint64_t)si * 8 + warp] = bits;
  if (cont) {
    const uint32_t j = atomicAdd(&st->msd_count[nxt], 1u);
    MsdSeg ns;
    ns.start = start;
    ns.len = c;
    ns.digit = sg.digit - 1;  // speculation: checked by the next level's plan
    ns.tile0 = 0;
    ns.buf = sg.buf ^ 1;
    ns.flags = 0;
    B.segs[nxt][j] = ns;
  } else if (!all_final && c >= 2) {
    const uint32_t w = start / kMsdWin;
    atomicMin(&B.win_lo[w], start);
    atomicMax(&B.win_hi[w], start + c);
  }
  if (tid == 0) {
    segp->flags = kSegPart;
    atomicAdd(&st->msd_keys_part, (unsigned long long)sg.len);
  }
}

// --------------------------------------------------------------- partition
// One kRadixTile-key tile of a segment: warp-striped loads, __match_any_sync ranking
// into per-warp digit counters (stable), the tile's digit counts published for
// the decoupled look-back, exchange through shared memory into digit order,
// scatter in runs of consecutive addresses to the scratch (continuing bucket)
// or home (final bucket) buffers.
__global__ void __launch_bounds__(kRadixThreads, kRadixMinBlocks)
    k_msd_partition(const DevState *st, MsdBufs B, int list, int level, uint32_t *tile_counter, uint32_t epoch) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t *xk = reinterpret_cast<uint64_t *>(smem);
  uint32_t *xv = reinterpret_cast<uint32_t *>(smem + kRadixTile * 8);
  uint32_t *cnt = reinterpret_cast<uint32_t *>(smem + kRadixTile * 12);
  __shared__ uint32_t s_tile, s_cont[8];
  __shared__ uint32_t s_local_start[256];
  __shared__ uint32_t s_gbase[256];
  __shared__ uint32_t s_wt[kMsdWarps + 1];

  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);  // dynamic ids: predecessors are resident
  for (int i = tid; i < kMsdWarps * 256; i += kRadixThreads) cnt[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  if (tile >= st->msd_tiles[list]) return;
  const uint32_t si = B.tile_seg[list][tile];
  const MsdSeg sg = B.segs[list][si];
  if (!(sg.flags & kSegPart)) return;  // re-queued segment: nothing moves this level
  if (tid < 8) s_cont[tid] = B.cont[(uint64_t)si * 8 + tid];
  const uint64_t beg = sg.start + (uint64_t)(tile - sg.tile0) * kRadixTile;
  const uint64_t end = min(beg + (uint64_t)kRadixTile, (uint64_t)sg.start + sg.len);
  const uint32_t n_valid = (uint32_t)(end - beg);
  const int shift = 8 * (int)sg.digit;
  const uint64_t *__restrict__ keys_in = B.k[sg.buf];
  const uint32_t *__restrict__ vals_in = level == 0 ? B.v_init : B.v[sg.buf];
  const bool synth = vals_in == nullptr;

  uint64_t k[kRadixItems];
  uint32_t v[kRadixItems];
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint32_t loc = warp * (kRadixItems * 32) + r * 32 + lane;
    if (loc < n_valid) {
      k[r] = __ldg(keys_in + beg + loc);
      v[r] = synth ? (uint32_t)(beg + loc) : __ldg(vals_in + beg + loc);
    } else {
      k[r] = ~0ull;
      v[r] = 0;
    }
  }
  const bool is_dg = tid < 256;
  const uint32_t dg = tid & 255;
  const uint32_t dstart = is_dg ? B.hist[(uint64_t)si * 256 + dg] : 0u;

  uint32_t *wc = cnt + warp * 256;
  uint32_t rank[kRadixItems];
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint32_t loc = warp * (kRadixItems * 32) + r * 32 + lane;
    const uint32_t d = loc < n_valid ? (uint32_t)(k[r] >> shift) & 0xFF : 256u;
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    uint32_t pre = d < 256 ? wc[d] : 0u;
    rank[r] = pre + __popc(peers & lanemask_lt());
    __syncwarp();
    if (d < 256 && lane == 31 - __clz(peers)) wc[d] = pre + __popc(peers);
    __syncwarp();
  }
  __syncthreads();

  uint32_t tot = 0;
  if (is_dg) {
#pragma unroll
    for (int w = 0; w < kMsdWarps; ++w) {
      const uint32_t c = cnt[w * 256 + dg];
      cnt[w * 256 + dg] = tot;
      tot += c;
    }
  }
  const bool first = tile == sg.tile0;
  unsigned long long *my_flag = B.lb + (uint64_t)tile * 256 + dg;
  if (is_dg) {
    if (first) st_relaxed_u64(my_flag, make_flag(kFlagInc, epoch, (unsigned long long)dstart + tot));
    else st_relaxed_u64(my_flag, make_flag(kFlagAgg, epoch, tot));
  }
  uint32_t block_total;
  const uint32_t local_start = block_exclusive_scan<uint32_t, kRadixThreads>(tot, &block_total, s_wt);
  if (is_dg) s_local_start[dg] = local_start;
  __syncthreads();

#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint32_t loc = warp * (kRadixItems * 32) + r * 32 + lane;
    if (loc < n_valid) {
      const uint32_t d = (uint32_t)(k[r] >> shift) & 0xFF;
      const uint32_t pos = s_local_start[d] + wc[d] + rank[r];
      xk[pos] = k[r];
      xv[pos] = v[r];
    }
  }

  if (is_dg) {
    unsigned long long excl;
    if (first) {
      excl = dstart;
    } else {
      excl = lookback_window<8>(B.lb + dg, tile, 256, epoch);
      st_relaxed_u64(my_flag, make_flag(kFlagInc, epoch, excl + tot));
    }
    s_gbase[dg] = (uint32_t)excl - local_start;
  }
  __syncthreads();

  uint64_t *__restrict__ knext = B.k[sg.buf ^ 1];
  uint32_t *__restrict__ vnext = B.v[sg.buf ^ 1];
#pragma unroll 4
  for (uint32_t i = tid; i < n_valid; i += kRadixThreads) {
    const uint64_t key = xk[i];
    const uint32_t d = (uint32_t)(key >> shift) & 0xFF;
    const uint32_t g = s_gbase[d] + i;
    if ((s_cont[d >> 5] >> (d & 31)) & 1u) {
      knext[g] = key;
      vnext[g] = xv[i];
    } else {
      B.kh[g] = key;
      B.vh[g] = xv[i];
    }
  }
}

// --------------------------------------------------------------- local sort
// small_n > 0: sort [0, small_n) from B.k[0] / B.v_init into the home buffers
// (the whole input fits one CTA); else window blockIdx.x, in place in home.
__global__ void __launch_bounds__(kRadixThreads, kRadixMinBlocks)
    k_msd_local(DevState *st, MsdBufs B, uint32_t small_n) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t *xk = reinterpret_cast<uint64_t *>(smem);
  uint32_t *xv = reinterpret_cast<uint32_t *>(smem + kRadixTile * 8);
  uint32_t *cnt = reinterpret_cast<uint32_t *>(smem + kRadixTile * 12);
  __shared__ uint32_t s_local_start[256];
  __shared__ uint32_t s_wt[kMsdWarps + 1];
  __shared__ unsigned long long s_vm[kMsdWarps];

  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  uint32_t lo, hi;
  const uint64_t *ksrc;
  const uint32_t *vsrc;
  if (small_n) {
    lo = 0;
    hi = small_n;
    ksrc = B.k[0];
    vsrc = B.v_init;
    if (tid == 0) st->sorted_keys = (unsigned long long)B.kh;
  } else {
    lo = B.win_lo[blockIdx.x];
    hi = B.win_hi[blockIdx.x];
    if (lo >= hi) return;
    ksrc = B.kh;
    vsrc = B.vh;
  }
  const uint32_t S = hi - lo;  // <= kMsdLocalCap
  const bool synth = vsrc == nullptr;
  uint64_t k[kRadixItems];
  uint32_t v[kRadixItems];
  const uint64_t k0 = __ldg(ksrc + lo);
  unsigned long long vm = 0;
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const uint32_t loc = warp * (kRadixItems * 32) + r * 32 + lane;
    if (loc < S) {
      k[r] = __ldg(ksrc + lo + loc);
      v[r] = synth ? lo + loc : __ldg(vsrc + lo + loc);
      vm |= k[r] ^ k0;
    } else {
      k[r] = 0;
      v[r] = 0;
    }
  }
  vm = warp_or64(vm);
  if (lane == 0) s_vm[warp] = vm;
  __syncthreads();
  vm = 0;
#pragma unroll
  for (int w = 0; w < kMsdWarps; ++w) vm |= s_vm[w];
  const bool warp_live = warp * (kRadixItems * 32) < S;  // warps past the span hold no keys
  const bool is_dg = tid < 256;
  const uint32_t dg = tid & 255;
  uint32_t *wc = cnt + warp * 256;
  for (int dgt = 0; dgt < 8; ++dgt) {
    if (((vm >> (8 * dgt)) & 0xFF) == 0) continue;  // byte shared by every key of the span
    const int shift = 8 * dgt;
    for (int i = tid; i < kMsdWarps * 256; i += kRadixThreads) cnt[i] = 0;
    __syncthreads();
    uint32_t rank[kRadixItems];
    if (warp_live) {
#pragma unroll
      for (int r = 0; r < kRadixItems; ++r) {
        const uint32_t loc = warp * (kRadixItems * 32) + r * 32 + lane;
        const uint32_t d = loc < S ? (uint32_t)(k[r] >> shift) & 0xFF : 256u;
        const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
        const uint32_t pre = d < 256 ? wc[d] : 0u;
        rank[r] = pre + __popc(peers & lanemask_lt());
        __syncwarp();
        if (d < 256 && lane == 31 - __clz(peers)) wc[d] = pre + __popc(peers);
        __syncwarp();
      }
    }
    __syncthreads();
    uint32_t tot = 0;
    if (is_dg) {
#pragma unroll
      for (int w = 0; w < kMsdWarps; ++w) {
        const uint32_t c = cnt[w * 256 + dg];
        cnt[w * 256 + dg] = tot;
        tot += c;
      }
    }
    uint32_t block_total;
    const uint32_t ls = block_exclusive_scan<uint32_t, kRadixThreads>(tot, &block_total, s_wt);
    if (is_dg) s_local_start[dg] = ls;
    __syncthreads();
    if (warp_live) {
#pragma unroll
      for (int r = 0; r < kRadixItems; ++r) {
        const uint32_t loc = warp * (kRadixItems * 32) + r * 32 + lane;
        if (loc < S) {
          const uint32_t d = (uint32_t)(k[r] >> shift) & 0xFF;
          const uint32_t pos = s_local_start[d] + wc[d] + rank[r];
          xk[pos] = k[r];
          xv[pos] = v[r];
        }
      }
    }
    __syncthreads();
    if (warp_live) {
#pragma unroll
      for (int r = 0; r < kRadixItems; ++r) {
        const uint32_t loc = warp * (kRadixItems * 32) + r * 32 + lane;
        if (loc < S) {
          k[r] = xk[loc];
          v[r] = xv[loc];
        }
      }
    }
  }
  if (vm == 0 && !small_n) return;  // equal keys, already in index order, in place
  if (warp_live) {
#pragma unroll
    for (int r = 0; r < kRadixItems; ++r) {
      const uint32_t loc = warp * (kRadixItems * 32) + r * 32 + lane;
      if (loc < S) {
        B.kh[lo + loc] = k[r];
        B.vh[lo + loc] = v[r];
      }
    }
  }
  if (tid == 0) atomicAdd(&st->msd_keys_local, (unsigned long long)S);
}

// all codes equal: the sorted keys are the codes, the payload is the index order
__global__ void k_msd_all_equal(const DevState *st, MsdBufs B, uint64_t n) {
  if (!st->msd_all_equal) return;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    B.vh[i] = B.v_init ? B.v_init[i] : (uint32_t)i;
}

// --------------------------------------------------------------- host driver
static void msd_configure() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k_msd_partition, cudaFuncAttributeMaxDynamicSharedMemorySize, kMsdXBytes);
  cudaFuncSetAttribute(k_msd_local, cudaFuncAttributeMaxDynamicSharedMemorySize, kMsdXBytes);
  done = true;
}

husky_status msd_key_sort(Sorter &S, const MsdBufs &B) {
  msd_configure();
  const uint64_t n = S.n;
  cudaStream_t s = S.s;
  DevState *st = S.st;
  if (n <= kMsdLocalCap) {
    HUSKY_SCOPE(ST_LOCAL_SORT, s, n);
    k_msd_local<<<1, kRadixThreads, kMsdXBytes, s>>>(st, B, (uint32_t)n);
    S.radix_passes = 0;
    return HUSKY_OK;
  }
  const uint64_t nwin = msd_windows(n);
  const unsigned map_grid = (unsigned)std::max(1, S.sms * 4);
  cudaMemsetAsync(B.win_lo, 0xFF, nwin * 4, s);
  cudaMemsetAsync(B.win_hi, 0, nwin * 4, s);
  {
    HUSKY_SCOPE(ST_HIST_SCAN, s, 0);
    k_msd_level0<<<1, 1, 0, s>>>(st, B, (uint32_t)n);
  }
  int list = 0, level = 0;
  uint32_t nsegs = 1;
  uint64_t tiles = radix_tiles_large(n);  // the MSD levels use kRadixTile-key tiles
  {
    HUSKY_SCOPE(ST_HIST_SCAN, s, 0);
    k_msd_tiles<<<1, 1024, 0, s>>>(st, B, 0);
  }
  {
    HUSKY_SCOPE(ST_HIST_SCAN, s, 0);
    k_msd_tilemap<<<map_grid, 256, 0, s>>>(st, B, 0);
  }
  for (;; ++level) {
    if (level >= 17) return fail(HUSKY_ERR_CUDA, "MSD key sort: level limit exceeded");
    {
      HUSKY_SCOPE(ST_HIST_SCAN, s, 0);
      k_msd_seg_init<<<std::min<uint32_t>(nsegs, 65535u), 256, 0, s>>>(st, B, list);
    }
    {
      HUSKY_SCOPE(ST_MSD_HIST, s, tiles * kRadixTile);
      k_msd_hist<<<(unsigned)tiles, kHistThreads, 0, s>>>(st, B, list);
    }
    cudaMemsetAsync(&st->msd_count[list ^ 1], 0, 4, s);
    {
      HUSKY_SCOPE(ST_HIST_SCAN, s, 0);
      k_msd_plan<<<nsegs, 256, 0, s>>>(st, B, list);
    }
    {
      HUSKY_SCOPE(ST_HIST_SCAN, s, 0);
      k_msd_tiles<<<1, 1024, 0, s>>>(st, B, list ^ 1);
    }
    {
      HUSKY_SCOPE(ST_HIST_SCAN, s, 0);
      k_msd_tilemap<<<map_grid, 256, 0, s>>>(st, B, list ^ 1);
    }
    {
      HUSKY_SCOPE(ST_RADIX, s, tiles * kRadixTile);
      k_msd_partition<<<(unsigned)tiles, kRadixThreads, kMsdXBytes, s>>>(st, B, list, level, S.next_counter(),
                                                                        S.next_epoch());
    }
    uint32_t nx[2] = {0, 0};
    cudaError_t e = cudaMemcpyAsync(&nx[0], &st->msd_count[list ^ 1], 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&nx[1], &st->msd_tiles[list ^ 1], 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(HUSKY_ERR_CUDA, "MSD key sort level %d: %s", level, cudaGetErrorString(e));
    if (nx[0] == 0) break;
    nsegs = nx[0];
    tiles = nx[1];
    list ^= 1;
  }
  {
    HUSKY_SCOPE(ST_LOCAL_SORT, s, n);
    k_msd_local<<<(unsigned)nwin, kRadixThreads, kMsdXBytes, s>>>(st, B, 0);
  }
  {
    HUSKY_SCOPE(ST_HIST_SCAN, s, 0);
    uint64_t blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)S.sms * 8);
    k_msd_all_equal<<<(unsigned)blocks, 256, 0, s>>>(st, B, n);
  }
  S.radix_passes = level + 1;
  return HUSKY_OK;
}

}  // namespace husky
