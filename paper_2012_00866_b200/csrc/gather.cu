// gather.cu -- A4: sorted-string gather.
//
// The paper's co-swap moves object references with the keys;
// here the strings themselves are materialised in sorted order once, after the
// permutation is final:
//   sorted_offsets = exclusive scan of len[perm[i]]  (single pass, look-back)
//   sorted_units   = concatenation of units[offsets[perm[i]] ..)
// A tile of 1024 sorted positions stages its strings in shared memory at the
// byte alignment of its output range (gathers are inherently scattered reads),
// then writes the range with aligned 16-byte stores; only the two boundary
// chunks use byte stores, so neighbouring tiles never race.
#include "husky_internal.cuh"
#include "kernels.cuh"

namespace husky {

template <int CODER>
__global__ void __launch_bounds__(kGatherThreads)
    k_gather(const uint32_t *__restrict__ perm, uint64_t n, const void *__restrict__ units,
             const int64_t *__restrict__ offsets, void *__restrict__ sorted_units,
             int64_t *__restrict__ sorted_offsets, unsigned long long *lb, uint32_t *tile_counter,
             uint32_t epoch, const int64_t *base_ptr) {
  constexpr int W = CoderTraits<CODER>::kUnitBytes;
  __shared__ __align__(16) uint8_t stage[kGatherStage + 16];
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_wt[kGatherThreads / 32 + 1];
  __shared__ unsigned long long s_base;
  const uint32_t tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  // re-gather of a span: output positions start at *base_ptr (unchanged by us)
  const unsigned long long gbase = base_ptr ? (unsigned long long)*base_ptr : 0ull;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t p0 = (uint64_t)tile * kGatherTile + (uint64_t)tid * kGatherItems;

  uint32_t idx[kGatherItems];
#pragma unroll
  for (int j = 0; j < kGatherItems; ++j) idx[j] = p0 + j < n ? __ldg(perm + p0 + j) : 0xFFFFFFFFu;
  int64_t src[kGatherItems];
  uint64_t len[kGatherItems];
  unsigned long long mine = 0;
#pragma unroll
  for (int j = 0; j < kGatherItems; ++j) {
    if (idx[j] != 0xFFFFFFFFu) {
      int64_t a = __ldg(offsets + idx[j]), b = __ldg(offsets + idx[j] + 1);
      src[j] = a;
      len[j] = (uint64_t)(b - a);
    } else {
      src[j] = 0;
      len[j] = 0;
    }
    mine += len[j];
  }
  unsigned long long tile_total;
  unsigned long long excl_t = block_exclusive_scan<unsigned long long, kGatherThreads>(mine, &tile_total, s_wt);
  if (tid == 0) {
    unsigned long long *f = lb + tile;
    unsigned long long ex;
    if (tile == 0) {
      ex = 0;
      st_relaxed_u64(f, make_flag(kFlagInc, epoch, tile_total));
    } else {
      st_relaxed_u64(f, make_flag(kFlagAgg, epoch, tile_total));
      ex = lookback(lb, tile, 1, epoch);
      st_relaxed_u64(f, make_flag(kFlagInc, epoch, ex + tile_total));
    }
    s_base = ex;
    if ((uint64_t)(tile + 1) * kGatherTile >= n) sorted_offsets[n] = (int64_t)(gbase + ex + tile_total);
  }
  __syncthreads();
  const unsigned long long tbase = gbase + s_base;  // units before this tile
  {
    unsigned long long d = tbase + excl_t;
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
      if (p0 + j < n) sorted_offsets[p0 + j] = (int64_t)d;
      d += len[j];
    }
  }
  if (sorted_units == nullptr) return;

  const uint8_t *ub = (const uint8_t *)units;
  uint8_t *ob = (uint8_t *)sorted_units;
  const uint64_t tile_bytes = tile_total * W;
  uint8_t *g0 = ob + tbase * W;  // first output byte of the tile
  if (tile_bytes + 16 <= (uint64_t)kGatherStage) {
    const uint32_t align = (uint32_t)((uintptr_t)g0 & 15);
    uint64_t d = (uint64_t)align + excl_t * W;
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
      uint64_t nb = len[j] * W;
      const uint8_t *sp = ub + src[j] * W;
      for (uint64_t c = 0; c < nb; c += 8) {
        int take = (int)(nb - c < 8 ? nb - c : 8);
        uint64_t v = load8_unaligned(sp + c, take);
        for (int b = 0; b < take; ++b) stage[d + c + b] = (uint8_t)(v >> (8 * b));
      }
      d += nb;
    }
    __syncthreads();
    // write [g0, g0 + tile_bytes) = stage[align, align + tile_bytes)
    uint8_t *a0 = g0 - align;  // 16-aligned
    const uint64_t end = align + tile_bytes;
    const uint64_t nchunks = (end + 15) / 16;
    for (uint64_t ch = tid; ch < nchunks; ch += kGatherThreads) {
      uint64_t lo = ch * 16, hi = lo + 16;
      if (lo >= align && hi <= end) {
        *reinterpret_cast<uint4 *>(a0 + lo) = *reinterpret_cast<const uint4 *>(stage + lo);
      } else {
        for (uint64_t b = (lo > align ? lo : align); b < (hi < end ? hi : end); ++b) a0[b] = stage[b];
      }
    }
  } else {
    // long strings: warp-cooperative byte copy, one string at a time per warp
    const uint32_t lane = lane_id(), warp = tid >> 5;
    for (int t = 0; t < 32; ++t) {
      uint32_t owner = warp * 32 + t;
      uint64_t d = tbase + __shfl_sync(0xFFFFFFFFu, excl_t, t);
#pragma unroll
      for (int j = 0; j < kGatherItems; ++j) {
        int64_t s = __shfl_sync(0xFFFFFFFFu, src[j], t);
        uint64_t l = __shfl_sync(0xFFFFFFFFu, len[j], t);
        uint64_t nb = l * W;
        for (uint64_t b = lane; b < nb; b += 32) ob[d * W + b] = ub[s * W + b];
        d += l;
      }
      (void)owner;
    }
  }
}

void launch_gather(int coder, const uint32_t *perm, uint64_t n, const void *units,
                   const int64_t *offsets, void *sorted_units, int64_t *sorted_offsets,
                   unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, cudaStream_t s,
                   const int64_t *base_ptr) {
  if (n == 0) return;
  Scope sc_(ST_GATHER, s, n);
  dim3 g((unsigned)gather_tiles(n)), b(kGatherThreads);
  if (coder == HUSKY_CODER_ASCII)
    k_gather<HUSKY_CODER_ASCII><<<g, b, 0, s>>>(perm, n, units, offsets, sorted_units, sorted_offsets, lb,
                                                tile_counter, epoch, base_ptr);
  else
    k_gather<HUSKY_CODER_UNICODE><<<g, b, 0, s>>>(perm, n, units, offsets, sorted_units, sorted_offsets, lb,
                                                  tile_counter, epoch, base_ptr);
}

// Re-gather the spans of the small/medium dirty runs after their fix-up
// rewrote perm inside them (the span [start, start+len) and its total length
// are unchanged; only the order inside moves).  One CTA per run.
template <int CODER>
__global__ void __launch_bounds__(256)
    k_regather_runs(const uint2 *__restrict__ list, uint64_t cap, const DevState *st,
                    const uint32_t *__restrict__ perm, const void *__restrict__ units,
                    const int64_t *__restrict__ offsets, void *__restrict__ sorted_units,
                    int64_t *__restrict__ sorted_offsets) {
  constexpr int W = CoderTraits<CODER>::kUnitBytes;
  __shared__ unsigned long long s_wt[256 / 32 + 1];
  const uint32_t ns = st->n_small, nm = st->n_medium;
  const uint8_t *ub = (const uint8_t *)units;
  uint8_t *ob = (uint8_t *)sorted_units;
  for (uint32_t e = blockIdx.x; e < ns + nm; e += gridDim.x) {
    uint2 ent = e < ns ? list[e] : list[cap - 1 - (e - ns)];
    const uint32_t start = ent.x, len = ent.y;
    const unsigned long long base = (unsigned long long)sorted_offsets[start];
    unsigned long long running = 0;
    for (uint32_t c = 0; c < len; c += 256) {
      uint32_t k = c + threadIdx.x;
      bool valid = k < len;
      uint32_t i = valid ? perm[start + k] : 0u;
      int64_t o = valid ? offsets[i] : 0;
      unsigned long long L = valid ? (unsigned long long)(offsets[i + 1] - o) : 0ull;
      unsigned long long tot;
      unsigned long long ex = block_exclusive_scan<unsigned long long, 256>(L, &tot, s_wt);
      unsigned long long d = base + running + ex;
      if (valid) {
        sorted_offsets[start + k] = (int64_t)d;
        uint64_t nb = L * W;
        const uint8_t *sp = ub + o * W;
        uint8_t *dp = ob + d * W;
        for (uint64_t q = 0; q < nb; q += 8) {
          int take = (int)(nb - q < 8 ? nb - q : 8);
          uint64_t v = load8_unaligned(sp + q, take);
          for (int b = 0; b < take; ++b) dp[q + b] = (uint8_t)(v >> (8 * b));
        }
      }
      running += tot;
      __syncthreads();
    }
  }
}

void launch_regather_runs(int coder, const uint2 *list_sm, uint64_t cap_sm, const DevState *st,
                          const uint32_t *perm, const void *units, const int64_t *offsets,
                          void *sorted_units, int64_t *sorted_offsets, int num_sms, cudaStream_t s) {
  Scope sc_(ST_FIX_SMALL, s, 0);
  dim3 g(num_sms * 4), b(256);
  if (coder == HUSKY_CODER_ASCII)
    k_regather_runs<HUSKY_CODER_ASCII><<<g, b, 0, s>>>(list_sm, cap_sm, st, perm, units, offsets, sorted_units,
                                                       sorted_offsets);
  else
    k_regather_runs<HUSKY_CODER_UNICODE><<<g, b, 0, s>>>(list_sm, cap_sm, st, perm, units, offsets, sorted_units,
                                                         sorted_offsets);
}

}  // namespace husky
