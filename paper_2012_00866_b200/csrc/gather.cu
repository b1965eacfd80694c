// gather.cu -- A4: sorted-string gather.
//
// The paper's co-swap moves object references with the keys;
// here the strings themselves are materialised in sorted order:
//   sorted_offsets = exclusive scan of len[perm[i]]  (single pass, look-back)
//   sorted_units   = concatenation of units[offsets[perm[i]] ..)
// A tile of 1024 sorted positions: perm (coalesced) -> offsets (random) ->
// tile-local scan; the tile's aggregate is published, then every thread stages
// its strings into shared memory at tile-local byte offsets (random reads,
// independent of the look-back), warp 0 resolves the tile's global base with a
// warp-wide look-back (32 predecessors per round trip), and the tile's output
// range is written with aligned 16-byte stores (funnel-shifted out of smem);
// only the two boundary chunks use byte stores, so neighbouring tiles never race.
#include "husky_internal.cuh"
#include "kernels.cuh"

namespace husky {

// Byte b of a string whose units are fully determined by its husky code (ASCII
// length <= 9, UNICODE length <= 3): the inverse of Alg. 4's packing.
template <int CODER>
__device__ __forceinline__ uint8_t decode_byte(uint64_t code, int b) {
  if (CODER == HUSKY_CODER_ASCII) return (uint8_t)((code >> (56 - 7 * b)) & 0x7F);
  uint32_t u = (uint32_t)(((code << 1) >> (48 - 16 * (b >> 1))) & 0xFFFF);
  return (uint8_t)(b & 1 ? u >> 8 : u);
}

// PACKED: perm holds index | min(len,15) << 28 (written by the encoder, carried
// through the radix as the payload).  Strings whose length is <= PL are then
// rebuilt from their sorted code (sequential reads only); perm is unpacked in
// place.  Only longer strings read offsets / units at random.
template <int CODER, bool PACKED>
__global__ void __launch_bounds__(kGatherThreads)
    k_gather(uint32_t *__restrict__ perm, uint64_t n, const void *__restrict__ units,
             const int64_t *__restrict__ offsets, void *__restrict__ sorted_units,
             int64_t *__restrict__ sorted_offsets, unsigned long long *lb, uint32_t *tile_counter,
             uint32_t epoch, const int64_t *base_ptr, int dbg, const uint64_t *__restrict__ codes) {
  constexpr int W = CoderTraits<CODER>::kUnitBytes;
  __shared__ __align__(16) uint8_t stage[kGatherStage + 32];
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_wt[kGatherThreads / 32 + 1];
  __shared__ unsigned long long s_base;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  // re-gather of a span: output positions start at *base_ptr (unchanged by us)
  const unsigned long long gbase = base_ptr ? (unsigned long long)*base_ptr : 0ull;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t p0 = (uint64_t)tile * kGatherTile + (uint64_t)tid * kGatherItems;
#ifdef HUSKY_TRACE
  if (tid == 0) printf("[husky trace] gather start tile %u n %llu gbase %llu\n", tile, (unsigned long long)n, gbase);
#endif

  constexpr uint32_t PL = CoderTraits<CODER>::kPL;
  uint32_t idx[kGatherItems];
#pragma unroll
  for (int j = 0; j < kGatherItems; ++j) idx[j] = p0 + j < n ? perm[p0 + j] : 0xFFFFFFFFu;
  int64_t src[kGatherItems];  // -1: rebuild from the code
  uint64_t len[kGatherItems];
  uint64_t code[kGatherItems];
  unsigned long long mine = 0;
#pragma unroll
  for (int j = 0; j < kGatherItems; ++j) {
    code[j] = 0;
    if (idx[j] == 0xFFFFFFFFu) {
      src[j] = 0;
      len[j] = 0;
    } else {
      uint32_t lc = 15;
      if (PACKED) {
        lc = idx[j] >> 28;
        idx[j] &= 0x0FFFFFFFu;
        perm[p0 + j] = idx[j];
      }
      if (PACKED && lc <= PL) {
        src[j] = -1;
        len[j] = lc;
        code[j] = __ldg(codes + p0 + j);
      } else {
        int64_t a = __ldg(offsets + idx[j]), b = __ldg(offsets + idx[j] + 1);
        src[j] = a;
        len[j] = (uint64_t)(b - a);
      }
    }
    mine += len[j];
  }
  unsigned long long tile_total;
  unsigned long long excl_t = block_exclusive_scan<unsigned long long, kGatherThreads>(mine, &tile_total, s_wt);
  if (tid == 0) st_relaxed_u64(lb + tile, make_flag(tile == 0 ? kFlagInc : kFlagAgg, epoch, tile_total));

  const uint8_t *ub = (const uint8_t *)units;
  uint8_t *ob = (uint8_t *)sorted_units;
  const uint64_t tile_bytes = tile_total * W;
  const bool staged = sorted_units != nullptr && tile_bytes <= (uint64_t)kGatherStage && !(dbg & 1);
  if (staged) {  // stage at tile-local byte offsets (needs no global base)
    uint64_t d = excl_t * W;
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
      uint64_t nb = len[j] * W;
      if (PACKED && src[j] < 0) {
        for (int b = 0; b < (int)nb; ++b) stage[d + b] = decode_byte<CODER>(code[j], b);
        d += nb;
        continue;
      }
      const uint8_t *sp = ub + src[j] * W;
      for (uint64_t c = 0; c < nb; c += 8) {
        int take = (int)(nb - c < 8 ? nb - c : 8);
        uint64_t v = load8_unaligned(sp + c, take);
        for (int b = 0; b < take; ++b) stage[d + c + b] = (uint8_t)(v >> (8 * b));
      }
      d += nb;
    }
  }

  if (warp == 0) {
    unsigned long long ex = tile == 0 ? 0ull : ((dbg & 2) ? lookback(lb, tile, 1, epoch) : warp_lookback(lb, tile, epoch));
    if (lane == 0) {
      if (tile != 0) st_relaxed_u64(lb + tile, make_flag(kFlagInc, epoch, ex + tile_total));
      s_base = ex;
      if ((uint64_t)(tile + 1) * kGatherTile >= n) sorted_offsets[n] = (int64_t)(gbase + ex + tile_total);
    }
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

  uint8_t *g0 = ob + tbase * W;  // first output byte of the tile
  if (staged) {
    // global chunk ch covers [a0 + 16 ch, +16); its bytes sit at stage[16 ch - align ..)
    const uint32_t align = (uint32_t)((uintptr_t)g0 & 15);
    uint8_t *a0 = g0 - align;  // 16-aligned
    const uint64_t end = align + tile_bytes;
    const uint64_t nchunks = (end + 15) / 16;
    const uint32_t *sw = reinterpret_cast<const uint32_t *>(stage);
    for (uint64_t ch = tid; ch < nchunks; ch += kGatherThreads) {
      uint64_t lo = ch * 16, hi = lo + 16;
      if (lo >= align && hi <= end) {
        uint32_t so = (uint32_t)(lo - align);  // stage byte offset of the chunk
        uint32_t wi = so >> 2, sh = (so & 3) * 8;
        uint32_t w0 = sw[wi], w1 = sw[wi + 1], w2 = sw[wi + 2], w3 = sw[wi + 3], w4 = sw[wi + 4];
        uint4 o;
        o.x = __funnelshift_r(w0, w1, sh);
        o.y = __funnelshift_r(w1, w2, sh);
        o.z = __funnelshift_r(w2, w3, sh);
        o.w = __funnelshift_r(w3, w4, sh);
        *reinterpret_cast<uint4 *>(a0 + lo) = o;
      } else {
        for (uint64_t b = (lo > align ? lo : align); b < (hi < end ? hi : end); ++b) a0[b] = stage[b - align];
      }
    }
  } else {
    // long strings: warp-cooperative byte copy, one string at a time per warp
    for (int t = 0; t < 32; ++t) {
      uint64_t d = tbase + __shfl_sync(0xFFFFFFFFu, excl_t, t);
#pragma unroll
      for (int j = 0; j < kGatherItems; ++j) {
        int64_t s = __shfl_sync(0xFFFFFFFFu, src[j], t);
        uint64_t l = __shfl_sync(0xFFFFFFFFu, len[j], t);
        uint64_t cd = __shfl_sync(0xFFFFFFFFu, code[j], t);
        uint64_t nb = l * W;
        if (PACKED && s < 0) {
          for (uint64_t b = lane; b < nb; b += 32) ob[d * W + b] = decode_byte<CODER>(cd, (int)b);
        } else {
          for (uint64_t b = lane; b < nb; b += 32) ob[d * W + b] = ub[s * W + b];
        }
        d += l;
      }
    }
  }
}

void launch_gather(int coder, uint32_t *perm, uint64_t n, const void *units, const int64_t *offsets,
                   void *sorted_units, int64_t *sorted_offsets, unsigned long long *lb,
                   uint32_t *tile_counter, uint32_t epoch, cudaStream_t s, const int64_t *base_ptr,
                   const uint64_t *packed_codes) {
  if (n == 0) return;
  Scope sc_(ST_GATHER, s, n);
  dim3 g((unsigned)gather_tiles(n)), b(kGatherThreads);
  // HUSKY_DEBUG_GATHER: bit 0 forces the unstaged copy, bit 1 the serial look-back
  static const int dbg = [] {
    const char *v = getenv("HUSKY_DEBUG_GATHER");
    return v ? atoi(v) : 0;
  }();
#define G_ARGS perm, n, units, offsets, sorted_units, sorted_offsets, lb, tile_counter, epoch, base_ptr, dbg, packed_codes
  if (coder == HUSKY_CODER_ASCII) {
    if (packed_codes) k_gather<HUSKY_CODER_ASCII, true><<<g, b, 0, s>>>(G_ARGS);
    else k_gather<HUSKY_CODER_ASCII, false><<<g, b, 0, s>>>(G_ARGS);
  } else {
    if (packed_codes) k_gather<HUSKY_CODER_UNICODE, true><<<g, b, 0, s>>>(G_ARGS);
    else k_gather<HUSKY_CODER_UNICODE, false><<<g, b, 0, s>>>(G_ARGS);
  }
#undef G_ARGS
}

// perm-only mode with a packed payload: strip the length bits
__global__ void k_unpack_perm(uint32_t *perm, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    perm[i] &= 0x0FFFFFFFu;
}

void launch_unpack_perm(uint32_t *perm, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  Scope sc_(ST_GATHER, s, n);
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_unpack_perm<<<(unsigned)blocks, 256, 0, s>>>(perm, n);
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
#ifdef HUSKY_TRACE
    if (threadIdx.x == 0) printf("[husky trace] regather entry %u/%u+%u: start %u len %u\n", e, ns, nm, start, len);
#endif
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
#ifdef HUSKY_TRACE
    if (threadIdx.x == 0) printf("[husky trace] regather entry %u done: running %llu\n", e, running);
#endif
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
