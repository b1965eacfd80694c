// gather.cu -- A4: sorted-string gather.
//
// The paper's co-swap moves object references with the keys;
// here the strings themselves are materialised in sorted order:
//   sorted_offsets = exclusive scan of len[perm[i]]  (single pass, look-back)
//   sorted_units   = concatenation of units[offsets[perm[i]] ..)
// A tile of 4096 sorted positions (512 threads x 8): perm (coalesced) ->
// lengths -> tile-local scan; the tile's aggregate is published, then the first
// window of the tile's output bytes is staged in shared memory at tile-local
// byte offsets (random reads, independent of the look-back), warp 0 resolves
// the tile's global base with a warp-wide look-back (32 predecessors per round
// trip), and the output is written with aligned 16-byte stores funnel-shifted
// out of smem.  Tiles larger than the stage are processed window by window.
// Boundary chunks use byte stores, so neighbouring tiles never race.
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
             uint32_t epoch, const int64_t *base_ptr, int dbg, const uint64_t *__restrict__ codes,
             const DevState *st) {
  constexpr int W = CoderTraits<CODER>::kUnitBytes;
  constexpr uint32_t PL = CoderTraits<CODER>::kPL;
  extern __shared__ __align__(16) uint8_t stage[];  // kGatherStage + 32 bytes
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_wt[kGatherThreads / 32 + 1];
  __shared__ unsigned long long s_base;
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (st) {
    if (st->violations & kOffsetsBad) return;  // invalid input: reported by the caller
    if (PACKED && codes == nullptr) codes = reinterpret_cast<const uint64_t *>(st->sorted_keys);
  }
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  // re-gather of a span: output positions start at *base_ptr (unchanged by us)
  const unsigned long long gbase = base_ptr ? (unsigned long long)*base_ptr : 0ull;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t p0 = (uint64_t)tile * kGatherTile + (uint64_t)tid * kGatherItems;

  // per item: len (units) and either the source offset or, for strings rebuilt
  // from their code, the code itself (bit j of `dec`)
  uint32_t raw[kGatherItems];
#pragma unroll
  for (int j = 0; j < kGatherItems; ++j) raw[j] = p0 + j < n ? perm[p0 + j] : 0xFFFFFFFFu;
  uint64_t sv[kGatherItems];
  uint32_t len[kGatherItems];
  uint32_t dec = 0;
  unsigned long long mine = 0;
#pragma unroll
  for (int j = 0; j < kGatherItems; ++j) {
    if (raw[j] == 0xFFFFFFFFu) {
      sv[j] = 0;
      len[j] = 0;
    } else {
      uint32_t idx = raw[j], lc = 15;
      if (PACKED) {
        lc = idx >> 28;
        idx &= 0x0FFFFFFFu;
        perm[p0 + j] = idx;
      }
      if (PACKED && lc <= PL) {
        dec |= 1u << j;
        len[j] = lc;
        sv[j] = __ldg(codes + p0 + j);
      } else {
        int64_t a = __ldg(offsets + idx), b = __ldg(offsets + idx + 1);
        sv[j] = (uint64_t)a;
        len[j] = (uint32_t)(b - a);
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
  const bool direct = (dbg & 1) != 0;

  // stage tile-local output bytes [w0, w1) of this thread's strings at stage[x - w0]
  auto stage_window = [&](uint64_t w0, uint64_t w1) {
    uint64_t d = excl_t * W;
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
      const uint64_t nb = (uint64_t)len[j] * W;
      const uint64_t lo = d > w0 ? d : w0, hi = d + nb < w1 ? d + nb : w1;
      if (lo < hi) {
        if (PACKED && ((dec >> j) & 1)) {
          for (uint64_t x = lo; x < hi; ++x) stage[x - w0] = decode_byte<CODER>(sv[j], (int)(x - d));
        } else {
          const uint8_t *sp = ub + sv[j] * W;
          for (uint64_t x = lo; x < hi; x += 8) {
            int take = (int)(hi - x < 8 ? hi - x : 8);
            uint64_t v = load8_unaligned(sp + (x - d), take);
            for (int b = 0; b < take; ++b) stage[x - w0 + b] = (uint8_t)(v >> (8 * b));
          }
        }
      }
      d += nb;
    }
  };
  // write tile-local bytes [w0, w1) (staged at stage[x - w0]) to g0 + x
  auto write_window = [&](uint8_t *g0, uint64_t w0, uint64_t w1) {
    const uint32_t align = (uint32_t)((uintptr_t)g0 & 15);
    uint8_t *a0 = g0 - align;  // 16-aligned; tile byte x lives at a0 + align + x
    const uint64_t lo_b = align + w0, hi_b = align + w1;
    const uint64_t c0 = lo_b / 16, c1 = (hi_b + 15) / 16;
    const uint32_t *sw = reinterpret_cast<const uint32_t *>(stage);
    for (uint64_t ch = c0 + tid; ch < c1; ch += kGatherThreads) {
      uint64_t lo = ch * 16, hi = lo + 16;
      if (lo >= lo_b && hi <= hi_b) {
        uint32_t so = (uint32_t)(lo - lo_b);  // stage offset of the chunk
        uint32_t wi = so >> 2, sh = (so & 3) * 8;
        uint32_t x0 = sw[wi], x1 = sw[wi + 1], x2 = sw[wi + 2], x3 = sw[wi + 3], x4 = sw[wi + 4];
        uint4 o;
        o.x = __funnelshift_r(x0, x1, sh);
        o.y = __funnelshift_r(x1, x2, sh);
        o.z = __funnelshift_r(x2, x3, sh);
        o.w = __funnelshift_r(x3, x4, sh);
        *reinterpret_cast<uint4 *>(a0 + lo) = o;
      } else {
        for (uint64_t b = (lo > lo_b ? lo : lo_b); b < (hi < hi_b ? hi : hi_b); ++b) a0[b] = stage[b - lo_b];
      }
    }
  };

  const uint64_t first_w1 = tile_bytes < (uint64_t)kGatherStage ? tile_bytes : (uint64_t)kGatherStage;
  if (sorted_units && !direct) stage_window(0, first_w1);  // overlaps the look-back

  if (warp == 0) {
    unsigned long long ex =
        tile == 0 ? 0ull : ((dbg & 2) ? lookback(lb, tile, 1, epoch) : warp_lookback(lb, tile, epoch));
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
  if (!direct) {
    write_window(g0, 0, first_w1);
    for (uint64_t w0 = first_w1; w0 < tile_bytes; w0 += kGatherStage) {  // large tiles: more windows
      const uint64_t w1 = w0 + kGatherStage < tile_bytes ? w0 + kGatherStage : tile_bytes;
      __syncthreads();
      stage_window(w0, w1);
      __syncthreads();
      write_window(g0, w0, w1);
    }
  } else {
    // debug path: warp-cooperative byte copy, one string at a time per warp
    for (int t = 0; t < 32; ++t) {
      uint64_t d = tbase + __shfl_sync(0xFFFFFFFFu, excl_t, t);
      uint32_t dt = __shfl_sync(0xFFFFFFFFu, dec, t);
#pragma unroll
      for (int j = 0; j < kGatherItems; ++j) {
        uint64_t s = __shfl_sync(0xFFFFFFFFu, sv[j], t);
        uint32_t l = __shfl_sync(0xFFFFFFFFu, len[j], t);
        uint64_t nb = (uint64_t)l * W;
        if (PACKED && ((dt >> j) & 1)) {
          for (uint64_t b = lane; b < nb; b += 32) ob[d * W + b] = decode_byte<CODER>(s, (int)b);
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
                   bool packed, const uint64_t *packed_codes, const DevState *st) {
  if (n == 0) return;
  constexpr int kSmem = kGatherStage + 32;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_gather<HUSKY_CODER_ASCII, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaFuncSetAttribute(k_gather<HUSKY_CODER_ASCII, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaFuncSetAttribute(k_gather<HUSKY_CODER_UNICODE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaFuncSetAttribute(k_gather<HUSKY_CODER_UNICODE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    configured = true;
  }
  Scope sc_(ST_GATHER, s, n);
  dim3 g((unsigned)gather_tiles(n)), b(kGatherThreads);
  // HUSKY_DEBUG_GATHER: bit 0 forces the unstaged copy, bit 1 the serial look-back
  static const int dbg = [] {
    const char *v = getenv("HUSKY_DEBUG_GATHER");
    return v ? atoi(v) : 0;
  }();
#define G_ARGS \
  perm, n, units, offsets, sorted_units, sorted_offsets, lb, tile_counter, epoch, base_ptr, dbg, packed_codes, st
  if (coder == HUSKY_CODER_ASCII) {
    if (packed) k_gather<HUSKY_CODER_ASCII, true><<<g, b, kSmem, s>>>(G_ARGS);
    else k_gather<HUSKY_CODER_ASCII, false><<<g, b, kSmem, s>>>(G_ARGS);
  } else {
    if (packed) k_gather<HUSKY_CODER_UNICODE, true><<<g, b, kSmem, s>>>(G_ARGS);
    else k_gather<HUSKY_CODER_UNICODE, false><<<g, b, kSmem, s>>>(G_ARGS);
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
                    int64_t *__restrict__ sorted_offsets, uint32_t first_small, uint32_t first_medium) {
  constexpr int W = CoderTraits<CODER>::kUnitBytes;
  __shared__ unsigned long long s_wt[256 / 32 + 1];
  if (st->violations & kOffsetsBad) return;
  // entries [first_small, n_small) of the small list, then [first_medium, n_medium) of the medium list
  const uint32_t ns = st->n_small - first_small, nm = st->n_medium - first_medium;
  const uint8_t *ub = (const uint8_t *)units;
  uint8_t *ob = (uint8_t *)sorted_units;
  for (uint32_t e = blockIdx.x; e < ns + nm; e += gridDim.x) {
    uint2 ent = e < ns ? list[first_small + e] : list[cap - 1 - (first_medium + e - ns)];
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
                          void *sorted_units, int64_t *sorted_offsets, int num_sms, cudaStream_t s,
                          uint32_t first_small, uint32_t first_medium) {
  Scope sc_(ST_FIX_SMALL, s, 0);
  dim3 g(num_sms * 4), b(256);
  if (coder == HUSKY_CODER_ASCII)
    k_regather_runs<HUSKY_CODER_ASCII><<<g, b, 0, s>>>(list_sm, cap_sm, st, perm, units, offsets, sorted_units,
                                                       sorted_offsets, first_small, first_medium);
  else
    k_regather_runs<HUSKY_CODER_UNICODE><<<g, b, 0, s>>>(list_sm, cap_sm, st, perm, units, offsets, sorted_units,
                                                         sorted_offsets, first_small, first_medium);
}

}  // namespace husky
