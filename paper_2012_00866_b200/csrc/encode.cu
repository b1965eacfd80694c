// encode.cu -- A1: husky coding of every string (Alg. 2-4).
//
// One thread per string (ENC_ITEMS strings in flight per thread, grid-stride
// over a persistent grid).  The prefix window (9 ASCII bytes or 4 UTF-16 units)
// is fetched with at most two aligned 8-byte loads; the 7-bit-per-char packing
// of asciiToLong is a 3-step mask/shift compaction instead of
// a 9-step fold, and unicodeToLong's 16-bit packing + ">>> 1"
// is a half-word swap.  Fused into the same pass (no extra HBM read):
//   * the 8 x 256 digit histograms the onesweep radix needs (A2),
//   * Alg. 3's `perfect` flag as an OR of "not perfect",
//   * the ASCII domain check (unit > 0x7F inside the code window; reading R5),
//   * the offsets monotonicity check.
#include "husky_internal.cuh"
#include "kernels.cuh"

namespace husky {

// asciiToLong on the (already length-masked) first 8 bytes `lo` (byte k at bits
// 8k..8k+7) and 9th byte `b8`:  code = sum_k (b_k & 0x7F) << 7*(8-k).
__device__ __forceinline__ uint64_t pack_ascii(uint64_t lo, uint64_t b8) {
  uint64_t x = ((uint64_t)__byte_perm((uint32_t)(lo >> 32), 0, 0x0123)) |
               ((uint64_t)__byte_perm((uint32_t)lo, 0, 0x0123) << 32);  // byte-swap: char 0 on top
  x &= 0x7F7F7F7F7F7F7F7Full;
  x = (x & 0x007F007F007F007Full) | ((x & 0x7F007F007F007F00ull) >> 1);
  x = (x & 0x00003FFF00003FFFull) | ((x & 0x3FFF00003FFF0000ull) >> 2);
  x = (x & 0x000000000FFFFFFFull) | ((x & 0x0FFFFFFF00000000ull) >> 4);
  return (x << 7) | (b8 & 0x7F);
}

// Code of one string from the two aligned words covering its window: w0 holds
// the byte at address `a` (sh = a & 7), w1 the next word (only read when the
// window crosses into it).
template <int CODER>
__device__ __forceinline__ uint64_t encode_words(uint64_t w0, uint64_t w1, int sh, int64_t len,
                                                 uint32_t &viol) {
  using T = CoderTraits<CODER>;
  if (len < 0) { viol |= kOffsetsBad; len = 0; }
  if (len > T::kPL) viol |= kNotPerfect;
  uint64_t lo = sh ? ((w0 >> (8 * sh)) | (w1 << (64 - 8 * sh))) : w0;
  if (CODER == HUSKY_CODER_ASCII) {
    int m = len < 9 ? (int)len : 9;
    uint64_t b8 = (m == 9) ? ((w1 >> (8 * sh)) & 0xFF) : 0ull;
    if (m < 8) lo &= (1ull << (8 * m)) - 1;  // m == 0 -> 0
    if ((lo & 0x8080808080808080ull) | (b8 & 0x80)) viol |= kDomainBad;
    return pack_ascii(lo, b8);
  } else {
    int m = len < 4 ? (int)len : 4;
    if (m < 4) lo &= (1ull << (16 * m)) - 1;
    // units u0..u3 little-endian in lo -> (u0<<48 | u1<<32 | u2<<16 | u3) >> 1
    uint64_t be = ((uint64_t)__byte_perm((uint32_t)lo, 0, 0x1032) << 32) |
                  (uint64_t)__byte_perm((uint32_t)(lo >> 32), 0, 0x1032);
    return be >> 1;
  }
}

template <int CODER, bool HIST>
__global__ void __launch_bounds__(kEncThreads) k_encode(const void *__restrict__ units,
                                                        const int64_t *__restrict__ offsets, uint64_t n,
                                                        uint64_t *__restrict__ codes, DevState *st,
                                                        uint32_t *__restrict__ packed) {
  __shared__ uint32_t sh_hist[HIST ? 8 * 256 : 1];
  __shared__ int64_t s_off[2][kEncTile + 1];
  __shared__ uint64_t s_stage[kEncStageWords + 2];
  if (HIST) {
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
  }
  uint32_t viol = 0;
  unsigned long long kor = 0, knand = 0;  // OR and NOT-AND of the codes (MSD level 0)
  const uint32_t lane = lane_id();
  constexpr int W = CoderTraits<CODER>::kUnitBytes;
  // Global word loads (fallback path) are clamped into [lo_word, hi_word], the
  // aligned words that cover units[offsets[0] .. offsets[n]): for valid offsets
  // the words a window needs are always inside, so they can be issued
  // unconditionally without ever leaving the caller's buffer.
  const uintptr_t ub = (uintptr_t)units;
  const int64_t ofirst = __ldg(offsets), olast = __ldg(offsets + n);
  const bool any_units = olast > ofirst;
  const uintptr_t lo_word = (ub + (uintptr_t)(ofirst * W)) & ~(uintptr_t)7;
  const uintptr_t hi_word = any_units ? ((ub + (uintptr_t)(olast * W) - 1) & ~(uintptr_t)7) : lo_word;
  const uint64_t stride = (uint64_t)gridDim.x * kEncTile;
  auto issue_offsets = [&](uint64_t b, int64_t *dst) {
    uint32_t c = (uint32_t)((n - b) < (uint64_t)kEncTile ? (n - b) : kEncTile);
    for (uint32_t i = threadIdx.x; i <= c; i += blockDim.x) cp_async8(&dst[i], offsets + b + i);
    cp_async_commit();
  };
  int buf = 0;
  if ((uint64_t)blockIdx.x * kEncTile < n) issue_offsets((uint64_t)blockIdx.x * kEncTile, s_off[0]);
  for (uint64_t base = (uint64_t)blockIdx.x * kEncTile; base < n; base += stride, buf ^= 1) {
    // ---- stage the tile: its offsets (prefetched one tile ahead), then its
    // contiguous unit span, with coalesced async copies (each byte read once)
    const uint32_t cnt = (uint32_t)((n - base) < (uint64_t)kEncTile ? (n - base) : kEncTile);
    const int64_t *so = s_off[buf];
    cp_async_wait_all();
    __syncthreads();
    const int64_t tstart = so[0], tend = so[cnt];
    const uintptr_t aw0 = (ub + (uintptr_t)(tstart * W)) & ~(uintptr_t)7;
    const int64_t nwords = tend > tstart ? (int64_t)(((ub + (uintptr_t)(tend * W)) - aw0 + 7) >> 3) : 0;
    const bool staged = nwords <= kEncStageWords;
    if (staged) {
      for (int64_t wd = threadIdx.x; wd < nwords; wd += blockDim.x) cp_async8(&s_stage[wd], (const uint64_t *)aw0 + wd);
      cp_async_commit();
    }
    const bool has_next = base + stride < n;
    if (has_next) issue_offsets(base + stride, s_off[buf ^ 1]);
    if (staged) {
      if (has_next) cp_async_wait_group<1>();
      else cp_async_wait_all();
    }
    __syncthreads();

    int64_t o0[kEncItems], o1[kEncItems];
#pragma unroll
    for (int k = 0; k < kEncItems; ++k) {
      uint32_t li = threadIdx.x + k * blockDim.x;
      if (li < cnt) { o0[k] = so[li]; o1[k] = so[li + 1]; }
      else { o0[k] = tstart; o1[k] = tstart; }
    }
    uint64_t w0[kEncItems], w1[kEncItems];
    int sh[kEncItems];
#pragma unroll
    for (int k = 0; k < kEncItems; ++k) {
      uintptr_t a = ub + (uintptr_t)(o0[k] * W);
      sh[k] = (int)(a & 7);
      if (staged && o0[k] >= tstart && o1[k] <= tend && o0[k] <= o1[k]) {
        uint64_t rel = (uint64_t)((a & ~(uintptr_t)7) - aw0) >> 3;
        w0[k] = s_stage[rel];
        w1[k] = s_stage[rel + 1];
      } else if (any_units) {  // long spans or invalid offsets: clamped global loads
        uintptr_t aw = a & ~(uintptr_t)7;
        aw = aw < lo_word ? lo_word : (aw > hi_word ? hi_word : aw);
        uintptr_t aw1 = aw + 8 > hi_word ? hi_word : aw + 8;
        w0[k] = __ldg((const uint64_t *)aw);
        w1[k] = __ldg((const uint64_t *)aw1);
      } else {
        w0[k] = 0;
        w1[k] = 0;
      }
    }
    uint64_t code[kEncItems];
#pragma unroll
    for (int k = 0; k < kEncItems; ++k) code[k] = encode_words<CODER>(w0[k], w1[k], sh[k], o1[k] - o0[k], viol);
#pragma unroll
    for (int k = 0; k < kEncItems; ++k) {
      uint64_t i = base + threadIdx.x + (uint64_t)k * blockDim.x;
      bool valid = threadIdx.x + k * blockDim.x < cnt;
      if (valid) {
        codes[i] = code[k];
        kor |= code[k];
        knand |= ~code[k];
        // initial radix payload: index | min(len, 15) << 28 (n <= 2^28 only)
        if (packed) {
          int64_t L = o1[k] - o0[k];
          packed[i] = (uint32_t)i | ((uint32_t)(L < 0 ? 0 : (L > 15 ? 15 : L)) << 28);
        }
      }
      if (HIST) {
        uint32_t vmask = __ballot_sync(0xFFFFFFFFu, valid);
        if (vmask == 0) continue;
        int leader = __ffs(vmask) - 1;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          uint32_t dig = (uint32_t)(code[k] >> (8 * d)) & 0xFF;
          uint32_t ld = __shfl_sync(0xFFFFFFFFu, dig, leader);
          if (__all_sync(0xFFFFFFFFu, !valid || dig == ld)) {
            if ((int)lane == leader) atomicAdd(&sh_hist[d * 256 + ld], __popc(vmask));
          } else if (valid) {
            atomicAdd(&sh_hist[d * 256 + dig], 1u);
          }
        }
      }
    }
    __syncthreads();  // s_off / s_stage are reused by the next tile
  }
  // reduce violation bits: one atomic per warp that saw any
  viol = __reduce_or_sync(0xFFFFFFFFu, viol);
  if (lane == 0 && viol) atomicOr(&st->violations, viol);
  {
    __shared__ unsigned long long s_ao[2][kEncThreads / 32];
    uint32_t a = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)kor), b = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)(kor >> 32));
    uint32_t c = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)knand), d = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)(knand >> 32));
    if (lane == 0) {
      s_ao[0][threadIdx.x >> 5] = ((unsigned long long)b << 32) | a;
      s_ao[1][threadIdx.x >> 5] = ((unsigned long long)d << 32) | c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long x = 0, y = 0;
      for (int w = 0; w < kEncThreads / 32; ++w) { x |= s_ao[0][w]; y |= s_ao[1][w]; }
      if (x) atomicOr(&st->key_or, x);
      if (y) atomicOr(&st->key_nand, y);
    }
  }
  if (HIST) {
    __syncthreads();
    uint32_t *g = &st->hist[0][0];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x)
      if (sh_hist[i]) atomicAdd(g + i, sh_hist[i]);
  }
}

void launch_encode(int coder, bool hist, const void *units, const int64_t *offsets, uint64_t n,
                   uint64_t *codes, DevState *st, int num_sms, cudaStream_t s, uint32_t *packed) {
  if (n == 0) return;
  Scope sc_(ST_ENCODE, s, n);
  uint64_t blocks = (n + kEncTile - 1) / kEncTile;
  uint64_t cap = (uint64_t)num_sms * kEncBlocksPerSM;
  if (blocks > cap) blocks = cap;
  dim3 g((unsigned)blocks), b(kEncThreads);
  if (coder == HUSKY_CODER_ASCII) {
    if (hist) k_encode<HUSKY_CODER_ASCII, true><<<g, b, 0, s>>>(units, offsets, n, codes, st, packed);
    else k_encode<HUSKY_CODER_ASCII, false><<<g, b, 0, s>>>(units, offsets, n, codes, st, packed);
  } else {
    if (hist) k_encode<HUSKY_CODER_UNICODE, true><<<g, b, 0, s>>>(units, offsets, n, codes, st, packed);
    else k_encode<HUSKY_CODER_UNICODE, false><<<g, b, 0, s>>>(units, offsets, n, codes, st, packed);
  }
}

}  // namespace husky
