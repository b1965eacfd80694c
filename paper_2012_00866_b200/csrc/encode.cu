// encode.cu -- A1: husky coding of every string (Alg. 2-4).
//
// One thread per string (ENC_ITEMS strings in flight per thread, grid-stride
// over a persistent grid).  The prefix window (9 ASCII bytes or 4 UTF-16 units)
// is fetched with at most two aligned 8-byte loads; the 7-bit-per-char packing
// of asciiToLong is a 3-step mask/shift compaction instead of
// a 9-step fold, and unicodeToLong's 16-bit packing + ">>> 1"
// is a half-word swap.  Fused into the same pass (no extra HBM read):
//   * Alg. 3's `perfect` flag as an OR of "not perfect",
//   * the ASCII domain check (unit > 0x7F inside the code window; reading R5),
//   * the offsets monotonicity check,
//   * the string slab (ASCII / UNICODE, when the caller asks for sorted
//     strings): a 16-byte record per string -- its length and the units that
//     follow the code window (ASCII units 9..23, UNICODE units 3..9) -- written
//     in input order, so the gather (A4) fetches a string of up to 24 / 10
//     units with ONE random 16-byte read (units [0, S) come back out of the
//     sorted code) instead of a random offsets read followed by a random units
//     read.  Random reads past ~2 GB are capped at ~36 G accesses/s whatever
//     their size (profiles/r02_random_access_probe.txt), so the number of
//     random accesses per string, not bytes, sets the gather's time.
// The LSD radix's 8 x 256 digit histograms come from a separate read of the
// codes (k_hist_slots), which measured cheaper than fusing them here.
#include <algorithm>

#include "coders.cuh"
#include "husky_internal.cuh"
#include "kernels.cuh"

namespace husky {

// Slab record of one string (ASCII / UNICODE): byte 0 = length if it is at
// most kSlabMax units, else 0xFF (the gather then reads offsets and units);
// bytes 1..15 = string bytes [S*W, S*W + 15), zero past the end.  `win` holds
// the string's bytes starting at window byte `sh` (words w0..w3 from the
// aligned word at or below the string start).
template <int CODER>
__device__ __forceinline__ uint4 make_slab(uint64_t w0, uint64_t w1, uint64_t w2, uint64_t w3, int sh, int64_t len) {
  using T = CoderTraits<CODER>;
  constexpr int W = T::kUnitBytes, SB = T::kS * W;  // slab's first string byte
  const uint32_t lcode = (len >= 0 && len <= T::kSlabMax) ? (uint32_t)len : 0xFFu;
  const int base = sh + SB;            // window byte of string byte SB
  const int q = base >> 3, r = (base & 7) * 8;
  const uint64_t a = q == 0 ? w0 : (q == 1 ? w1 : w2);
  const uint64_t b = q == 0 ? w1 : (q == 1 ? w2 : w3);
  const uint64_t c = q == 0 ? w2 : w3;
  uint64_t lo = r ? ((a >> r) | (b << (64 - r))) : a;  // string bytes SB .. SB+7
  uint64_t hi = r ? ((b >> r) | (c << (64 - r))) : b;  // SB+8 .. SB+15
  // zero the bytes past the end of the string
  const int64_t keep = len > T::kS ? (len - T::kS) * W : 0;  // string bytes present from SB
  if (keep < 8) { lo &= keep > 0 ? ((1ull << (8 * keep)) - 1) : 0ull; hi = 0; }
  else if (keep < 15) hi &= (1ull << (8 * (keep - 8))) - 1;
  // record bytes: [0] = lcode, [1..8] = lo, [9..15] = hi bytes 0..6
  const uint64_t r0 = (uint64_t)lcode | (lo << 8), r1 = (lo >> 56) | (hi << 8);
  return make_uint4((uint32_t)r0, (uint32_t)(r0 >> 32), (uint32_t)r1, (uint32_t)(r1 >> 32));
}

// One thread per string, IT strings in flight per thread (grid-stride over a
// persistent grid).  Lane i of a warp codes string i of 32 consecutive strings,
// whose units are contiguous, so the window loads of a warp fall in a few
// consecutive 128-B lines (L1 reuse); no shared-memory staging.  Measured on C2
// (1e7 words): 72.6 us vs 82.9 us for a cp.async-staged variant.
// Global word loads are clamped into [lo_word, hi_word], the aligned words that
// cover units[offsets[0] .. offsets[n]): for valid offsets the words a window
// needs are always inside, so they are issued unconditionally without ever
// leaving the caller's buffer.
// slab (nullable): the slab records; slab_all: write every string's record
// (the gather needs every length), else only those longer than PL (the packed
// payload carries the others' lengths and the code their units).
constexpr int kEncIT = 4;
template <int CODER>
// 4 CTAs per SM (64 registers): measured per C2 / C3 encode 76 / 62 us, against
// 81 / 71 us unbounded (79 registers, 3 CTAs), 87 / 83 us at 5 and 92 / 89 us at
// 6 CTAs per SM (spills) -- the kernel is latency-bound on its two dependent loads
__global__ void __launch_bounds__(kEncThreads, 4) k_encode(const void *__restrict__ units,
                                                        const int64_t *__restrict__ offsets, uint64_t n,
                                                        uint64_t *__restrict__ codes, uint32_t *viol_out,
                                                        uint32_t *__restrict__ packed, uint4 *__restrict__ slab,
                                                        int slab_all, uint32_t *alpha) {
  constexpr int W = CoderTraits<CODER>::kUnitBytes;
  constexpr bool kSlabCoder = CODER == HUSKY_CODER_ASCII || CODER == HUSKY_CODER_UNICODE;
  uint32_t viol = 0;
  // ASCII: which 7-bit field values occur in the code windows, as one byte
  // flag per value in shared memory (plain byte stores of 1: racing writers
  // agree), OR-ed into DevState::alpha at the end -- cheaper in the loop than
  // a 128-bit register mask (C5 encode 16.3 ms with the mask)
  __shared__ uint8_t s_pres[128];
  const bool want_alpha = CODER == HUSKY_CODER_ASCII && alpha != nullptr;
  if (want_alpha) {
    if (threadIdx.x < 128) s_pres[threadIdx.x] = 0;
    __syncthreads();
  }
  const uint32_t lane = lane_id();
  const uintptr_t ub = (uintptr_t)units;
  const int64_t ofirst = __ldg(offsets), olast = __ldg(offsets + n);
  const bool any_units = olast > ofirst;
  const uintptr_t lo_word = (ub + (uintptr_t)(ofirst * W)) & ~(uintptr_t)7;
  const uintptr_t hi_word = any_units ? ((ub + (uintptr_t)(olast * W) - 1) & ~(uintptr_t)7) : lo_word;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * kEncIT;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * kEncIT; base < n; base += stride) {
    int64_t o0[kEncIT], o1[kEncIT];
#pragma unroll
    for (int k = 0; k < kEncIT; ++k) {
      const uint64_t i = base + threadIdx.x + (uint64_t)k * blockDim.x;
      if (i < n) {
        o0[k] = __ldg(offsets + i);
        o1[k] = __ldg(offsets + i + 1);
      } else {
        o0[k] = ofirst;
        o1[k] = ofirst;
      }
    }
    constexpr bool kThird = CODER == HUSKY_CODER_ENGLISH5 || CODER == HUSKY_CODER_ENGLISH6;
    uint64_t w0[kEncIT], w1[kEncIT], w2[kEncIT];
    uintptr_t awk[kEncIT];
    int sh[kEncIT];
#pragma unroll
    for (int k = 0; k < kEncIT; ++k) {
      const uintptr_t a = ub + (uintptr_t)(o0[k] * W);
      sh[k] = (int)(a & 7);
      w2[k] = 0;
      awk[k] = lo_word;
      if (any_units) {
        uintptr_t aw = a & ~(uintptr_t)7;
        aw = aw < lo_word ? lo_word : (aw > hi_word ? hi_word : aw);
        awk[k] = aw;
        const uintptr_t aw1 = aw + 8 > hi_word ? hi_word : aw + 8;
        w0[k] = __ldg((const uint64_t *)aw);
        w1[k] = __ldg((const uint64_t *)aw1);
        if (kThird) {
          const uintptr_t aw2 = aw1 + 8 > hi_word ? hi_word : aw1 + 8;
          w2[k] = __ldg((const uint64_t *)aw2);
        }
      } else {
        w0[k] = 0;
        w1[k] = 0;
      }
    }
#pragma unroll
    for (int k = 0; k < kEncIT; ++k) {
      const uint64_t i = base + threadIdx.x + (uint64_t)k * blockDim.x;
      const int64_t L = o1[k] - o0[k];
      const uint64_t c = encode_words<CODER>(w0[k], w1[k], w2[k], sh[k], L, viol);
      if (want_alpha && i < n) {
        // the nine 7-bit fields of the code (padding fields are 0: always counted)
#pragma unroll
        for (int f = 0; f < 9; ++f) s_pres[(uint32_t)(c >> (7 * (8 - f))) & 0x7Fu] = 1;
      }
      if (i < n) {
        codes[i] = c;
        // initial radix payload: index | min(len, 15) << 28 (n <= 2^28 only)
        if (packed) packed[i] = (uint32_t)i | ((uint32_t)(L < 0 ? 0 : (L > 15 ? 15 : L)) << 28);
        if constexpr (kSlabCoder) {
          if (slab && (slab_all || L > CoderTraits<CODER>::kPL)) {
            // the words after the code window (mostly the same lines: L1
            // hits), only for strings that reach past it
            uint64_t x2 = 0, x3 = 0;
            if (L > CoderTraits<CODER>::kS) {
              const uintptr_t aw2 = awk[k] + 16 > hi_word ? hi_word : awk[k] + 16;
              const uintptr_t aw3 = awk[k] + 24 > hi_word ? hi_word : awk[k] + 24;
              x2 = __ldg((const uint64_t *)aw2);
              x3 = __ldg((const uint64_t *)aw3);
            }
            slab[i] = make_slab<CODER>(w0[k], w1[k], x2, x3, sh[k], L);
          }
        }
      }
    }
  }
  // reduce violation bits: one atomic per warp that saw any
  viol = __reduce_or_sync(0xFFFFFFFFu, viol);
  if (lane == 0 && viol) atomicOr(viol_out, viol);
  if (want_alpha) {
    __syncthreads();
    if (threadIdx.x < 128) {
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, s_pres[threadIdx.x] != 0);
      if (lane == 0 && m) atomicOr(alpha + (threadIdx.x >> 5), m);
    }
  }
}

void launch_encode(int coder, const void *units, const int64_t *offsets, uint64_t n, uint64_t *codes,
                   uint32_t *viol, int num_sms, cudaStream_t s, uint32_t *packed, uint4 *slab, bool slab_all,
                   uint32_t *alpha) {
  if (n == 0) return;
  Scope sc_(ST_ENCODE, s, n);
  uint64_t blocks = (n + kEncThreads * kEncIT - 1) / (kEncThreads * kEncIT);
  const uint64_t cap = (uint64_t)num_sms * kEncBlocksPerSM;
  if (blocks > cap) blocks = cap;
  const int sa = slab_all ? 1 : 0;
  switch (coder) {
    case HUSKY_CODER_ASCII:
      k_encode<HUSKY_CODER_ASCII><<<(unsigned)blocks, kEncThreads, 0, s>>>(units, offsets, n, codes, viol, packed,
                                                                           slab, sa, alpha);
      break;
    case HUSKY_CODER_UNICODE:
      k_encode<HUSKY_CODER_UNICODE><<<(unsigned)blocks, kEncThreads, 0, s>>>(units, offsets, n, codes, viol, packed,
                                                                             slab, sa, nullptr);
      break;
    case HUSKY_CODER_ENGLISH5:
      k_encode<HUSKY_CODER_ENGLISH5><<<(unsigned)blocks, kEncThreads, 0, s>>>(units, offsets, n, codes, viol, packed,
                                                                              nullptr, 0, nullptr);
      break;
    default:
      k_encode<HUSKY_CODER_ENGLISH6><<<(unsigned)blocks, kEncThreads, 0, s>>>(units, offsets, n, codes, viol, packed,
                                                                              nullptr, 0, nullptr);
      break;
  }
}

}  // namespace husky
