// coders.cuh -- Alg. 4 (stringToLong) over the aligned
// 8-byte words that cover a string's code window: shared by the encoder
// (encode.cu) and the small-input sort (small.cu).  Not part of the ABI.
#pragma once
#include "husky_internal.cuh"

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

// Code of one string from the aligned words covering its window: w0 holds
// the byte at address `a` (sh = a & 7), w1 / w2 the next words (w2 is used only
// by the 10- and 12-unit English windows).
template <int CODER>
__device__ __forceinline__ uint64_t encode_words(uint64_t w0, uint64_t w1, uint64_t w2, int sh, int64_t len,
                                                 uint32_t &viol) {
  using T = CoderTraits<CODER>;
  if (len < 0) { viol |= kOffsetsBad; len = 0; }
  if (len > T::kPL) viol |= kNotPerfect;
  uint64_t lo = sh ? ((w0 >> (8 * sh)) | (w1 << (64 - 8 * sh))) : w0;
  if constexpr (CODER == HUSKY_CODER_ENGLISH5 || CODER == HUSKY_CODER_ENGLISH6) {
    // Alg. 4 with (K, bits, 2^bits - 1): fold the first m = min(len, K) bytes,
    // then shift by bits * (K - m) -- the same arithmetic as the closed form
    // sum_{i<m} (u_i & mask) << bits * (K - 1 - i)
    constexpr int K = T::kK, B = T::kBits;
    constexpr uint32_t mask = (1u << B) - 1;
    const uint64_t hi = sh ? ((w1 >> (8 * sh)) | (w2 << (64 - 8 * sh))) : w1;  // bytes 8..15
    const int m = len < K ? (int)len : K;
    uint64_t r = 0;
    uint32_t bad_lo = 0, bad_up = 0, bad_letter = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const uint32_t u = (uint32_t)(((i < 8) ? (lo >> (8 * i)) : (hi >> (8 * (i - 8)))) & 0xFF);
      const bool in = i < m;
      const bool lower = u >= 0x61 && u <= 0x7A, upper = u >= 0x41 && u <= 0x5A;
      bad_lo |= in && !lower;
      bad_up |= in && !upper;
      bad_letter |= in && !(lower || upper);
      r = (r << B) | (in ? (u & mask) : 0u);
    }
    if (CODER == HUSKY_CODER_ENGLISH5) viol |= (bad_lo ? kNotLower : 0u) | (bad_up ? kNotUpper : 0u);
    else if (bad_letter) viol |= kDomainBad;
    return r;
  } else if constexpr (CODER == HUSKY_CODER_ASCII) {
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

}  // namespace husky
