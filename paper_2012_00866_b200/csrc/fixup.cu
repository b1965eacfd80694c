// fixup.cu -- A5 segmented fix-up of dirty equal-code runs and A6 giant-run
// refinement keys.
//
// The paper's step 3 re-sorts the whole array with Timsort (PAPER.md:188, 297,
// 433), relying on there being "very few inversions" left.
// Because every remaining inversion is inside an equal-code run (R6),
// only dirty runs are re-sorted here, each independently:
//   small  (<= 32 strings): one warp; every lane owns a string and computes its
//          rank with the exact comparator against all others (rank sort);
//   medium (<= 4096): one CTA, bitonic sort of indices in shared memory;
//   giant  (> 4096): refinement rounds (host loop in husky.cu): the run is
//          re-keyed from its common prefix (k_seg_prep / k_seg_key2) and sorted
//          with the onesweep radix; sub-runs that are still ambiguous go round
//          again or drop into the small/medium lists.
// All comparisons use the exact comparator (units, length, original index).
#include "husky_internal.cuh"
#include "kernels.cuh"

namespace husky {

template <int CODER>
__global__ void __launch_bounds__(256)
    k_fix_small(const uint2 *__restrict__ list, const DevState *st, uint32_t *perm,
                const void *__restrict__ units, const int64_t *__restrict__ offsets, uint32_t first) {
  using T = CoderTraits<CODER>;
  pdl_wait();
  if (st->violations & kOffsetsBad) return;
  const uint32_t lane = lane_id();
  const uint32_t nsmall = st->n_small;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t e = first + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); e < nsmall; e += warps) {
    uint2 ent = list[e];
    const uint32_t start = ent.x, len = ent.y;
    uint32_t my = lane < len ? perm[start + lane] : 0xFFFFFFFFu;
    uint32_t rank = 0;
    const bool general = st->general != 0;
    for (uint32_t j = 0; j < len; ++j) {
      uint32_t other = __shfl_sync(0xFFFFFFFFu, my, j);
      if (lane < len && j != lane &&
          (general ? cmp_general<CODER>(units, offsets, other, my)
                   : cmp_equal_code<CODER>(units, offsets, other, my, T::kS)) < 0)
        ++rank;
    }
    __syncwarp();
    if (lane < len) perm[start + rank] = my;
    __syncwarp();
  }
}

template <int CODER>
__global__ void __launch_bounds__(1024)
    k_fix_medium(const uint2 *__restrict__ list, uint64_t cap, const DevState *st, uint32_t *perm,
                 const void *__restrict__ units, const int64_t *__restrict__ offsets, uint32_t first) {
  using T = CoderTraits<CODER>;
  __shared__ uint32_t s[kMediumMax];
  pdl_wait();
  if (st->violations & kOffsetsBad) return;
  const uint32_t nmed = st->n_medium;
  const bool general = st->general != 0;
  for (uint32_t e = first + blockIdx.x; e < nmed; e += gridDim.x) {
    uint2 ent = list[cap - 1 - e];
    const uint32_t start = ent.x, len = ent.y;
#ifdef HUSKY_TRACE
    if (threadIdx.x == 0) printf("[husky trace] fix_medium entry %u/%u: start %u len %u cap %llu\n", e, nmed, start, len,
                                 (unsigned long long)cap);
#endif
    uint32_t P = 1;
    while (P < len) P <<= 1;
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) s[i] = i < len ? perm[start + i] : 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
          uint32_t ixj = i ^ j;
          if (ixj > i) {
            uint32_t a = s[i], b = s[ixj];
            bool gt;  // a > b ?  (0xFFFFFFFF = +infinity padding)
            if (a == 0xFFFFFFFFu) gt = b != 0xFFFFFFFFu;
            else if (b == 0xFFFFFFFFu) gt = false;
            else gt = (general ? cmp_general<CODER>(units, offsets, a, b)
                               : cmp_equal_code<CODER>(units, offsets, a, b, T::kS)) > 0;
            bool asc = (i & k) == 0;
            if (gt == asc) { s[i] = b; s[ixj] = a; }
          }
        }
        __syncthreads();
      }
    }
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) perm[start + i] = s[i];
    __syncthreads();
  }
}

void launch_fix_small(int coder, const uint2 *list_sm, const DevState *st, uint32_t *perm,
                      const void *units, const int64_t *offsets, int num_sms, cudaStream_t s, uint32_t first) {
  Scope sc_(ST_FIX_SMALL, s, 0);
  dim3 g(num_sms * 4), b(256);
  if (coder == HUSKY_CODER_ASCII)
    launch_pdl(k_fix_small<HUSKY_CODER_ASCII>, g, b, 0, s, list_sm, st, perm, units, offsets, first);
  else
    launch_pdl(k_fix_small<HUSKY_CODER_UNICODE>, g, b, 0, s, list_sm, st, perm, units, offsets, first);
}

void launch_fix_medium(int coder, const uint2 *list_sm, uint64_t cap_sm, const DevState *st,
                       uint32_t *perm, const void *units, const int64_t *offsets, int num_sms,
                       cudaStream_t s, uint32_t first) {
  Scope sc_(ST_FIX_MEDIUM, s, 0);
  dim3 g(num_sms), b(1024);
  if (coder == HUSKY_CODER_ASCII)
    launch_pdl(k_fix_medium<HUSKY_CODER_ASCII>, g, b, 0, s, list_sm, cap_sm, st, perm, units, offsets, first);
  else
    launch_pdl(k_fix_medium<HUSKY_CODER_UNICODE>, g, b, 0, s, list_sm, cap_sm, st, perm, units, offsets, first);
}

// ------------------------------------------------------------------ A6
// Common prefix of a giant segment (all strings share units [0, from)):
// seg_L = min over strings of LCP(s_i, s_0), capped at from + 256 units;
// seg_has_short = some string has length <= PL (only possible in round 0).
constexpr uint32_t kLcpCap = 256;

template <int CODER>
__global__ void __launch_bounds__(256)
    k_seg_prep(const uint32_t *__restrict__ perm_seg, uint64_t len, const void *__restrict__ units,
               const int64_t *__restrict__ offsets, uint32_t from, DevState *st) {
  using T = CoderTraits<CODER>;
  constexpr int W = T::kUnitBytes;
  const uint32_t i0 = perm_seg[0];
  const int64_t o0 = offsets[i0], l0 = offsets[i0 + 1] - o0;
  uint32_t best = from + kLcpCap;
  uint32_t has_short = 0;
  const uint8_t *ub = (const uint8_t *)units;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t i = perm_seg[e];
    int64_t o = offsets[i], l = offsets[i + 1] - o;
    if (l <= T::kPL && !st->general) has_short = 1;  // short rule: equal codes only (R6)
    int64_t m = l < l0 ? l : l0;
    int64_t lim = (int64_t)from + kLcpCap;
    if (m > lim) m = lim;
    int64_t k = from;
    while (k < m) {
      int64_t rem = m - k;
      int take = (int)(rem * W < 8 ? rem * W : 8);
      uint64_t x = load8_unaligned(ub + (o + k) * W, take), y = load8_unaligned(ub + (o0 + k) * W, take);
      if (take < 8) {
        uint64_t msk = (1ull << (8 * take)) - 1;
        x &= msk;
        y &= msk;
      }
      uint64_t d = x ^ y;
      if (d) { k += (__ffsll((long long)d) - 1) / (8 * W); break; }
      k += take / W;
    }
    if (k > m) k = m;
    if ((uint32_t)k < best) best = (uint32_t)k;
  }
  best = __reduce_min_sync(0xFFFFFFFFu, best);
  has_short = __reduce_or_sync(0xFFFFFFFFu, has_short);
  if (lane_id() == 0) {
    atomicMin(&st->seg_L, best);
    if (has_short) atomicOr(&st->seg_has_short, 1u);
  }
}

void launch_seg_prep(int coder, const uint32_t *perm_seg, uint64_t len, const void *units,
                     const int64_t *offsets, uint32_t from, DevState *st, cudaStream_t s) {
  Scope sc_(ST_REFINE, s, len);
  uint64_t blocks = (len + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  if (coder == HUSKY_CODER_ASCII)
    k_seg_prep<HUSKY_CODER_ASCII><<<(unsigned)blocks, 256, 0, s>>>(perm_seg, len, units, offsets, from, st);
  else
    k_seg_prep<HUSKY_CODER_UNICODE><<<(unsigned)blocks, 256, 0, s>>>(perm_seg, len, units, offsets, from, st);
}

// Refinement key at offset L (R6/A6): a string with len <= PL (only in
// round 0, L = S) gets key = len (< 16); otherwise
//   ASCII:   key = (units[L..L+7) big-endian, zero padded) << 8  | (16 + min(len-L, 8))
//   UNICODE: key = (units[L..L+3) big-endian, zero padded) << 16 | (16 + min(len-L, 4))
// Equal keys with tag < cap are identical strings; tag == cap continues at L + window.
template <int CODER>
__global__ void __launch_bounds__(256)
    k_seg_key2(const uint32_t *__restrict__ perm_seg, uint64_t len, const void *__restrict__ units,
               const int64_t *__restrict__ offsets, uint32_t from, uint64_t *__restrict__ key2,
               DevState *st) {
  using T = CoderTraits<CODER>;
  __shared__ uint32_t sh_hist[8 * 256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) sh_hist[i] = 0;
  __syncthreads();
  const uint32_t L = st->seg_has_short ? from : st->seg_L;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < len; base += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t e = base + threadIdx.x;
    bool valid = e < len;
    uint64_t key = 0;
    if (valid) {
      uint32_t i = perm_seg[e];
      int64_t o = offsets[i], l = offsets[i + 1] - o;
      if (l <= T::kPL && st->seg_has_short) {
        key = (uint64_t)l;
      } else {
        int64_t rem = l - (int64_t)L;
        if (rem < 0) rem = 0;
        int take = (int)(rem < T::kWin ? rem : T::kWin);
        uint64_t win = 0;
        if (take > 0) {
          uint64_t x = load8_unaligned((const uint8_t *)units + (o + L) * T::kUnitBytes, take * T::kUnitBytes);
          if (take * T::kUnitBytes < 8) x &= (1ull << (8 * take * T::kUnitBytes)) - 1;
          if (CODER == HUSKY_CODER_ASCII) {
            // bytes b0..b6 little-endian -> big-endian 56-bit window
            uint64_t be = ((uint64_t)__byte_perm((uint32_t)x, 0, 0x0123) << 32) |
                          (uint64_t)__byte_perm((uint32_t)(x >> 32), 0, 0x0123);
            win = be >> 8;  // keep 7 bytes
            key = (win << 8) | (uint64_t)(16 + (rem < 8 ? rem : 8));
          } else {
            uint64_t be = ((uint64_t)__byte_perm((uint32_t)x, 0, 0x1032) << 32) |
                          (uint64_t)__byte_perm((uint32_t)(x >> 32), 0, 0x1032);
            win = be >> 16;  // keep 3 units
            key = (win << 16) | (uint64_t)(16 + (rem < 4 ? rem : 4));
          }
        } else {
          key = (uint64_t)16;  // rem == 0: empty window, tag 16
        }
      }
      key2[e] = key;
    }
    uint32_t vmask = __ballot_sync(0xFFFFFFFFu, valid);
    if (vmask == 0) continue;
    int leader = __ffs(vmask) - 1;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      uint32_t dig = (uint32_t)(key >> (8 * d)) & 0xFF;
      uint32_t ld = __shfl_sync(0xFFFFFFFFu, dig, leader);
      if (__all_sync(0xFFFFFFFFu, !valid || dig == ld)) {
        if ((int)lane_id() == leader) atomicAdd(&sh_hist[d * 256 + ld], __popc(vmask));
      } else if (valid) {
        atomicAdd(&sh_hist[d * 256 + dig], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x)
    if (sh_hist[i]) atomicAdd(&st->hist[i >> 8][i & 255], sh_hist[i]);
}

void launch_seg_key2(int coder, const uint32_t *perm_seg, uint64_t len, const void *units,
                     const int64_t *offsets, uint32_t from, uint64_t *key2, DevState *st,
                     int num_sms, cudaStream_t s) {
  Scope sc_(ST_REFINE, s, len);
  uint64_t blocks = (len + 255) / 256;
  uint64_t cap = (uint64_t)num_sms * 4;
  if (blocks > cap) blocks = cap;
  if (coder == HUSKY_CODER_ASCII)
    k_seg_key2<HUSKY_CODER_ASCII><<<(unsigned)blocks, 256, 0, s>>>(perm_seg, len, units, offsets, from, key2, st);
  else
    k_seg_key2<HUSKY_CODER_UNICODE><<<(unsigned)blocks, 256, 0, s>>>(perm_seg, len, units, offsets, from, key2, st);
}

}  // namespace husky
