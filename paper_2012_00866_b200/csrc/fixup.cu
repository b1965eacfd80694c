// fixup.cu -- A5 segmented fix-up of dirty equal-code runs and A6 giant-run
// refinement keys.
//
// The paper's step 3 re-sorts the whole array with Timsort (PAPER.md:188, 297,
// 433), relying on there being "very few inversions" left.
// Because every remaining inversion is inside an equal-code run (R6),
// only dirty runs are re-sorted here, each independently:
//   staged (the main pass, sorted strings present, 32 < run <= 4096 strings
//          and <= kFixStageBytes of units): one CTA per run.  The run's strings are
//          contiguous after the gather, so they are staged into shared memory
//          with ONE bulk async copy (cp.async.bulk, the TMA engine) completing
//          on an mbarrier; each string gets a 48-bit big-endian key of its
//          units after the S that equal codes already fix (+ its 16-bit slot),
//          and the CTA merge-sorts those items (cub::BlockMergeSort, 512
//          threads x 8) with a comparator that falls back to a full compare of
//          the staged units only on equal keys (a bitonic network measured
//          2.8 ms on 2^23 D1 strings: too many barrier-separated stages).  The sorted run
//          is written back in place -- perm, sorted offsets and sorted units --
//          so no re-gather follows.
//   small  (<= 32 strings): one warp; every lane owns a string and computes
//          its rank with the exact comparator (rank sort);
//   gather-staged (perm-only mode, sub-runs after a refinement: the run's
//          strings are not contiguous): as staged, but the strings are gathered
//          into the stage from the input (perm -> offsets -> units) and only
//          perm is written back (D1 perm-only: 19.1 -> 3.6 ms);
//   medium (<= 4096, others): one CTA, bitonic sort of indices in shared memory
//          with global-memory comparisons (runs whose units exceed the stage);
//   giant  (> 4096): refinement rounds (host loop in husky.cu): the run is
//          re-keyed from its common prefix (k_seg_prep / k_seg_key2) and sorted
//          with the onesweep radix; sub-runs that are still ambiguous go round
//          again or drop into the small/medium lists.
// All comparisons use the exact comparator (units, length, original index).
#include <cub/block/block_merge_sort.cuh>

#include "husky_internal.cuh"
#include "kernels.cuh"

namespace husky {

// A run the staged kernel handled (main pass only: so != NULL): the other
// fix-up kernels and the re-gather skip it.  Not when every code was equal:
// the gather then left the sorted offsets inside the one run unwritten (the
// run is refined and gathered again), so nothing is staged.
template <int W>
__device__ __forceinline__ bool staged_run(const DevState *st, const int64_t *so, uint32_t start, uint32_t len) {
  return so != nullptr && st->trivial_mask != 0xFFu &&
         (uint64_t)(so[start + len] - so[start]) * W <= (uint64_t)kFixStageBytes;
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(a), "r"(phase)
                 : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completing on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}

constexpr int kFixThreads = 1024, kFixItems = kMediumMax / kFixThreads;  // 4 strings per thread
// dynamic shared memory of k_fix_staged: the stage (+16 B of alignment slack +
// read slack), per string: offset in the stage (n + 1 entries: lengths are
// differences) and global index; then the output image (the run's bytes in
// the new order)
constexpr int kFixArrBytes = ((kMediumMax + 1) * 4 + kMediumMax * 4 + 15) / 16 * 16;
constexpr int kFixSmem = kFixStageBytes + 32 + kFixArrBytes + kFixStageBytes + 32;

// Order of two sort items of a staged run: item = (top 48 bits of the 8-byte
// big-endian key of the string's units from byte kstart) << 16 | slot.
// Equal 48-bit prefixes fall back to the full comparison of the staged units
// from byte kstart + 6, then the lengths, then the original indices; slot
// 0xFFFF is padding (after everything).
struct FixLess {
  const uint8_t *stage;
  const uint32_t *soff, *sgid;  // string i: stage bytes [soff[i], soff[i + 1])
  uint32_t kstart, w;
  __device__ __forceinline__ bool operator()(const uint64_t &a, const uint64_t &b) const {
    const uint32_t sa = (uint32_t)(a & 0xFFFFu), sb = (uint32_t)(b & 0xFFFFu);
    if (sa == 0xFFFFu || sb == 0xFFFFu) return sb == 0xFFFFu && sa != 0xFFFFu;
    if ((a >> 16) != (b >> 16)) return (a >> 16) < (b >> 16);
    if (sa == sb) return false;
    const uint32_t la = soff[sa + 1] - soff[sa], lb = soff[sb + 1] - soff[sb], m = la < lb ? la : lb;
    for (uint32_t k = kstart + 6; k < m; k += 8) {
      uint64_t x = stage_load8(stage, soff[sa] + k), y = stage_load8(stage, soff[sb] + k);
      const uint32_t take = m - k < 8 ? m - k : 8;
      if (take < 8) {
        const uint64_t msk = (1ull << (8 * take)) - 1;
        x &= msk;
        y &= msk;
      }
      const uint64_t d = x ^ y;
      if (d) {
        const int sh = ((__ffsll((long long)d) - 1) / (8 * w)) * (8 * w);
        const uint64_t um = w == 1 ? 0xFFull : 0xFFFFull;
        return ((x >> sh) & um) < ((y >> sh) & um);
      }
    }
    if (la != lb) return la < lb;
    return sgid[sa] < sgid[sb];
  }
};

#ifdef HUSKY_FIX_TIMING
// lab builds: per-CTA cycles spent in each phase of k_fix_staged (stage, keys,
// sort, write-back), summed over its runs
__device__ unsigned long long g_fix_phase[1024][4];
#define FT(i) do { if (threadIdx.x == 0) { const long long t_ = clock64(); g_fix_phase[blockIdx.x][i] += t_ - ft_last; ft_last = t_; } } while (0)
#else
#define FT(i) do { } while (0)
#endif

// GSTAGE (perm-only mode and the sub-runs after a refinement, where the run's
// strings are not contiguous): the run's strings are gathered into the stage
// from the input (perm -> offsets -> units) instead, only perm is written back,
// and the entry is marked (kRunDone) so k_fix_medium skips the run.
template <int CODER, bool GSTAGE>
__global__ void __launch_bounds__(kFixThreads, 1)
    k_fix_staged(uint2 *__restrict__ list, uint64_t cap, const DevState *st, uint32_t *perm,
                 uint8_t *__restrict__ su, int64_t *__restrict__ so, const void *__restrict__ units,
                 const int64_t *__restrict__ offsets, uint32_t first) {
  using T = CoderTraits<CODER>;
  constexpr int W = T::kUnitBytes;
  using Sort = cub::BlockMergeSort<uint64_t, kFixThreads, kFixItems>;
  extern __shared__ __align__(16) uint8_t sm[];
  uint8_t *stage = sm;
  uint32_t *soff = reinterpret_cast<uint32_t *>(sm + kFixStageBytes + 32);
  uint32_t *sgid = soff + kMediumMax + 1;
  __shared__ typename Sort::TempStorage sort_tmp;
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_wt[kFixThreads / 32 + 1];
  pdl_wait();
  if (st->violations & kOffsetsBad) return;
  if (!GSTAGE && st->trivial_mask == 0xFFu) return;  // all codes equal: see staged_run
  const bool general = st->general != 0;
  // compare from unit S (equal codes fix units [0, S)), or from 0 off-domain
  const RunRule rule = run_rule<CODER>(st);
  const uint32_t kstart0 = general ? 0u : rule.S * W;
  // medium runs only: runs of <= 32 strings go to k_fix_small (a warp each;
  // a CTA-wide staged sort per 2-string run measured 0.8 ms for the ~10K
  // extra pairs of a partial key sort at 2^30)
  const uint32_t nm = st->n_medium;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the init, seen by the async proxy
  }
  __syncthreads();
  uint32_t phase = 0;
  const bool bulk_ok = ((uintptr_t)su & 15) == 0;
  __shared__ uint32_t s_lcp;
#ifdef HUSKY_FIX_TIMING
  long long ft_last = clock64();
#endif
  for (uint32_t e = first + blockIdx.x; e < nm; e += gridDim.x) {
    const uint2 ent = list[cap - 1 - e];
    const uint32_t start = ent.x, len = ent.y;
    if (GSTAGE) {
      // ---- gather-stage: lengths and source offsets of my strings (blocked:
      // thread t holds strings 4t .. 4t + 3), their stage offsets by a scan
      uint32_t Lg[kFixItems], tsum = 0;
      int64_t og[kFixItems];
#pragma unroll
      for (int j = 0; j < kFixItems; ++j) {
        const uint32_t i = threadIdx.x * kFixItems + j;
        Lg[j] = 0;
        og[j] = 0;
        if (i < len) {
          const uint32_t id = perm[start + i];
          sgid[i] = id;
          og[j] = offsets[id];
          Lg[j] = (uint32_t)(offsets[id + 1] - og[j]) * W;
        }
        tsum += Lg[j];
      }
      uint32_t tot;
      uint32_t d = block_exclusive_scan<uint32_t, kFixThreads>(tsum, &tot, s_wt);
      if (tot > (uint32_t)kFixStageBytes) continue;  // (uniform) left to k_fix_medium
#pragma unroll
      for (int j = 0; j < kFixItems; ++j) {
        const uint32_t i = threadIdx.x * kFixItems + j;
        if (i < len) {
          soff[i] = d;
          const uint8_t *src = (const uint8_t *)units + og[j] * W;
          for (uint32_t b = 0; b < Lg[j]; b += 8) {
            const int take = (int)(Lg[j] - b < 8 ? Lg[j] - b : 8);
            const uint64_t v = load8_unaligned(src + b, take);
            for (int q = 0; q < take; ++q) stage[d + b + q] = (uint8_t)(v >> (8 * q));
          }
        }
        d += Lg[j];
      }
      if (threadIdx.x == 0) soff[len] = tot;
      __syncthreads();
    }
    const int64_t B0u = GSTAGE ? 0 : so[start], B1u = GSTAGE ? 0 : so[start + len];
    const uint64_t B0 = (uint64_t)B0u * W, B1 = (uint64_t)B1u * W;  // the run's bytes in su
    if (B1 - B0 > (uint64_t)kFixStageBytes) continue;  // left to k_fix_small / k_fix_medium
#ifdef HUSKY_CHECKED
    if (threadIdx.x == 0) {
      HCHK(kChkFixStagedOffsets, (uint64_t)start + len, st->chk_n + 1);
      HCHK(kChkFixStagedUnits, B1, st->chk_units + 1);
    }
#endif
    // ---- stage: bytes [a0, B1) with a0 = B0 rounded down to 16; the aligned
    // body by one bulk copy (TMA engine, completing on the mbarrier), the
    // ragged tail by plain loads
    const uint64_t a0 = bulk_ok ? (B0 & ~15ull) : B0, a1 = bulk_ok ? (B1 & ~15ull) : B0;
    if (!GSTAGE) {
      if (threadIdx.x == 0 && a1 > a0) {
        // the previous run's generic-proxy accesses to the stage come first
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar, (uint32_t)(a1 - a0));
        bulk_g2s(stage, su + a0, (uint32_t)(a1 - a0), &bar);
      }
      for (uint64_t x = (a1 > a0 ? a1 : B0) + threadIdx.x; x < B1; x += kFixThreads) stage[x - a0] = su[x];
      // per string: offset in the stage (n + 1 entries) / global index
      for (uint32_t i = threadIdx.x; i <= len; i += kFixThreads) {
        soff[i] = (uint32_t)((uint64_t)so[start + i] * W - a0);
        if (i < len) sgid[i] = perm[start + i];
      }
      if (a1 > a0) mbar_wait(&bar, phase);
      phase ^= (a1 > a0) ? 1u : 0u;
      __syncthreads();
    }
    // ---- the run's common prefix: every string agrees with string 0 on its
    // first lcp bytes, so keys and compares start there (strings of a dirty
    // run often share more than the S units their codes fix, e.g. URLs)
    if (threadIdx.x == 0) s_lcp = 0xFFFFFFFFu;
    __syncthreads();
    {
      uint32_t my = 0xFFFFFFFFu;
      const uint32_t o0 = soff[0], l0 = soff[1] - soff[0];
#pragma unroll
      for (int j = 0; j < kFixItems; ++j) {
        const uint32_t i = threadIdx.x * kFixItems + j;
        if (i >= len || i == 0) continue;
        const uint32_t oi = soff[i], li = soff[i + 1] - oi, m = li < l0 ? li : l0;
        uint32_t cp = m;
        for (uint32_t k = kstart0; k < m; k += 8) {
          uint64_t x = stage_load8(stage, oi + k) ^ stage_load8(stage, o0 + k);
          const uint32_t take = m - k < 8 ? m - k : 8;
          if (take < 8) x &= (1ull << (8 * take)) - 1;
          if (x) {
            cp = k + (uint32_t)((__ffsll((long long)x) - 1) >> 3);
            break;
          }
        }
        my = cp < my ? cp : my;
      }
      my = __reduce_min_sync(0xFFFFFFFFu, my);
      if (lane_id() == 0 && my != 0xFFFFFFFFu) atomicMin(&s_lcp, my);
    }
    __syncthreads();
    const uint32_t lcp = s_lcp == 0xFFFFFFFFu ? 0u : (s_lcp / W) * W;  // whole units
    const uint32_t kstart = lcp > kstart0 ? lcp : kstart0;
    const FixLess less{stage, soff, sgid, kstart, (uint32_t)W};
    FT(0);
    // ---- sort items, blocked: thread t holds strings 8t .. 8t + 7
    uint64_t item[kFixItems];
#pragma unroll
    for (int j = 0; j < kFixItems; ++j) {
      const uint32_t i = threadIdx.x * kFixItems + j;
      uint64_t k = ~0ull;
      if (i < len) {
        const uint32_t nb = soff[i + 1] - soff[i];
        uint64_t key = 0;
        if (nb > kstart) {
          const uint32_t take = nb - kstart < 8 ? nb - kstart : 8;
          const uint64_t v = stage_load8(stage, soff[i] + kstart);  // little-endian bytes
          const uint64_t m = take == 8 ? ~0ull : ((1ull << (8 * take)) - 1);
          // big-endian by unit: bytes reversed (W = 1) / 16-bit units reversed (W = 2)
          constexpr uint32_t sel = W == 1 ? 0x0123u : 0x1032u;
          key = __byte_perm((uint32_t)((v & m) >> 32), 0, sel) |
                ((uint64_t)__byte_perm((uint32_t)(v & m), 0, sel) << 32);
        }
        k = (key & ~0xFFFFull) | i;  // top 48 bits of the key, then the slot
      }
      item[j] = k;
    }
    FT(1);
    Sort(sort_tmp).Sort(item, less);
    __syncthreads();
    FT(2);
    // ---- write back in the new order: perm, offsets (scan of the lengths), units
    uint32_t L[kFixItems], mine = 0;
#pragma unroll
    for (int j = 0; j < kFixItems; ++j) {
      const uint32_t q = (uint32_t)(item[j] & 0xFFFFu);
      L[j] = q != 0xFFFFu ? (soff[q + 1] - soff[q]) / W : 0u;
      mine += L[j];
    }
    if (GSTAGE) {
#pragma unroll
      for (int j = 0; j < kFixItems; ++j) {
        const uint32_t r = threadIdx.x * kFixItems + j, q = (uint32_t)(item[j] & 0xFFFFu);
        if (r < len) perm[start + r] = sgid[q];
      }
      if (threadIdx.x == 0) list[cap - 1 - e].y = len | kRunDone;  // done: k_fix_medium skips it
      __syncthreads();  // the stage and the sort storage are reused by the next run
      continue;
    }
    uint32_t tot;
    uint32_t d = block_exclusive_scan<uint32_t, kFixThreads>(mine, &tot, s_wt);
    uint32_t dq[kFixItems];  // output unit offset of each of my items
#pragma unroll
    for (int j = 0; j < kFixItems; ++j) {
      const uint32_t r = threadIdx.x * kFixItems + j, q = (uint32_t)(item[j] & 0xFFFFu);
      if (r < len) {
        perm[start + r] = sgid[q];
        so[start + r] = B0u + d;
      }
      dq[j] = d;
      d += L[j];
    }
    // the units: the run's bytes in the new order are assembled in shared
    // memory at the output's 16-byte phase (image byte x <-> su byte a0 + x,
    // the same phase as the stage), then the aligned body leaves with ONE
    // bulk async store (cp.async.bulk shared -> global) and the ragged edges
    // with plain stores
    uint8_t *image = stage + kFixStageBytes + 32 + kFixArrBytes;  // 16-byte aligned
    const uint32_t lead = (uint32_t)(B0 - a0);
#pragma unroll
    for (int j = 0; j < kFixItems; ++j) {
      const uint32_t q = (uint32_t)(item[j] & 0xFFFFu);
      if (q == 0xFFFFu) continue;
      const uint8_t *src = stage + soff[q];
      uint8_t *dst = image + lead + dq[j] * W;
      for (uint32_t b = 0; b < L[j] * W; ++b) dst[b] = src[b];
    }
    __syncthreads();
    const uint64_t c0 = (B0 + 15) & ~15ull;  // first aligned output byte inside the run
    if (bulk_ok && a1 > c0) {
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the image stores, for the async proxy
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(su + c0),
                     "r"((uint32_t)__cvta_generic_to_shared(image + (c0 - a0))), "r"((uint32_t)(a1 - c0))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      for (uint64_t x = B0 + threadIdx.x; x < c0; x += kFixThreads) su[x] = image[x - a0];
      for (uint64_t x = a1 + threadIdx.x; x < B1; x += kFixThreads) su[x] = image[x - a0];
      // the image (and the stage next to it) may be rewritten only after the
      // bulk store has read it
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    } else {
      for (uint64_t x = B0 + threadIdx.x; x < B1; x += kFixThreads) su[x] = image[x - a0];
    }
    __syncthreads();  // the stage and the sort storage are reused by the next run
    FT(3);
  }
}

extern "C" int husky_debug_fix_phases(unsigned long long *out) {
#ifdef HUSKY_FIX_TIMING
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_fix_phase, sizeof(g_fix_phase));
  return 1024;
#else
  (void)out;
  return 0;
#endif
}

void launch_fix_staged(int coder, const uint2 *list_sm, uint64_t cap_sm, const DevState *st, uint32_t *perm,
                       void *sorted_units, int64_t *sorted_offsets, int num_sms, cudaStream_t s,
                       const void *units, const int64_t *offsets, uint32_t first) {
  Scope sc_(ST_FIX_MEDIUM, s, 0);
  static SmemAttr a0, a1, a2, a3;
  dim3 g(num_sms), b(kFixThreads);
  uint2 *list = const_cast<uint2 *>(list_sm);
  const bool gst = sorted_units == nullptr;  // perm-only / after a refinement: gather-stage
#define FS_LAUNCH(C, G, A)                                                                                \
  do {                                                                                                  \
    A.ensure(k_fix_staged<C, G>, kFixSmem);                                                             \
    launch_pdl(k_fix_staged<C, G>, g, b, kFixSmem, s, list, cap_sm, st, perm, (uint8_t *)sorted_units,  \
               sorted_offsets, units, offsets, first);                                                  \
  } while (0)
  if (coder == HUSKY_CODER_ASCII) {
    if (gst) FS_LAUNCH(HUSKY_CODER_ASCII, true, a2);
    else FS_LAUNCH(HUSKY_CODER_ASCII, false, a0);
  } else {
    if (gst) FS_LAUNCH(HUSKY_CODER_UNICODE, true, a3);
    else FS_LAUNCH(HUSKY_CODER_UNICODE, false, a1);
  }
#undef FS_LAUNCH
}

// A tiny dirty run (<= kTinyMax strings) by ONE thread: the strings' offsets
// are loaded once, every pair is compared independently (their loads overlap)
// and each string goes to its rank.  A partial key sort (R19) leaves ~10^6
// two-string runs at 2^30 strings; a warp each left most lanes idle.
template <int CODER>
__device__ __forceinline__ void fix_tiny(uint32_t start, uint32_t len, uint32_t *perm, const void *units,
                                         const int64_t *offsets, const RunRule &rule, bool general,
                                         void *sorted_units, int64_t *sorted_offsets) {
  uint32_t id[kTinyMax], rank[kTinyMax];
  int64_t o[kTinyMax], l[kTinyMax];
#pragma unroll
  for (uint32_t i = 0; i < kTinyMax; ++i) {
    id[i] = i < len ? perm[start + i] : 0u;
    rank[i] = 0;
  }
#pragma unroll
  for (uint32_t i = 0; i < kTinyMax; ++i) {
    o[i] = i < len ? offsets[id[i]] : 0;
    l[i] = i < len ? offsets[id[i] + 1] - o[i] : 0;
  }
#pragma unroll
  for (uint32_t i = 1; i < kTinyMax; ++i) {
#pragma unroll
    for (uint32_t j = 0; j < i; ++j) {
      if (i >= len) continue;
      int c;  // string j against string i
      if (general) c = cmp_units_from<CODER>(units, o[j], l[j], o[i], l[i], 0);
      else if (l[j] <= rule.PL || l[i] <= rule.PL) c = l[j] < l[i] ? -1 : (l[j] > l[i] ? 1 : 0);
      else c = cmp_units_from<CODER>(units, o[j], l[j], o[i], l[i], rule.S);
      if (c == 0) c = id[j] < id[i] ? -1 : 1;
      if (c < 0) ++rank[i];
      else ++rank[j];
    }
  }
#pragma unroll
  for (uint32_t i = 0; i < kTinyMax; ++i)
    if (i < len) perm[start + rank[i]] = id[i];
  if (sorted_units) {
    // the main pass: the run's span in the sorted strings (its base and total
    // length are unchanged), rewritten in the new order -- no re-gather needed
    constexpr int W = CoderTraits<CODER>::kUnitBytes;
    const uint64_t base = (uint64_t)sorted_offsets[start];
#pragma unroll
    for (uint32_t i = 0; i < kTinyMax; ++i) {
      if (i >= len) continue;
      uint64_t d = base;
#pragma unroll
      for (uint32_t k = 0; k < kTinyMax; ++k)
        if (k < len && rank[k] < rank[i]) d += (uint64_t)l[k];
      sorted_offsets[start + rank[i]] = (int64_t)d;
      copy_units<W>((const uint8_t *)units, o[i], (uint8_t *)sorted_units, d, (uint64_t)l[i]);
    }
  }
}

// Small dirty runs (<= kSmallMax strings): each lane takes one list entry;
// runs of <= kTinyMax strings are fixed by that lane alone, larger ones by the
// whole warp, one after another (every lane ranks one string with the exact
// comparator).
template <int CODER>
__global__ void __launch_bounds__(256)
    k_fix_small(const uint2 *__restrict__ list, const DevState *st, uint32_t *perm,
                const void *__restrict__ units, const int64_t *__restrict__ offsets, uint32_t first,
                void *sorted_units, int64_t *sorted_offsets) {
  pdl_wait();
  if (st->violations & kOffsetsBad) return;
  const uint32_t lane = lane_id();
  const RunRule rule = run_rule<CODER>(st);
  const uint32_t nsmall = st->n_small;
  const bool general = st->general != 0;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t b = first + (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; b < nsmall; b += warps * 32) {
    const uint32_t e = b + lane;
    const uint2 mine = e < nsmall ? list[e] : make_uint2(0, 0);
    if (mine.y) HCHK(kChkFixSmallPerm, (uint64_t)mine.x + mine.y, st->chk_n + 1);
    if (mine.y >= 2 && mine.y <= kTinyMax)
      fix_tiny<CODER>(mine.x, mine.y, perm, units, offsets, rule, general, sorted_units, sorted_offsets);
    uint32_t big = __ballot_sync(0xFFFFFFFFu, mine.y > kTinyMax);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const uint32_t start = __shfl_sync(0xFFFFFFFFu, mine.x, src), len = __shfl_sync(0xFFFFFFFFu, mine.y, src);
      uint32_t my = lane < len ? perm[start + lane] : 0xFFFFFFFFu;
      uint32_t rank = 0;
      for (uint32_t j = 0; j < len; ++j) {
        uint32_t other = __shfl_sync(0xFFFFFFFFu, my, j);
        if (lane < len && j != lane &&
            (general ? cmp_general<CODER>(units, offsets, other, my)
                     : cmp_equal_code<CODER>(units, offsets, other, my, rule.S, rule.PL)) < 0)
          ++rank;
      }
      __syncwarp();
      if (lane < len) perm[start + rank] = my;
      __syncwarp();
    }
  }
}

template <int CODER>
__global__ void __launch_bounds__(1024)
    k_fix_medium(const uint2 *__restrict__ list, uint64_t cap, const DevState *st, uint32_t *perm,
                 const void *__restrict__ units, const int64_t *__restrict__ offsets, uint32_t first,
                 const int64_t *__restrict__ so) {
  using T = CoderTraits<CODER>;
  __shared__ uint32_t s[kMediumMax];
  pdl_wait();
  if (st->violations & kOffsetsBad) return;
  const uint32_t nmed = st->n_medium;
  const RunRule rule = run_rule<CODER>(st);
  const bool general = st->general != 0;
  for (uint32_t e = first + blockIdx.x; e < nmed; e += gridDim.x) {
    uint2 ent = list[cap - 1 - e];
    if (ent.y & kRunDone) continue;  // sorted by the gather-staged kernel
    const uint32_t start = ent.x, len = ent.y;
    if (staged_run<T::kUnitBytes>(st, so, start, len)) continue;
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
                               : cmp_equal_code<CODER>(units, offsets, a, b, rule.S, rule.PL)) > 0;
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
                      const void *units, const int64_t *offsets, int num_sms, cudaStream_t s, uint32_t first,
                      void *sorted_units, int64_t *sorted_offsets) {
  Scope sc_(ST_FIX_SMALL, s, 0);
  dim3 g(num_sms * 4), b(256);
  if (coder == HUSKY_CODER_ASCII)
    launch_pdl(k_fix_small<HUSKY_CODER_ASCII>, g, b, 0, s, list_sm, st, perm, units, offsets, first, sorted_units,
               sorted_offsets);
  else
    launch_pdl(k_fix_small<HUSKY_CODER_UNICODE>, g, b, 0, s, list_sm, st, perm, units, offsets, first,
               sorted_units, sorted_offsets);
}

void launch_fix_medium(int coder, const uint2 *list_sm, uint64_t cap_sm, const DevState *st,
                       uint32_t *perm, const void *units, const int64_t *offsets, int num_sms,
                       cudaStream_t s, uint32_t first, const int64_t *staged_so) {
  Scope sc_(ST_FIX_MEDIUM, s, 0);
  dim3 g(num_sms), b(1024);
  if (coder == HUSKY_CODER_ASCII)
    launch_pdl(k_fix_medium<HUSKY_CODER_ASCII>, g, b, 0, s, list_sm, cap_sm, st, perm, units, offsets, first,
               staged_so);
  else
    launch_pdl(k_fix_medium<HUSKY_CODER_UNICODE>, g, b, 0, s, list_sm, cap_sm, st, perm, units, offsets, first,
               staged_so);
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
  const int64_t pl = run_rule<CODER>(st).PL;  // the short rule of this sort (R6 / R19)
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
    if (l <= pl && !st->general) has_short = 1;  // short rule: equal codes only (R6)
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
  const int64_t pl = run_rule<CODER>(st).PL;  // the short rule of this sort (R6 / R19)
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
      if (l <= pl && st->seg_has_short) {
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
