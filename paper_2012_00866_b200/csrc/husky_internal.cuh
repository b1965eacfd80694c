// husky_internal.cuh -- shared device helpers and the workspace-resident state
// of libhusky (sm_100a only).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/husky.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libhusky is written for sm_100a (B200) only"
#endif

namespace husky {

// ---------------------------------------------------------------- constants
// Code windows: ASCII 9 units x 7 bits, UNICODE 4 x 16 bits.
// S  = number of leading units fully determined by equal codes (R6):
//      ASCII 9; UNICODE 3 (unit 3 loses its low bit to ">>> 1").
// PL = perfect length (reading R4): ASCII 9, UNICODE 3.
template <int CODER> struct CoderTraits;
template <> struct CoderTraits<HUSKY_CODER_ASCII> {
  using unit_t = uint8_t;
  static constexpr int kUnitBytes = 1, kS = 9, kPL = 9;
  static constexpr int kWin = 7;    // refinement window: 7 units x 8 bits
  static constexpr int kTagCap = 8; // tag value meaning "continues past the window"
  static constexpr int kSlabMax = 24; // slab record: units [9, 24) after the code's 9
};
template <> struct CoderTraits<HUSKY_CODER_UNICODE> {
  using unit_t = uint16_t;
  static constexpr int kUnitBytes = 2, kS = 3, kPL = 3;
  static constexpr int kWin = 3;    // 3 units x 16 bits
  static constexpr int kTagCap = 4;
  static constexpr int kSlabMax = 10; // slab record: units [3, 10) after the code's 3
};

// ENGLISH5 / ENGLISH6 (reading R15): byte units; only the
// encoder is specific to them -- every other kernel runs its ASCII (byte)
// instantiation, whose S = 9 / PL = 9 are conservative for these coders (equal
// 5/6-bit codes on the coder's domain imply equal first 12 / 10 units).
template <> struct CoderTraits<HUSKY_CODER_ENGLISH5> {
  using unit_t = uint8_t;
  static constexpr int kUnitBytes = 1, kS = 12, kPL = 12, kK = 12, kBits = 5;
  static constexpr int kWin = 7, kTagCap = 8;
};
template <> struct CoderTraits<HUSKY_CODER_ENGLISH6> {
  using unit_t = uint8_t;
  static constexpr int kUnitBytes = 1, kS = 10, kPL = 10, kK = 10, kBits = 6;
  static constexpr int kWin = 7, kTagCap = 8;
};

constexpr int kSmallMax = 32;    // dirty runs up to this many strings: one warp
constexpr uint32_t kTinyMax = 4; // ... and up to this many: one thread
// medium-list entry flag (length field): the run was sorted by the
// gather-staged fix-up (perm-only mode / after a refinement)
constexpr uint32_t kRunDone = 0x80000000u;
constexpr int kMediumMax = 4096; // ... up to this many: one CTA (bitonic in smem)

// violation bits (OR-reduced; zero-initialised state)
constexpr uint32_t kNotPerfect = 1u, kDomainBad = 2u, kOffsetsBad = 4u;
// ENGLISH5 domain (reading R15): a window unit that is not a lowercase / not an
// uppercase letter; the domain holds unless both bits are set
constexpr uint32_t kNotLower = 8u, kNotUpper = 16u;

// ------------------------------------------------------ device-resident state
// LSD digits: 8 bits (9-bit digits -- 7 passes for the 63-bit codes -- measured
// ~14% slower per pass, so no faster in total: DESIGN.md 6.1).
constexpr int kDigitBits = 8;
constexpr int kBins = 1 << kDigitBits;
// Lives at the start of the caller's workspace; zeroed once per husky_sort.
struct DevState {
  uint32_t hist[8][kBins];        // digit histograms of the 64-bit keys
  uint32_t digit_start[8][kBins]; // their exclusive scans
  uint32_t trivial_mask;      // bit d: all keys share digit d
  uint32_t violations;        // kNotPerfect | kDomainBad | kOffsetsBad
  uint32_t tile_counter[64];  // dynamic tile ids, one per launch slot
  uint32_t n_runs;            // runs (>= 2 equal keys) found by the last run scan
  uint32_t n_small, n_medium, n_giant; // dirty-run list fill counts
  unsigned long long n_in_runs, max_run;
  unsigned long long runs_by_class[4];
  uint32_t seg_L;             // refinement: common-prefix length of the segment
  uint32_t seg_has_short;     // refinement: segment contains a string with len <= PL
  unsigned long long runs_total; // runs found by the main (code) scan
  // device-side radix plan (launch_hist_plan): the non-trivial digits in pass order
  // and which ping-pong key buffer ends up holding the sorted codes
  uint32_t np;
  uint32_t hist_done;       // k_hist_slots<true>: CTAs that have added their histograms
  uint32_t pass_digit[8];
  unsigned long long sorted_keys;  // uint64_t* of the sorted keys
  // general cleanup (NEXT-4): the coder is not monotone on this input, so the
  // refinement / fix-up kernels compare whole strings from unit 0 instead of
  // relying on equal codes (no short rule, no known-equal prefix)
  uint32_t general;
  // alphabet compression of ASCII codes (radix.cu): which 7-bit field values
  // occur in the code windows (bit v of alpha), and whether the sort's keys
  // were re-packed with cbits bits per field (ccomp)
  uint32_t alpha[4];
  uint32_t ccomp, cbits;
  // the run rule of this sort (k_hist_slots<PLAN>; 0 = the coder's defaults):
  // keys are equal for run detection when equal under key_mask; equal masked
  // keys fix units [0, seq_units), and a string of <= short_len units is then
  // a prefix of the other (R6 / R19)
  uint32_t seq_units, short_len;
  unsigned long long key_mask;
  uint32_t pad[1];
  // checked builds (HUSKY_CHECKED): n and the byte end of the units
  // (offsets[n] x unit bytes) of this sort, the bounds HCHK compares against
  unsigned long long chk_n, chk_units;
};

// The run rule kernels apply: by default equal codes fix units [0, S) and the
// short rule holds for lengths <= PL (R6); a sort whose plan leaves the lowest
// digit unsorted (R19) has a shorter fixed prefix and masks that digit out of
// run detection.
struct RunRule {
  uint32_t S, PL;
  unsigned long long mask;
};
template <int CODER>
__device__ __forceinline__ RunRule run_rule(const DevState *st) {
  using T = CoderTraits<CODER>;
  if (st == nullptr || st->seq_units == 0) return RunRule{(uint32_t)T::kS, (uint32_t)T::kPL, ~0ull};
  return RunRule{st->seq_units, st->short_len, st->key_mask};
}

// Alphabet compression (ASCII): the code's nine 7-bit fields re-packed as
// their ranks among the field values present (0 -- padding / NUL -- always
// counted), cbits = ceil(log2(#values)) bits each.  A monotone bijection of
// each field, so the order of codes, equality of codes, and hence every run is
// unchanged; with <= 64 values (cbits <= 6) the key fits 56 bits and the LSD
// sort needs 7 passes instead of 8 (<= 32 values, e.g. one letter case: 6).
__device__ __forceinline__ uint32_t alpha_bits(const uint32_t a[4]) {
  const uint32_t cnt = __popc(a[0] | 1u) + __popc(a[1]) + __popc(a[2]) + __popc(a[3]);
  return cnt <= 1 ? 0u : 32u - __clz(cnt - 1);  // ceil(log2(cnt))
}
// rank of field value v (0..127) among the present values
__device__ __forceinline__ uint32_t alpha_rank(const uint32_t a[4], uint32_t v) {
  const uint32_t w = v >> 5, below = (1u << (v & 31)) - 1u;
  uint32_t r = __popc((w == 0 ? (a[0] | 1u) : a[w]) & below);
  if (w > 0) r += __popc(a[0] | 1u);
  if (w > 1) r += __popc(a[1]);
  if (w > 2) r += __popc(a[2]);
  return r;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per device and kernel:
// the attribute belongs to the kernel's function handle in each device's
// context, so a process that sorts on several GPUs sets it on each of them.
struct SmemAttr {
  std::atomic<unsigned long long> done{0};
  template <typename F>
  cudaError_t ensure(F *func, int bytes) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
  }
};

// ----------------------------------------------------------- small helpers
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
// programmatic dependent launch: wait for the preceding kernel's results (a
// no-op for kernels launched without the PDL attribute)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Lanes holding the same 8-bit label as this lane (converged warp): one ballot
// per label bit -- an alternative to __match_any_sync whose cost on sm_100a
// depends on the label distribution.
template <int BITS>
__device__ __forceinline__ uint32_t match_ballot(uint32_t label) {
  uint32_t m = 0xFFFFFFFFu;
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
    const bool bit = (label >> b) & 1u;
    const uint32_t v = __ballot_sync(0xFFFFFFFFu, bit);
    m &= bit ? v : ~v;
  }
  return m;
}


__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back flag word: [63:62] status (1 = aggregate, 2 = inclusive),
// [61:54] epoch (1..255), [53:0] value.
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 54) - 1;
__device__ __forceinline__ unsigned long long make_flag(unsigned long long status, uint32_t epoch,
                                                        unsigned long long v) {
  return status | ((unsigned long long)epoch << 54) | (v & kValMask);
}
// Walks predecessors of `tile` at stride `stride` (flags[t*stride]) until an
// inclusive prefix is found; returns the exclusive prefix for `tile`.
__device__ __forceinline__ unsigned long long lookback(const unsigned long long *flags, uint32_t tile,
                                                       uint32_t stride, uint32_t epoch) {
  unsigned long long excl = 0;
  int64_t j = (int64_t)tile - 1;
  while (j >= 0) {
    unsigned long long w = ld_relaxed_u64(flags + (uint64_t)j * stride);
    uint32_t ep = (uint32_t)(w >> 54) & 0xFF;
    unsigned long long st = w & (3ull << 62);
    if (ep != epoch || st == 0) continue;  // not yet published in this epoch
    excl += w & kValMask;
    if (st == kFlagInc) break;
    --j;
  }
  return excl;
}

// Windowed look-back for one value per thread: loads W predecessor words at
// once (nearest first) and consumes them in order; an unpublished word stops
// the window and is re-read.  One round trip covers up to W tiles.
template <int W>
__device__ __forceinline__ unsigned long long lookback_window(const unsigned long long *flags, uint32_t tile,
                                                              uint32_t stride, uint32_t epoch,
                                                              uint32_t *stats = nullptr) {
  unsigned long long excl = 0;
  int64_t j = (int64_t)tile - 1;
  while (j >= 0) {
    if (stats) stats[0]++;
    unsigned long long w[W];
#pragma unroll
    for (int q = 0; q < W; ++q)
      w[q] = (j - q >= 0) ? ld_relaxed_u64(flags + (uint64_t)(j - q) * stride) : make_flag(kFlagInc, epoch, 0);
    int used = 0;
    bool done = false;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      if (done || used != q) break;
      unsigned long long x = w[q];
      bool ok = ((uint32_t)(x >> 54) & 0xFF) == epoch && (x & (3ull << 62)) != 0;
      if (!ok) break;
      excl += x & kValMask;
      used = q + 1;
      if ((x & (3ull << 62)) == kFlagInc) done = true;
    }
    if (done) break;
    j -= used;
    if (used == 0) {
      // the nearest predecessor has not published yet: poll just that word,
      // backing off so the spinning warp leaves issue slots to working warps
      unsigned ns = 32;
      for (;;) {
        unsigned long long x = ld_relaxed_u64(flags + (uint64_t)j * stride);
        if (((uint32_t)(x >> 54) & 0xFF) == epoch && (x & (3ull << 62)) != 0) break;
        if (stats) stats[1]++;
        __nanosleep(ns);
        if (ns < 512) ns <<= 1;
      }
    }
  }
  return excl;
}


// Warp-cooperative look-back (all 32 lanes call it): one round trip reads the
// 32*V nearest unconsumed predecessors (lane l the V words of tiles
// base - V*l - v, v = 0..V-1); the nearest inclusive word ends the walk.
// Returns the exclusive prefix of `tile` in every lane.
// A walk that starts d tiles past the inclusive frontier takes d / (32 V)
// round trips, so a single-pass scan cannot retire more than 32 V tiles per
// round trip whatever its concurrency (the gather at 2^30 strings was bound
// there with V = 1: 21.6 G strings/s = 32 tiles of 1024 per ~1.5 us).
template <int V = 1>
__device__ __forceinline__ unsigned long long warp_lookback(const unsigned long long *flags, uint32_t tile,
                                                            uint32_t epoch) {
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long excl = 0;
  int64_t base = (int64_t)tile - 1;
  while (base >= 0) {
    unsigned long long x[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int64_t j = base - (int64_t)(V * lane + v);
      x[v] = j >= 0 ? ld_relaxed_u64(flags + j) : make_flag(kFlagInc, epoch, 0);
    }
    // this lane's consumable prefix of its V words (nearest first): up to the
    // first unpublished word (exclusive) or the first inclusive word (inclusive)
    uint32_t k = 0;
    bool inc = false;
    unsigned long long part = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (k != (uint32_t)v || inc) break;
      const bool valid = ((uint32_t)(x[v] >> 54) & 0xFF) == epoch && (x[v] & (3ull << 62)) != 0;
      if (!valid) break;
      part += x[v] & kValMask;
      k = v + 1;
      inc = (x[v] & (3ull << 62)) == kFlagInc;
    }
    const bool full = k == (uint32_t)V && !inc;
    const uint32_t notfull = __ballot_sync(0xFFFFFFFFu, !full);
    const uint32_t L = notfull ? (uint32_t)(__ffs(notfull) - 1) : 32u;  // first lane that stopped
    unsigned long long v = lane <= L ? part : 0ull;  // lanes before L: all V words; lane L: its prefix
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    excl += v;
    if (L == 32) {
      base -= 32 * V;
      continue;
    }
    const uint32_t kL = __shfl_sync(0xFFFFFFFFu, k, L);
    const bool stop = __shfl_sync(0xFFFFFFFFu, (int)inc, L) != 0;
    if (stop) break;
    const uint32_t take = L * V + kL;
    base -= take;
    if (take == 0) __nanosleep(64);  // nearest predecessor unpublished: back off
  }
  return excl;
}

// Warp inclusive scan (Kogge-Stone over shuffles).
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xFFFFFFFFu, v, o);
    if (lane >= (uint32_t)o) v += t;
  }
  return v;
}

// Block-wide exclusive scan for blockDim.x == THREADS.  `warp_tot` is smem of
// THREADS/32 elements.  Returns the exclusive prefix; *total = block sum.
// Contains __syncthreads (all threads must call).
template <typename T, int THREADS>
__device__ __forceinline__ T block_exclusive_scan(T v, T *total, T *warp_tot) {
  constexpr int NW = THREADS / 32;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T x = lane < NW ? warp_tot[lane] : T(0);
    T xi = warp_inclusive_scan(x);
    if (lane < NW) warp_tot[lane] = xi - x;  // exclusive per warp
    if (lane == NW - 1) warp_tot[NW] = xi;   // block total (warp_tot has NW+1 slots)
  }
  __syncthreads();
  T r = warp_tot[warp] + inc - v;
  *total = warp_tot[NW];
  return r;
}

// Asynchronous global -> shared copies (LDGSTS): many in flight per thread, no
// register round trip.  cp_async_wait_all() + __syncthreads() before reading.
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gmem_src) {
  uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem_dst, const void *gmem_src) {
  uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Unaligned little-endian load of 8 bytes at byte address p, reading only the
// aligned 8-byte words that contain bytes [p, p + need) (need in 1..8), so it
// never touches a word without a needed byte.
__device__ __forceinline__ uint64_t load8_unaligned(const uint8_t *p, int need) {
  uintptr_t a = (uintptr_t)p;
  const uint64_t *w = (const uint64_t *)(a & ~(uintptr_t)7);
  int sh = (int)(a & 7);
  uint64_t lo = __ldg(w);
  if (sh == 0) return lo;
  uint64_t v = lo >> (8 * sh);
  if (sh + need > 8) v |= __ldg(w + 1) << (64 - 8 * sh);
  return v;
}

// Byte b (0..8) of an ASCII string rebuilt from its alphabet-compressed code:
// field b holds the rank, unrank[] maps it back to the unit.
__device__ __forceinline__ uint8_t decode_byte_c(uint64_t code, int b, uint32_t bits, const uint8_t *unrank) {
  return unrank[(uint32_t)(code >> (bits * (8 - b))) & ((1u << bits) - 1u)];
}

// Byte k (1..15) of a slab record held in registers.
__device__ __forceinline__ uint8_t slab_byte(const uint4 &v, int k) {
  const uint32_t w = (k >> 2) == 0 ? v.x : ((k >> 2) == 1 ? v.y : ((k >> 2) == 2 ? v.z : v.w));
  return (uint8_t)(w >> (8 * (k & 3)));
}

// Compare two unit strings a[0..la), b[0..lb) lexicographically (unsigned units),
// starting at unit `from` (units before it are known equal).  Returns <0, 0, >0
// where 0 means equal content AND equal length.
template <int CODER>
__device__ __forceinline__ int cmp_units_from(const void *units, int64_t oa, int64_t la, int64_t ob,
                                              int64_t lb, int64_t from) {
  constexpr int W = CoderTraits<CODER>::kUnitBytes;
  int64_t m = (la < lb ? la : lb);
  const uint8_t *base = (const uint8_t *)units;
  for (int64_t k = from; k < m;) {
    int64_t rem_units = m - k;
    int take = (int)(rem_units * W < 8 ? rem_units * W : 8);  // bytes
    uint64_t x = load8_unaligned(base + (oa + k) * W, take);
    uint64_t y = load8_unaligned(base + (ob + k) * W, take);
    if (take < 8) {
      uint64_t msk = (1ull << (8 * take)) - 1;
      x &= msk;
      y &= msk;
    }
    uint64_t d = x ^ y;
    if (d) {
      int bit = __ffsll((long long)d) - 1;
      int sh = (bit / (8 * W)) * (8 * W);
      uint64_t um = W == 1 ? 0xFFull : 0xFFFFull;
      uint64_t ux = (x >> sh) & um, uy = (y >> sh) & um;
      return ux < uy ? -1 : 1;
    }
    k += take / W;
  }
  if (la != lb) return la < lb ? -1 : 1;
  return 0;
}

// Byte b of a string whose units are fully determined by its husky code (ASCII
// length <= 9, UNICODE length <= 3): the inverse of Alg. 4's packing.
template <int CODER>
__device__ __forceinline__ uint8_t decode_byte(uint64_t code, int b) {
  if (CODER == HUSKY_CODER_ASCII) return (uint8_t)((code >> (56 - 7 * b)) & 0x7F);
  uint32_t u = (uint32_t)(((code << 1) >> (48 - 16 * (b >> 1))) & 0xFFFF);
  return (uint8_t)(b & 1 ? u >> 8 : u);
}

// 8 bytes at an arbitrary byte offset of the stage (little-endian), from three
// aligned 32-bit words (the stage has 32 bytes of slack past its end)
__device__ __forceinline__ uint64_t stage_load8(const uint8_t *stage, uint32_t off) {
  const uint32_t *sw = reinterpret_cast<const uint32_t *>(stage) + (off >> 2);
  const uint32_t sh = (off & 3) * 8;
  const uint32_t x0 = sw[0], x1 = sw[1], x2 = sw[2];
  return (uint64_t)__funnelshift_r(x0, x1, sh) | ((uint64_t)__funnelshift_r(x1, x2, sh) << 32);
}

// Copy one string's units (L units of W bytes) from ub + o*W to ob + d*W:
// unaligned 8-byte loads, byte stores.
template <int W>
__device__ __forceinline__ void copy_units(const uint8_t *ub, int64_t o, uint8_t *ob, uint64_t d, uint64_t L) {
  const uint64_t nb = L * W;
  const uint8_t *sp = ub + o * W;
  uint8_t *dp = ob + d * W;
  // bytes up to the destination's next 8-byte boundary, then aligned 8-byte
  // stores, then the tail: a 24-byte string takes ~2 wide stores and <= 14 byte
  // stores instead of 24 byte stores (scattered byte stores are what a
  // one-thread-per-run fix-up pays for, C5: ~1.2 M runs)
  const uint64_t head = (8 - ((uintptr_t)dp & 7)) & 7;
  uint64_t q = head < nb ? head : nb;
  if (q) {
    const uint64_t v = load8_unaligned(sp, (int)q);
    for (int b = 0; b < (int)q; ++b) dp[b] = (uint8_t)(v >> (8 * b));
  }
  for (; q + 8 <= nb; q += 8) *reinterpret_cast<uint64_t *>(dp + q) = load8_unaligned(sp + q, 8);
  if (q < nb) {
    const int take = (int)(nb - q);
    const uint64_t v = load8_unaligned(sp + q, take);
    for (int b = 0; b < take; ++b) dp[q + b] = (uint8_t)(v >> (8 * b));
  }
}

// Exact comparator with no assumption on the codes (general cleanup, NEXT-4):
// units from 0, a proper prefix first, then the index.
template <int CODER>
__device__ __forceinline__ int cmp_general(const void *units, const int64_t *offsets, uint32_t ia, uint32_t ib) {
  int64_t oa = offsets[ia], la = offsets[ia + 1] - oa;
  int64_t ob = offsets[ib], lb = offsets[ib + 1] - ob;
  int c = cmp_units_from<CODER>(units, oa, la, ob, lb, 0);
  if (c) return c;
  return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

// Exact comparator for two strings whose husky codes are EQUAL (under the run
// rule's mask, R6 / R19): if either length <= pl the shorter one is
// a prefix of the longer (order by length, then index); otherwise units [0, S)
// are equal and the comparison starts at unit `from` (>= S).
// pl: the short-rule length (RunRule::PL).
template <int CODER>
__device__ __forceinline__ int cmp_equal_code(const void *units, const int64_t *offsets, uint32_t ia,
                                              uint32_t ib, int64_t from, int64_t pl) {
  int64_t oa = offsets[ia], la = offsets[ia + 1] - oa;
  int64_t ob = offsets[ib], lb = offsets[ib + 1] - ob;
  int c;
  if (la <= pl || lb <= pl) c = (la < lb) ? -1 : (la > lb ? 1 : 0);
  else c = cmp_units_from<CODER>(units, oa, la, ob, lb, from);
  if (c) return c;
  return ia < ib ? -1 : (ia > ib ? 1 : 0);
}


// ---------------------------------------------------------------- checked build
// HUSKY_NVCC_DEFS=-DHUSKY_CHECKED (a separate lab build, tools/gpu_checked.sh):
// the kernels' output indices and random-read indices are checked against
// their bounds and violations counted -- never trapping, so a bad index cannot
// take the GPU down.  husky_sort / husky_sort_multi_exec then fail with
// HUSKY_ERR_CUDA and "checked build: ...".  This stands in for
// compute-sanitizer memcheck, which is closed on this GPU pool
// (profiles/r02_sanitizer.txt).  Site ids: kChk* below.
enum : unsigned {
  kChkRadixScatter = 1, kChkGatherPerm = 2, kChkGatherOffsets = 3, kChkGatherUnits = 4, kChkGatherRuns = 5,
  kChkFixStagedUnits = 6, kChkFixStagedOffsets = 7, kChkFixTiny = 8, kChkRegather = 9, kChkEncodeSlab = 10,
  kChkFixSmallPerm = 11, kChkPeer = 12
};
#ifdef HUSKY_CHECKED
// one counter pair per translation unit (no relocatable device code); the
// host side sums them through the readers each unit registers at load time
static __device__ unsigned long long g_chk[2];  // [0] violations, [1] first: site << 48 | index
#define HCHK(site, idx, bound)                                                                         \
  do {                                                                                                 \
    const unsigned long long i_ = (unsigned long long)(idx), b_ = (unsigned long long)(bound);          \
    if (i_ >= b_ && atomicAdd(&::husky::g_chk[0], 1ull) == 0ull)                                       \
      ::husky::g_chk[1] = ((unsigned long long)(site) << 48) | (i_ & 0xFFFFFFFFFFFFull);                \
  } while (0)
typedef unsigned long long (*ChkReader)(unsigned long long *first);
int checked_register(ChkReader r);  // husky.cu
// violations since the last call (summed over the units), *first = one of them
unsigned long long checked_take(unsigned long long *first);
static unsigned long long chk_read_unit(unsigned long long *first) {
  unsigned long long h[2] = {0, 0}, z[2] = {0, 0};
  cudaMemcpyFromSymbol(h, g_chk, sizeof h);
  cudaMemcpyToSymbol(g_chk, z, sizeof z);
  if (h[0] && first) *first = h[1];
  return h[0];
}
static const int g_chk_registered = checked_register(chk_read_unit);
#else
#define HCHK(site, idx, bound) \
  do {                         \
  } while (0)
#endif

}  // namespace husky
