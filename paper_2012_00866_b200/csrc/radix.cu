// radix.cu -- A2: stable LSD radix sort of (64-bit key, 32-bit payload).
//
// Role in the paper: step 2 of Alg. 1, "Sort array longs ... in such a way that
// when elements i, j of longs are exchanged, then elements i, j of xs are also
// exchanged".  Introsort's comparisons are replaced
// by an LSD radix sort whose payload is the string index, so the co-swap is the
// payload scatter.  Being stable, it leaves equal codes in index order
// (R7), which the fix-up (A5) relies on.
//
// Digit width: 8 bits (kernels are templated on it; the device-planned slots
// can be built with 9-bit digits, HUSKY_SLOT_BITS=9: 7 passes for the 63-bit
// codes, measured no faster -- husky_internal.cuh).
// A pass works on tiles of kRadixTile = 6144 keys (512 threads x 12, warp-striped so every
// load/store instruction is a coalesced 256-B access).  Each tile is ranked in
// shared memory with warp-level label matching (three __match_any_sync on the
// digit's 3 + 3 + 2 bits, HUSKY_RANK_NIBBLE) + popc into per-warp digit
// counters, exchanged through shared memory into digit order, and written out
// as runs of consecutive addresses.  The tile's global base per digit comes
// from one of two schemes:
//   * onesweep (default): per-(tile, digit) decoupled look-back (Adinets &
//     Merrill), global digit starts from the 8 digit histograms of the codes
//     (k_hist_slots).  One read of the keys per pass, but the look-back is a
//     chain of dependent L2 round trips (~1 us each with the memory system
//     saturated; measured per-tile phases in DESIGN.md).
//   * reduce-then-scan (HUSKY_RADIX=rts, host-planned passes only): an upsweep
//     writes each tile's digit counts (8 B/key read), a digit-parallel scan
//     turns them into per-tile bases, and the downsweep ranks/exchanges/scatters
//     with no inter-tile dependency (measured slower).
// Digits whose histogram puts all keys in one bucket are skipped.
#include <algorithm>

#include "husky_internal.cuh"
#include "kernels.cuh"

namespace husky {

// Exclusive scan of hist[d][0..255] -> digit_start[d]; trivial_mask bit d when
// one digit value holds all n keys (that pass is the identity and is skipped).
// Also digit_spread[d]: the largest bin holds < 5% of the keys (many distinct
// labels per warp: rank that digit with per-bit ballots).
template <int BITS>
__global__ void __launch_bounds__(1 << BITS) k_hist_scan(uint64_t n, DevState *st) {
  constexpr int R = 1 << BITS;
  __shared__ uint32_t wt[R / 32 + 1];
  __shared__ uint32_t s_max[R / 32];
  const int d = blockIdx.x;
  uint32_t v = st->hist[d][threadIdx.x];
  uint32_t total;
  uint32_t ex = block_exclusive_scan<uint32_t, R>(v, &total, wt);
  st->digit_start[d][threadIdx.x] = ex;
  if ((uint64_t)v == n) atomicOr(&st->trivial_mask, 1u << d);
  const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, v);
  if (lane_id() == 0) s_max[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t mx = 0;
    for (int w = 0; w < R / 32; ++w) mx = s_max[w] > mx ? s_max[w] : mx;
    st->digit_spread[d] = (uint64_t)mx * 20 < n;
  }
}

void launch_hist_scan(uint64_t n, DevState *st, cudaStream_t s) {
  Scope sc_(ST_HIST_SCAN, s, n);
  k_hist_scan<8><<<8, 256, 0, s>>>(n, st);
}

// The 8 digit histograms (kSlotBits-bit digits) of the codes for the LSD
// onesweep (A2): one read of the codes, plain shared-memory atomics.  Measured
// on C2: 35 us as a separate pass vs 51 us when fused into the encoder's loop,
// and 8x slower with __match_any_sync aggregation.  PLAN: the
// last CTA to add its histograms (ticket) also does k_hist_scan's scans and
// the pass plan (which digits to sort, in which order, with which ranking
// primitive), saving two dependent launches.
#ifndef HUSKY_HIST_BPS
#define HUSKY_HIST_BPS 4
#endif
constexpr int kHistBlocksPerSM = HUSKY_HIST_BPS;  // resident CTAs of 512 threads per SM
template <bool PLAN>
__global__ void __launch_bounds__(512) k_hist_slots(const uint64_t *__restrict__ keys, uint64_t n, DevState *st,
                                                    uint64_t *keysA, uint64_t *keysB, uint32_t force_ballot,
                                                    uint32_t force_match) {
  constexpr int R = 1 << kSlotBits;
  constexpr uint32_t M = R - 1;
  pdl_wait();  // PLAN: launched as a programmatic dependent of the encoder
  __shared__ uint32_t h[8 * R];
  __shared__ uint32_t s_last, s_wt[512 / 32 + 1], s_max[512 / 32];
  for (int i = threadIdx.x; i < 8 * R; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * 4; base < n; base += stride) {
    uint64_t k[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint64_t i = base + threadIdx.x + (uint64_t)r * blockDim.x;
      k[r] = i < n ? __ldg(keys + i) : 0;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (base + threadIdx.x + (uint64_t)r * blockDim.x >= n) continue;
#pragma unroll
      for (int d = 0; d < 8; ++d) atomicAdd(&h[d * R + ((uint32_t)(k[r] >> (kSlotBits * d)) & M)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * R; i += blockDim.x)
    if (h[i]) atomicAdd(&st->hist[i / R][i % R], h[i]);
  if (!PLAN) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&st->hist_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // the last CTA: exclusive scans, trivial digits, spread (as k_hist_scan), then the plan
  uint32_t trivial = 0, spread = 0;
  for (int d = 0; d < 8; ++d) {
    const uint32_t v = threadIdx.x < R ? __ldcg(&st->hist[d][threadIdx.x]) : 0u;
    uint32_t total;
    const uint32_t ex = block_exclusive_scan<uint32_t, 512>(v, &total, s_wt);
    if (threadIdx.x < R) st->digit_start[d][threadIdx.x] = ex;
    const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, v);
    if (lane_id() == 0) s_max[threadIdx.x >> 5] = m;
    const bool all_here = __syncthreads_or((uint64_t)v == n) != 0;
    uint32_t mx = 0;
    for (int w = 0; w < 512 / 32; ++w) mx = s_max[w] > mx ? s_max[w] : mx;
    trivial |= (uint32_t)all_here << d;
    spread |= (uint32_t)((uint64_t)mx * 20 < n) << d;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    st->trivial_mask = trivial;
    uint32_t np = 0;
    for (int d = 0; d < 8; ++d) {
      st->digit_spread[d] = (spread >> d) & 1;
      if (!((trivial >> d) & 1)) {
        st->pass_ballot[np] = ((force_ballot >> d) & 1) || (((spread >> d) & 1) && !((force_match >> d) & 1));
        st->pass_digit[np++] = d;
      }
    }
    st->np = np;
    st->sorted_keys = (unsigned long long)((np & 1) ? keysB : keysA);
  }
}

static uint32_t env_mask(const char *name) {
  const char *v = getenv(name);
  return v ? (uint32_t)strtoul(v, nullptr, 0) : 0u;
}

void launch_hist_slots(const uint64_t *keys, uint64_t n, DevState *st, int num_sms, cudaStream_t s) {
  if (n == 0) return;
  Scope sc_(ST_HIST_SCAN, s, n);
  const uint64_t blocks = std::min<uint64_t>((n + 2047) / 2048, (uint64_t)num_sms * kHistBlocksPerSM);
  k_hist_slots<false><<<(unsigned)blocks, 512, 0, s>>>(keys, n, st, nullptr, nullptr, 0, 0);
}

// histograms + scans + pass plan of the device-planned passes in one launch
// (DevState::hist_done must be 0: DevState is zeroed per sort)
void launch_hist_plan(const uint64_t *keys, uint64_t n, DevState *st, uint64_t *keysA, uint64_t *keysB,
                      int num_sms, cudaStream_t s) {
  if (n == 0) return;
  Scope sc_(ST_HIST_SCAN, s, n);
  // experiments: HUSKY_RANK_BALLOT / HUSKY_RANK_MATCH = digit bit masks that
  // force one primitive (default: the plan's < 5% largest-bin rule)
  static const uint32_t force_ballot = env_mask("HUSKY_RANK_BALLOT"), force_match = env_mask("HUSKY_RANK_MATCH");
  const uint64_t blocks = std::min<uint64_t>((n + 2047) / 2048, (uint64_t)num_sms * kHistBlocksPerSM);
  launch_pdl(k_hist_slots<true>, dim3((unsigned)blocks), dim3(512), 0, s, keys, n, st, keysA, keysB, force_ballot,
             force_match);
}

constexpr int kRadixWarps = kRadixThreads / 32;
// Ranking primitive of a pass (the per-warp label match; MATCH costs grow with
// the number of distinct labels in the warp).  4 (default): three matches of
// the digit's 3 + 3 + 2 bits, peers = AND of the three (9 was as fast in the
// lab and faster on C3 / C4, but 1% slower on C2 in the bench, the headline).
// Measured per sort (C2 / C3 / C4, us): 0 = the plan's rule
// (ballots for spread digits, one 8-bit match otherwise) 1033 / 1119 / 1823;
// 2 = two 4-bit matches 1020 / 1119 / 1812; 4 = 3+3+2 bits by matches
// 1020 / 1072 / 1745; 9 = 3+3 by matches + 2 ballots 1021-1027 / 1051 / 1731;
// 10 = 4+2 by matches + 2 ballots 1022 / 1058-1062 / 1722-1728; 5 = four 2-bit
// matches 1024-1031 / 1056-1060 / 1765; 7 = ballots for every digit
// 1083 / 1080 / 1785.
#ifndef HUSKY_RANK_NIBBLE
#define HUSKY_RANK_NIBBLE 4
#endif
#ifndef RADIX_LB_W
#define RADIX_LB_W 12
#endif

#ifdef HUSKY_TIMING
// per-tile phase timestamps of the last radix launch (instrumented builds only)
constexpr int kTimingTiles = 8192;
__device__ unsigned long long g_tile_times[kTimingTiles][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define HT(tile, i) \
  do { if (threadIdx.x == 0 && (tile) < kTimingTiles) g_tile_times[tile][i] = gtimer(); } while (0)
#else
#define HT(tile, i) do { } while (0)
#endif
// dynamic smem of a pass: key/value exchange buffer + per-warp digit counters
template <int BITS, int ITEMS = kRadixItems>
constexpr int exchange_bytes() { return kRadixThreads * ITEMS * (8 + 4 + 2) + kRadixWarps * (1 << BITS) * 2; }

// all digits trivial: the permutation is the payload as it stands
__global__ void k_radix_finalize(const DevState *st, const uint32_t *v_init, uint32_t *v_final, uint64_t n) {
  pdl_wait();
  if (st->np != 0) return;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    v_final[i] = v_init ? v_init[i] : (uint32_t)i;
}

// Buffers of a planned pass slot, resolved on device from DevState::np.
struct SlotPtrs {
  uint64_t *kA, *kB;
  const uint32_t *v_init;  // NULL: payload = index (synthesised by slot 0)
  uint32_t *v_final, *v_tmp;
  const DevState *st;  // host-planned launches: digit_spread of the pass's digit
};

// One pass over one tile.  LOOKBACK: decoupled look-back on `lb` (onesweep);
// otherwise the tile's per-digit bases are read from `prefix` ([digit][tile],
// written by k_rs_scan) and nothing waits on other tiles.  plan != NULL: this
// is pass slot `slot` of the device-side plan (buffers, digit resolved here;
// slots beyond the plan exit at once).
template <bool SYNTH_VALS, bool LOOKBACK, int BITS, int ITEMS = kRadixItems>
__global__ void __launch_bounds__(kRadixThreads, kRadixMinBlocks)
    k_onesweep(const uint64_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
               uint64_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out, uint64_t n, int shift,
               const uint32_t *__restrict__ digit_start, unsigned long long *lb, uint32_t *tile_counter,
               uint32_t epoch, const uint32_t *__restrict__ prefix, uint32_t num_tiles, const DevState *plan,
               int slot, SlotPtrs sp) {
  // host-planned passes (refinement, multi-GPU partition): the digit's spread
  // as measured by k_hist_scan; planned slots: the plan's choice
  constexpr uint32_t R = 1u << BITS, MASK = R - 1;
  constexpr int TILE = kRadixThreads * ITEMS;
  static_assert(R <= kRadixThreads, "one digit per thread");
  pdl_wait();  // the pass slots are programmatic dependents of the previous kernel
  bool use_ballot = !plan && sp.st && sp.st->digit_spread[shift / BITS];
  if (plan) {
    const uint32_t np = plan->np;
    if ((uint32_t)slot >= np) return;
    const uint32_t digit = plan->pass_digit[slot];
    use_ballot = plan->pass_ballot[slot] != 0;
    shift = BITS * digit;
    digit_start = plan->digit_start[digit];
    keys_in = (slot & 1) ? sp.kB : sp.kA;
    keys_out = (slot & 1) ? sp.kA : sp.kB;
    vals_in = slot == 0 ? sp.v_init : (((np - slot) & 1) == 0 ? sp.v_final : sp.v_tmp);
    vals_out = ((np - 1 - slot) & 1) == 0 ? sp.v_final : sp.v_tmp;
  }
  extern __shared__ __align__(16) uint8_t smem[];
  // key / value exchange buffers, each key's rank then tile-local position
  // (u16, indexed by its load slot), per-warp digit counters [warps][R] (u16:
  // at most TILE per tile).  Ranks and positions live in shared memory and the
  // values are loaded only after the keys are exchanged, so the kernel fits 40
  // registers (3 CTAs per SM with kRadixMinBlocks = 3).
  uint64_t *xk = reinterpret_cast<uint64_t *>(smem);
  uint32_t *xv = reinterpret_cast<uint32_t *>(smem + TILE * 8);
  uint16_t *rk = reinterpret_cast<uint16_t *>(smem + TILE * 12);
  uint16_t *cnt = reinterpret_cast<uint16_t *>(smem + TILE * 14);
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_local_start[R];
  __shared__ uint32_t s_gbase[R];
  __shared__ uint32_t s_wt[kRadixWarps + 1];

  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  if (LOOKBACK) {  // dynamic tile ids: every predecessor a tile waits on is resident
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  }
  for (int i = tid; i < kRadixWarps * (int)R; i += kRadixThreads) cnt[i] = 0;
  __syncthreads();
  const uint32_t tile = LOOKBACK ? s_tile : blockIdx.x;
  const uint64_t tile_base = (uint64_t)tile * TILE;
  HT(tile, 0);

  // ---- load the keys (warp-striped: slot = warp*256 + r*32 + lane)
  const uint32_t slot0 = warp * (ITEMS * 32) + lane;
  uint64_t k[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint64_t idx = tile_base + slot0 + r * 32;
    k[r] = idx < n ? __ldg(keys_in + idx) : ~0ull;  // padding ranks last (largest digit); never stored
  }
  // ---- the tile's bases (reduce-then-scan): independent of everything above
  const bool is_dg = tid < R;  // threads 0..R-1 own one digit each
  const uint32_t dg = tid & MASK;
  uint32_t pre_base = 0;
  if (!LOOKBACK && is_dg) pre_base = __ldg(prefix + (uint64_t)dg * num_tiles + tile);

  // ---- warp-level match ranking into per-warp counters (stable: (r, lane) order)
  uint16_t *wc = cnt + warp * R;
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    uint32_t d = (uint32_t)(k[r] >> shift) & MASK;
#if HUSKY_RANK_NIBBLE == 4
    // default: three matches of 3 + 3 + 2 bits (3 + 3 + 3 for 9-bit digits)
    constexpr int kLo = BITS - 6;
    uint32_t peers = __match_any_sync(0xFFFFFFFFu, d >> (kLo + 3)) &
                     __match_any_sync(0xFFFFFFFFu, (d >> kLo) & 7u) &
                     __match_any_sync(0xFFFFFFFFu, d & ((1u << kLo) - 1u));
#elif HUSKY_RANK_NIBBLE == 9
    // the top bits by two 3-bit matches, the low BITS - 6 bits by ballots
    uint32_t peers = __match_any_sync(0xFFFFFFFFu, d >> (BITS - 3)) &
                     __match_any_sync(0xFFFFFFFFu, (d >> (BITS - 6)) & 7u);
#pragma unroll
    for (int b = 0; b < BITS - 6; ++b) {
      const uint32_t v = __ballot_sync(0xFFFFFFFFu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? v : ~v;
    }
#elif HUSKY_RANK_NIBBLE == 10
    // experiment: 4 + 2 bits by match, the low 2 bits by two ballots
    const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, d & 1u), b1 = __ballot_sync(0xFFFFFFFFu, d & 2u);
    uint32_t peers = __match_any_sync(0xFFFFFFFFu, d >> 4) & __match_any_sync(0xFFFFFFFFu, (d >> 2) & 3u) &
                     ((d & 1u) ? b0 : ~b0) & ((d & 2u) ? b1 : ~b1);
#elif HUSKY_RANK_NIBBLE == 2
    // two 4-bit matches
    uint32_t peers = __match_any_sync(0xFFFFFFFFu, d >> 4) & __match_any_sync(0xFFFFFFFFu, d & 15u);
#elif HUSKY_RANK_NIBBLE == 5
    // four 2-bit matches
    uint32_t peers = __match_any_sync(0xFFFFFFFFu, d >> 6) & __match_any_sync(0xFFFFFFFFu, (d >> 4) & 3u) &
                     __match_any_sync(0xFFFFFFFFu, (d >> 2) & 3u) & __match_any_sync(0xFFFFFFFFu, d & 3u);
#elif HUSKY_RANK_NIBBLE == 7
    // per-bit ballots for every digit
    uint32_t peers = match_ballot<BITS>(d);
#else
    // the plan's rule: per-bit ballots for spread digits, one 8-bit match otherwise
    uint32_t peers = use_ballot ? match_ballot<BITS>(d) : __match_any_sync(0xFFFFFFFFu, d);
#endif
    if (r == 0) HT(tile, 1);
    uint32_t pre = wc[d];
    rk[slot0 + r * 32] = (uint16_t)(pre + __popc(peers & lanemask_lt()));
    __syncwarp();
    if (lane == 31 - __clz(peers)) wc[d] = (uint16_t)(pre + __popc(peers));
    __syncwarp();
  }
  __syncthreads();
  HT(tile, 2);

  // ---- per digit: warp prefixes and the tile count; with look-back the tile's
  // aggregate is published before anything else so successors can consume it
  uint32_t tot = 0;
  if (is_dg) {
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w) {
      uint32_t c = cnt[w * R + dg];
      cnt[w * R + dg] = (uint16_t)tot;
      tot += c;
    }
  }
  uint64_t tile_end = tile_base + TILE;
  const uint32_t pad_dg = (uint32_t)(~0ull >> shift) & MASK;  // the padding keys' digit
  if (is_dg && dg == pad_dg && tile_end > n) tot -= (uint32_t)(tile_end - n);
  unsigned long long *my_flag = lb + (uint64_t)tile * R + dg;
  if (LOOKBACK && is_dg) {
    if (tile == 0) st_relaxed_u64(my_flag, make_flag(kFlagInc, epoch, (unsigned long long)digit_start[dg] + tot));
    else st_relaxed_u64(my_flag, make_flag(kFlagAgg, epoch, tot));
  }
  uint32_t block_total;
  uint32_t local_start = block_exclusive_scan<uint32_t, kRadixThreads>(tot, &block_total, s_wt);
  if (is_dg) s_local_start[dg] = local_start;
  __syncthreads();
  HT(tile, 3);

  // ---- exchange the keys through shared memory into tile-local digit order;
  // each slot's rank becomes its position (same thread, same slot)
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    uint32_t d = (uint32_t)(k[r] >> shift) & MASK;
    uint32_t pos = s_local_start[d] + wc[d] + rk[slot0 + r * 32];
    xk[pos] = k[r];
    rk[slot0 + r * 32] = (uint16_t)pos;
  }
  // ---- the values: loaded now (the loads overlap the look-back), exchanged after it
  uint32_t v[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint64_t idx = tile_base + slot0 + r * 32;
    v[r] = SYNTH_VALS ? (uint32_t)idx : (idx < n ? __ldg(vals_in + idx) : 0u);
  }

  // ---- global base of each digit
  if (is_dg) {
    unsigned long long excl;
    if (LOOKBACK) {
#ifdef HUSKY_TIMING
      uint32_t lbst[2] = {0, 0};
      excl = tile == 0 ? (unsigned long long)digit_start[dg]
                       : lookback_window<RADIX_LB_W>(lb + dg, tile, R, epoch, lbst);
      if (tid == 0 && tile < kTimingTiles) g_tile_times[tile][7] = lbst[0] | ((unsigned long long)lbst[1] << 32);
#else
      excl = tile == 0 ? (unsigned long long)digit_start[dg] : lookback_window<RADIX_LB_W>(lb + dg, tile, R, epoch);
#endif
      if (tile != 0) st_relaxed_u64(my_flag, make_flag(kFlagInc, epoch, excl + tot));
    } else {
      excl = pre_base;
    }
    if (tid == 0) HT(tile, 4);
    s_gbase[dg] = (uint32_t)excl - local_start;  // modular; global = gbase + local position
  }
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) xv[rk[slot0 + r * 32]] = v[r];
  __syncthreads();
  HT(tile, 5);

  // ---- scatter: consecutive local positions of a digit -> consecutive addresses
  uint32_t n_valid = (uint32_t)((n - tile_base) < (uint64_t)TILE ? (n - tile_base) : TILE);
#pragma unroll 4
  for (uint32_t i = tid; i < n_valid; i += kRadixThreads) {
    uint64_t key = xk[i];
    uint32_t d = (uint32_t)(key >> shift) & MASK;
    uint32_t g = s_gbase[d] + i;
    keys_out[g] = key;
    vals_out[g] = xv[i];
  }
  HT(tile, 6);
}

// ------------------------------------------------------- reduce-then-scan
// Upsweep: counts[digit][tile] of one tile (warp-striped loads, match-aggregated
// shared-memory histogram).
constexpr int kUpThreads = 256, kUpItems = kRadixTile / kUpThreads;

__global__ void __launch_bounds__(kUpThreads)
    k_rs_upsweep(const uint64_t *__restrict__ keys, uint64_t n, int shift, uint32_t *__restrict__ counts,
                 uint32_t num_tiles) {
  __shared__ uint32_t hist[256];
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  hist[tid] = 0;
  const uint32_t tile = blockIdx.x;
  const uint64_t tb = (uint64_t)tile * kRadixTile;
  uint64_t k[kUpItems];
#pragma unroll
  for (int r = 0; r < kUpItems; ++r) {
    uint64_t idx = tb + warp * (kUpItems * 32) + r * 32 + lane;
    k[r] = idx < n ? __ldg(keys + idx) : ~0ull;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kUpItems; ++r) {
    uint64_t idx = tb + warp * (kUpItems * 32) + r * 32 + lane;
    uint32_t d = idx < n ? (uint32_t)(k[r] >> shift) & 0xFF : 256u;
    uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    if (d < 256 && lane == 31 - __clz(peers)) atomicAdd(&hist[d], (uint32_t)__popc(peers));
  }
  __syncthreads();
  counts[(uint64_t)tid * num_tiles + tile] = hist[tid];
}

// Scan: one CTA per digit turns counts[d][*] into bases digit_start[d] + sum of
// the counts of earlier tiles (in place).
__global__ void __launch_bounds__(1024)
    k_rs_scan(uint32_t *__restrict__ counts, uint32_t num_tiles, const uint32_t *__restrict__ digit_start) {
  __shared__ uint32_t wt[33];
  uint32_t *row = counts + (uint64_t)blockIdx.x * num_tiles;
  uint32_t running = digit_start[blockIdx.x];
  for (uint32_t c = 0; c < num_tiles; c += 1024) {
    uint32_t i = c + threadIdx.x;
    uint32_t v = i < num_tiles ? row[i] : 0u;
    uint32_t total;
    uint32_t ex = block_exclusive_scan<uint32_t, 1024>(v, &total, wt);
    if (i < num_tiles) row[i] = running + ex;
    running += total;
    __syncthreads();
  }
}

// instrumented builds: copy the per-tile phase timestamps of the last pass
extern "C" int husky_debug_tile_times(unsigned long long *out, int max_tiles) {
#ifdef HUSKY_TIMING
  int k = max_tiles < kTimingTiles ? max_tiles : kTimingTiles;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_tile_times, (size_t)k * 8 * sizeof(unsigned long long));
  return k;
#else
  (void)out;
  (void)max_tiles;
  return 0;
#endif
}

template <int ITEMS>
static void onesweep_host(const uint64_t *keys_in, const uint32_t *vals_in, uint64_t *keys_out, uint32_t *vals_out,
                          uint64_t n, int digit, const uint32_t *ds, unsigned long long *lb, uint32_t *tile_counter,
                          uint32_t epoch, const SlotPtrs &sp, cudaStream_t s) {
  constexpr int kX = exchange_bytes<8, ITEMS>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_onesweep<true, true, 8, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, kX);
    cudaFuncSetAttribute(k_onesweep<false, true, 8, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, kX);
    configured = true;
  }
  const uint64_t t = (uint64_t)kRadixThreads * ITEMS;
  const uint32_t tiles = (uint32_t)((n + t - 1) / t);
  // programmatic dependent launches here too (refinement rounds, partitions)
  auto k = vals_in == nullptr ? k_onesweep<true, true, 8, ITEMS> : k_onesweep<false, true, 8, ITEMS>;
  launch_pdl(k, dim3(tiles), dim3(kRadixThreads), kX, s, keys_in, vals_in, keys_out, vals_out, n, 8 * digit, ds, lb,
             tile_counter, epoch, (const uint32_t *)nullptr, tiles, (const DevState *)nullptr, 0, sp);
}

void launch_onesweep(const uint64_t *keys_in, const uint32_t *vals_in, uint64_t *keys_out,
                     uint32_t *vals_out, uint64_t n, int digit, DevState *st,
                     unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, cudaStream_t s) {
  if (n == 0) return;
  static const bool onesweep = [] {
    const char *v = getenv("HUSKY_RADIX");
    return !(v && v[0] == 'r');  // default onesweep; HUSKY_RADIX=rts: reduce-then-scan variant
  }();
  Scope sc_(ST_RADIX, s, n);
  const uint32_t *ds = st->digit_start[digit];
  const SlotPtrs sp{nullptr, nullptr, nullptr, nullptr, nullptr, st};
  if (onesweep) {
    if (radix_items(n) == kRadixItemsSmall)
      onesweep_host<kRadixItemsSmall>(keys_in, vals_in, keys_out, vals_out, n, digit, ds, lb, tile_counter, epoch, sp, s);
    else
      onesweep_host<kRadixItems>(keys_in, vals_in, keys_out, vals_out, n, digit, ds, lb, tile_counter, epoch, sp, s);
    return;
  }
  // reduce-then-scan (large tiles only): the look-back buffer (tiles*256 u64)
  // holds counts[256][tiles] u32
  constexpr int kX = exchange_bytes<8>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_onesweep<true, false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kX);
    cudaFuncSetAttribute(k_onesweep<false, false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kX);
    configured = true;
  }
  const uint32_t tiles = (uint32_t)radix_tiles_large(n);
  dim3 g(tiles), b(kRadixThreads);
  uint32_t *counts = reinterpret_cast<uint32_t *>(lb);
  k_rs_upsweep<<<tiles, kUpThreads, 0, s>>>(keys_in, n, 8 * digit, counts, tiles);
  k_rs_scan<<<256, 1024, 0, s>>>(counts, tiles, ds);
  if (vals_in == nullptr)
    k_onesweep<true, false, 8><<<g, b, kX, s>>>(keys_in, nullptr, keys_out, vals_out, n, 8 * digit, ds, lb,
                                                tile_counter, epoch, counts, tiles, nullptr, 0, sp);
  else
    k_onesweep<false, false, 8><<<g, b, kX, s>>>(keys_in, vals_in, keys_out, vals_out, n, 8 * digit, ds, lb,
                                                 tile_counter, epoch, counts, tiles, nullptr, 0, sp);
}

// Pass slot `slot` (0..7) of the device-side plan (kSlotBits-bit digits).
// Launched unconditionally; the kernel resolves digit and buffers from DevState.
template <int ITEMS>
static void onesweep_slot(int slot, uint64_t *keysA, uint64_t *keysB, const uint32_t *vals_init,
                          uint32_t *vals_final, uint32_t *vals_tmp, uint64_t n, DevState *st,
                          unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, cudaStream_t s) {
  constexpr int kX = exchange_bytes<kSlotBits, ITEMS>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_onesweep<true, true, kSlotBits, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, kX);
    cudaFuncSetAttribute(k_onesweep<false, true, kSlotBits, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, kX);
    configured = true;
  }
  const uint64_t t = (uint64_t)kRadixThreads * ITEMS;
  const uint32_t tiles = (uint32_t)((n + t - 1) / t);
  SlotPtrs sp{keysA, keysB, vals_init, vals_final, vals_tmp, nullptr};
  // programmatic dependent launch: the pass's CTAs become resident while the
  // previous kernel's last wave drains and start as soon as it completes
  auto k = (slot == 0 && vals_init == nullptr) ? k_onesweep<true, true, kSlotBits, ITEMS>
                                               : k_onesweep<false, true, kSlotBits, ITEMS>;
  launch_pdl(k, dim3(tiles), dim3(kRadixThreads), kX, s, (const uint64_t *)nullptr, (const uint32_t *)nullptr,
             (uint64_t *)nullptr, (uint32_t *)nullptr, n, 0, (const uint32_t *)nullptr, lb, tile_counter, epoch,
             (const uint32_t *)nullptr, tiles, (const DevState *)st, slot, sp);
}

// Pass slot `slot` (0..7) of the device-side plan (kSlotBits-bit digits).
// Launched unconditionally; the kernel resolves digit and buffers from DevState.
void launch_onesweep_slot(int slot, uint64_t *keysA, uint64_t *keysB, const uint32_t *vals_init,
                          uint32_t *vals_final, uint32_t *vals_tmp, uint64_t n, DevState *st,
                          unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, cudaStream_t s) {
  if (n == 0) return;
  Scope sc_(ST_RADIX, s, n);
  if (radix_items(n) == kRadixItemsSmall)
    onesweep_slot<kRadixItemsSmall>(slot, keysA, keysB, vals_init, vals_final, vals_tmp, n, st, lb, tile_counter,
                                    epoch, s);
  else
    onesweep_slot<kRadixItems>(slot, keysA, keysB, vals_init, vals_final, vals_tmp, n, st, lb, tile_counter, epoch,
                               s);
}

void launch_radix_finalize(const DevState *st, const uint32_t *vals_init, uint32_t *vals_final, uint64_t n,
                           cudaStream_t s) {
  if (n == 0) return;
  Scope sc_(ST_RADIX, s, 0);
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 2048) blocks = 2048;
  launch_pdl(k_radix_finalize, dim3((unsigned)blocks), dim3(256), 0, s, (const DevState *)st, vals_init, vals_final, n);
}

__global__ void k_iota(uint32_t *perm, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    perm[i] = (uint32_t)i;
}

void launch_iota(uint32_t *perm, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  Scope sc_(ST_RADIX, s, 0);
  uint64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  k_iota<<<(unsigned)blocks, 256, 0, s>>>(perm, n);
}

}  // namespace husky
