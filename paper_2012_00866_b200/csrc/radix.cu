// radix.cu -- A2: stable LSD radix sort of (64-bit key, 32-bit payload).
//
// Role in the paper: step 2 of Alg. 1, "Sort array longs ... in such a way that
// when elements i, j of longs are exchanged, then elements i, j of xs are also
// exchanged".  Introsort's comparisons are replaced
// by an LSD radix sort whose payload is the string index, so the co-swap is the
// payload scatter.  Being stable, it leaves equal codes in index order
// (R7), which the fix-up (A5) relies on.
//
// Digit width: 8 bits (9-bit digits -- 7 passes for the 63-bit codes -- measured
// no faster).
// A pass works on tiles of kRadixTile = 6144 keys (512 threads x 12, warp-striped so every
// load/store instruction is a coalesced 256-B access).  Each tile is ranked in
// shared memory with warp-level peer masks (one __match_any_sync on the high 3
// bits of the digit, a ballot per low bit) + popc into per-warp digit counters, exchanged
// through shared memory into digit order, and written out as runs of
// consecutive addresses.  The tile's global base per digit comes from a
// per-(tile, digit) decoupled look-back (onesweep, Adinets & Merrill) on top of
// the global digit starts from the 8 digit histograms of the codes
// (k_hist_slots): one read of the keys per pass; the look-back is a chain of
// dependent L2 round trips (~1 us each with the memory system saturated;
// measured per-tile phases in DESIGN.md).  Reduce-then-scan measured slower
// and was removed.
// Digits whose histogram puts all keys in one bucket are skipped.
#include <algorithm>

#include "husky_internal.cuh"
#include "kernels.cuh"

namespace husky {

// Exclusive scan of hist[d][0..255] -> digit_start[d]; trivial_mask bit d when
// one digit value holds all n keys (that pass is the identity and is skipped).
__global__ void __launch_bounds__(kBins) k_hist_scan(uint64_t n, DevState *st) {
  __shared__ uint32_t wt[kBins / 32 + 1];
  const int d = blockIdx.x;
  uint32_t v = st->hist[d][threadIdx.x];
  uint32_t total;
  uint32_t ex = block_exclusive_scan<uint32_t, kBins>(v, &total, wt);
  st->digit_start[d][threadIdx.x] = ex;
  if ((uint64_t)v == n) atomicOr(&st->trivial_mask, 1u << d);
}

void launch_hist_scan(uint64_t n, DevState *st, cudaStream_t s) {
  Scope sc_(ST_HIST_SCAN, s, n);
  k_hist_scan<<<8, kBins, 0, s>>>(n, st);
}

// The 8 digit histograms of the codes for the LSD onesweep (A2): one read of
// the codes, plain shared-memory atomics.  Measured on C2: 35 us as a separate
// pass vs 51 us when fused into the encoder's loop, and 8x slower with
// __match_any_sync aggregation.  PLAN: the last CTA to add its
// histograms (ticket) also does k_hist_scan's scans and the pass plan (which
// digits to sort, in which order), saving two dependent launches.
constexpr int kHistBlocksPerSM = 4;  // resident CTAs of 512 threads per SM
// compress (ASCII, PLAN): alphabet compression first (husky_internal.cuh):
// every key is re-packed in place from DevState::alpha when that needs at most
// 56 bits, and the histograms are those of the re-packed keys.
// skip (PLAN, ASCII codes; R19): 1 = leave the lowest one or two
// varying digits unsorted when the other varying digits carry enough entropy
// that the extra equal-key pairs this creates are rare (the run machinery
// resolves them exactly), 2 / 3 = one / two digits whenever possible (tests),
// 0 = never.  def_s / def_pl: the
// coder's run rule when nothing is skipped.
#ifndef HUSKY_SKIP2_BAR
#define HUSKY_SKIP2_BAR 1e-2f
#endif
constexpr float kSkip2Bar = HUSKY_SKIP2_BAR;
// one pass costs ~7 ps per key at 2^30 (C5), one extra dirty run ~0.8 ns: the
// break-even is ~0.02 n extra pairs per pass saved; the bars stay below it
// because the estimate assumes independent digits
#ifndef HUSKY_SKIP1_BAR
#define HUSKY_SKIP1_BAR 5e-3f
#endif
constexpr float kSkip1Bar = HUSKY_SKIP1_BAR;
template <bool PLAN>
__global__ void __launch_bounds__(512) k_hist_slots(uint64_t *__restrict__ keys, uint64_t n, DevState *st,
                                                    uint64_t *keysA, uint64_t *keysB, int compress, int skip,
                                                    uint32_t def_s, uint32_t def_pl, int uni) {
  constexpr uint32_t M = kBins - 1;
  pdl_wait();  // PLAN: launched as a programmatic dependent of the encoder
  __shared__ uint32_t h[8 * kBins];
  __shared__ uint32_t s_last, s_wt[512 / 32 + 1];
  __shared__ uint8_t s_rank[128];
  for (int i = threadIdx.x; i < 8 * kBins; i += blockDim.x) h[i] = 0;
  uint32_t cbits = 7;
  if (compress) {
    const uint32_t a[4] = {st->alpha[0], st->alpha[1], st->alpha[2], st->alpha[3]};
    cbits = alpha_bits(a);
    if (threadIdx.x < 128) s_rank[threadIdx.x] = (uint8_t)alpha_rank(a, threadIdx.x);
  }
  const bool cmp = cbits <= 6;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * 4; base < n; base += stride) {
    uint64_t k[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint64_t i = base + threadIdx.x + (uint64_t)r * blockDim.x;
      k[r] = i < n ? keys[i] : 0;
    }
    if (cmp) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint64_t i = base + threadIdx.x + (uint64_t)r * blockDim.x;
        uint64_t c = 0;
#pragma unroll
        for (int f = 0; f < 9; ++f) c |= (uint64_t)s_rank[(uint32_t)(k[r] >> (7 * (8 - f))) & 0x7Fu] << (cbits * (8 - f));
        k[r] = c;
        if (i < n) keys[i] = c;
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (base + threadIdx.x + (uint64_t)r * blockDim.x >= n) continue;
#pragma unroll
      for (int d = 0; d < 8; ++d) atomicAdd(&h[d * kBins + ((uint32_t)(k[r] >> (kDigitBits * d)) & M)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * kBins; i += blockDim.x)
    if (h[i]) atomicAdd(&st->hist[i / kBins][i % kBins], h[i]);
  if (!PLAN) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&st->hist_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // the last CTA: exclusive scans and trivial digits (as k_hist_scan), the
  // entropy of each digit's histogram, then the plan.  One warp per digit
  // (8 bins per lane, shuffle scans): all 8 digits' counts in one round trip
  // and no block barriers (a digit-serial block scan cost ~12 us of a 1e5 sort)
  __shared__ float s_h[8];
  __shared__ uint32_t s_triv[8];
  {
    const uint32_t w = threadIdx.x >> 5, lane = lane_id();
    if (w < 8) {
      uint32_t v[8], t = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[q] = __ldcg(&st->hist[w][lane * 8 + q]);
        t += v[q];
      }
      uint32_t incl = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((int)lane >= o) incl += y;
      }
      uint32_t run = incl - t;
      bool all_here = false;
      float hsum = 0.f;  // H_d = -sum p log2 p over the digit's bins
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        st->digit_start[w][lane * 8 + q] = run;
        run += v[q];
        all_here |= (uint64_t)v[q] == n;
        const float pr = (float)v[q] / (float)n;
        hsum += v[q] ? -pr * __log2f(pr) : 0.f;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) hsum += __shfl_xor_sync(0xFFFFFFFFu, hsum, o);
      const bool triv = __any_sync(0xFFFFFFFFu, all_here);
      if (lane == 0) {
        s_h[w] = hsum;
        s_triv[w] = triv ? 1u : 0u;
      }
    }
  }
  __syncthreads();
  uint32_t trivial = 0;
#pragma unroll
  for (int d = 0; d < 8; ++d) trivial |= s_triv[d] << d;
  if (threadIdx.x == 0) {
    st->trivial_mask = trivial;
    st->ccomp = cmp ? 1u : 0u;
    st->cbits = cbits;
    uint32_t np = 0, dig[8];
    for (int d = 0; d < 8; ++d)
      if (!((trivial >> d) & 1)) dig[np++] = d;
    uint32_t seq = def_s, pl = def_pl;
    unsigned long long mask = ~0ull;
    if (skip && np >= 2) {
      // leave the k lowest varying digits unsorted (k = 2 then 1): equal keys
      // above them fix the fields that lie wholly above bit 8 (dig[k-1] + 1)
      const uint32_t fb = cmp ? cbits : 7u;
      for (uint32_t k = 2; k >= 1; --k) {
        if (np < k + 1 || (skip == 2 && k != 1) || (skip == 3 && k != 2)) continue;
        const uint32_t dtop = dig[k - 1];
        // units wholly above the masked bits [0, 8 (dtop + 1)): ASCII fields of
        // fb bits from bit fb * 8 down; UNICODE units 0..2 at bits 47 - 16 u ..
        // 62 - 16 u (unit 3 lost its low bit to the >>> 1 and is never fixed)
        int sp = 9 - (int)((8 * (dtop + 1) + fb - 1) / fb);
        if (uni) {
          sp = 0;
          for (int u = 0; u < 3; ++u) sp += (47 - 16 * u >= (int)(8 * (dtop + 1))) ? 1 : 0;
        }
        float hhi = 0.f;
        for (uint32_t i = k; i < np; ++i) hhi += s_h[dig[i]];
        // expected extra equal-key pairs if the other digits were independent;
        // one more pass costs ~24 B per key, one extra pair a check and at
        // worst a two-string fix-up, so the bar is a small fraction of n
        const float extra = 0.5f * (float)n * (float)n * exp2f(-hhi);
        const float bar = (k == 1 ? kSkip1Bar : kSkip2Bar) * (float)n;
        if (sp >= 1 && (skip >= 2 || extra < bar)) {
          for (uint32_t i = 0; i + k < np; ++i) dig[i] = dig[i + k];
          np -= k;
          seq = (uint32_t)sp;
          pl = (uint32_t)sp;
          mask = ~((1ull << (8 * (dtop + 1))) - 1ull);
          break;
        }
      }
    }
    for (uint32_t i = 0; i < np; ++i) st->pass_digit[i] = dig[i];
    st->seq_units = seq;
    st->short_len = pl;
    st->key_mask = mask;
    st->np = np;
    st->sorted_keys = (unsigned long long)((np & 1) ? keysB : keysA);
  }
}

void launch_hist_slots(const uint64_t *keys, uint64_t n, DevState *st, int num_sms, cudaStream_t s) {
  if (n == 0) return;
  Scope sc_(ST_HIST_SCAN, s, n);
  const uint64_t blocks = std::min<uint64_t>((n + 2047) / 2048, (uint64_t)num_sms * kHistBlocksPerSM);
  k_hist_slots<false><<<(unsigned)blocks, 512, 0, s>>>(const_cast<uint64_t *>(keys), n, st, nullptr, nullptr, 0, 0,
                                                      0u, 0u, 0);
}

// histograms + scans + pass plan of the device-planned passes in one launch
// (DevState::hist_done must be 0: DevState is zeroed per sort)
void launch_hist_plan(const uint64_t *keys, uint64_t n, DevState *st, uint64_t *keysA, uint64_t *keysB,
                      int num_sms, cudaStream_t s, bool compress, int skip, uint32_t def_s, uint32_t def_pl,
                      bool unicode) {
  if (n == 0) return;
  Scope sc_(ST_HIST_SCAN, s, n);
  GroupScope grp(ST_HIST_SCAN, s);
  const uint64_t blocks = std::min<uint64_t>((n + 2047) / 2048, (uint64_t)num_sms * kHistBlocksPerSM);
  launch_pdl(k_hist_slots<true>, dim3((unsigned)blocks), dim3(512), 0, s, const_cast<uint64_t *>(keys), n, st, keysA,
             keysB, compress ? 1 : 0, skip, def_s, def_pl, unicode ? 1 : 0);
}

constexpr int kRadixWarps = kRadixThreads / 32;
// ranking: ballots on the low kRankBallots bits of the digit, one label match
// on the rest
#ifndef HUSKY_RANK_BALLOTS
#define HUSKY_RANK_BALLOTS 5
#endif
constexpr int kRankBallots = HUSKY_RANK_BALLOTS;

// Look-back window: predecessors read per round trip (with the ballot
// ranking, C5 radix per sort: 6 / 8 / 10 / 12 / 16 -> 38.16 / 38.22 / 38.75 /
// 38.43 / 43.2 ms; C2 flat)
#ifndef RADIX_LB_W
#define RADIX_LB_W 6
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
template <int ITEMS>
constexpr int exchange_bytes() { return kRadixThreads * ITEMS * (8 + 4 + 2) + kRadixWarps * kBins * 2; }

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
};

// One pass over one tile, decoupled look-back on `lb`.  SYNTH: payload =
// index (no payload read; the first pass).  plan != NULL: this is pass slot
// `slot` of the device-side plan (buffers, digit resolved here; slots beyond
// the plan exit at once).  Two instantiations per tile size (SYNTH or not).
template <bool SYNTH, int ITEMS>
__global__ void __launch_bounds__(kRadixThreads, 2)
    k_onesweep(const uint64_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
               uint64_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out, uint64_t n, int shift,
               const uint32_t *__restrict__ digit_start, unsigned long long *lb, uint32_t *tile_counter,
               uint32_t epoch, const DevState *plan, int slot, SlotPtrs sp) {
  constexpr uint32_t R = kBins, MASK = R - 1;
  constexpr int TILE = kRadixThreads * ITEMS;
  static_assert(R <= kRadixThreads, "one digit per thread");
  pdl_wait();  // the pass slots are programmatic dependents of the previous kernel
  if (plan) {
    const uint32_t np = plan->np;
    if ((uint32_t)slot >= np) return;
    const uint32_t digit = plan->pass_digit[slot];
    shift = kDigitBits * digit;
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
  // values are loaded only after the keys are exchanged, so the kernel fits 64
  // registers at 2 CTAs per SM.
  uint64_t *xk = reinterpret_cast<uint64_t *>(smem);
  uint32_t *xv = reinterpret_cast<uint32_t *>(smem + TILE * 8);
  uint16_t *rk = reinterpret_cast<uint16_t *>(smem + TILE * 12);
  uint16_t *cnt = reinterpret_cast<uint16_t *>(smem + TILE * 14);
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_local_start[R];
  __shared__ uint32_t s_gbase[R];
  __shared__ uint32_t s_wt[kRadixWarps + 1];

  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  // dynamic tile ids: every predecessor a tile waits on is resident
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = tid; i < kRadixWarps * (int)R; i += kRadixThreads) cnt[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t tile_base = (uint64_t)tile * TILE;
  HT(tile, 0);

  // ---- load the keys (warp-striped: slot = warp*ITEMS*32 + r*32 + lane)
  const uint32_t slot0 = warp * (ITEMS * 32) + lane;
  uint64_t k[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const uint64_t idx = tile_base + slot0 + r * 32;
    k[r] = idx < n ? __ldg(keys_in + idx) : ~0ull;  // padding ranks last (largest digit); never stored
  }
  const bool is_dg = tid < R;  // threads 0..R-1 own one digit each
  const uint32_t dg = tid & MASK;

  // ---- warp-level ranking into per-warp counters (stable: (r, lane) order)
  uint16_t *wc = cnt + warp * R;
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    uint32_t d = (uint32_t)(k[r] >> shift) & MASK;
    // lanes with the same digit: one label match on the high bits, a ballot
    // per low bit (a match costs more the more distinct labels a warp holds, a
    // ballot one vote; measured, C5 / C2 radix per sort: 3 + 3 + 2-bit matches
    // 40.3 / 0.430 ms, match + 4 ballots 38.8 / 0.423, + 5 ballots 38.4 /
    // 0.436, + 6 39.2 / 0.451, 8 ballots 40.5 / 0.473; a per-digit choice made
    // at run time cost more than it saved)
    uint32_t peers = __match_any_sync(0xFFFFFFFFu, d >> kRankBallots);
#pragma unroll
    for (int b = 0; b < kRankBallots; ++b) {
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bal : ~bal;
    }
    if (r == 0) HT(tile, 1);
    uint32_t pre = wc[d];
    rk[slot0 + r * 32] = (uint16_t)(pre + __popc(peers & lanemask_lt()));
    __syncwarp();
    if (lane == 31 - __clz(peers)) wc[d] = (uint16_t)(pre + __popc(peers));
    __syncwarp();
  }
  __syncthreads();
  HT(tile, 2);

  // ---- per digit: warp prefixes and the tile count; the tile's aggregate is
  // published before anything else so successors can consume it
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
  if (is_dg) {
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
    v[r] = SYNTH ? (uint32_t)idx : (idx < n ? __ldg(vals_in + idx) : 0u);
  }

  // ---- global base of each digit
  if (is_dg) {
    unsigned long long excl;
#ifdef HUSKY_TIMING
    uint32_t lbst[2] = {0, 0};
    excl = tile == 0 ? (unsigned long long)digit_start[dg]
                     : lookback_window<RADIX_LB_W>(lb + dg, tile, R, epoch, lbst);
    if (tid == 0 && tile < kTimingTiles) g_tile_times[tile][7] = lbst[0] | ((unsigned long long)lbst[1] << 32);
#else
    excl = tile == 0 ? (unsigned long long)digit_start[dg] : lookback_window<RADIX_LB_W>(lb + dg, tile, R, epoch);
#endif
    if (tile != 0) st_relaxed_u64(my_flag, make_flag(kFlagInc, epoch, excl + tot));
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
    HCHK(kChkRadixScatter, g, n);
    keys_out[g] = key;
    vals_out[g] = xv[i];
  }
  HT(tile, 6);
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
static void onesweep_launch(const uint64_t *keys_in, const uint32_t *vals_in, uint64_t *keys_out,
                            uint32_t *vals_out, uint64_t n, int digit, const uint32_t *ds, unsigned long long *lb,
                            uint32_t *tile_counter, uint32_t epoch, const DevState *plan, int slot,
                            const SlotPtrs &sp, cudaStream_t s) {
  constexpr int kX = exchange_bytes<ITEMS>();
  static SmemAttr attr_s, attr_v;
  attr_s.ensure(k_onesweep<true, ITEMS>, kX);
  attr_v.ensure(k_onesweep<false, ITEMS>, kX);
  const uint64_t t = (uint64_t)kRadixThreads * ITEMS;
  const uint32_t tiles = (uint32_t)((n + t - 1) / t);
  // the first planned slot synthesises the index when there is no initial payload
  const bool synth = plan ? (slot == 0 && sp.v_init == nullptr) : vals_in == nullptr;
  // programmatic dependent launch: the pass's CTAs become resident while the
  // previous kernel's last wave drains and start as soon as it completes
  launch_pdl(synth ? k_onesweep<true, ITEMS> : k_onesweep<false, ITEMS>, dim3(tiles), dim3(kRadixThreads), kX, s,
             keys_in, vals_in, keys_out, vals_out, n, kDigitBits * digit, ds, lb, tile_counter, epoch, plan, slot, sp);
}

void launch_onesweep(const uint64_t *keys_in, const uint32_t *vals_in, uint64_t *keys_out,
                     uint32_t *vals_out, uint64_t n, int digit, DevState *st,
                     unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, cudaStream_t s) {
  if (n == 0) return;
  Scope sc_(ST_RADIX, s, n);
  const uint32_t *ds = st->digit_start[digit];
  const SlotPtrs sp{nullptr, nullptr, nullptr, nullptr, nullptr};
  if (radix_items(n) == kRadixItemsSmall)
    onesweep_launch<kRadixItemsSmall>(keys_in, vals_in, keys_out, vals_out, n, digit, ds, lb, tile_counter, epoch,
                                      nullptr, 0, sp, s);
  else
    onesweep_launch<kRadixItems>(keys_in, vals_in, keys_out, vals_out, n, digit, ds, lb, tile_counter, epoch,
                                 nullptr, 0, sp, s);
}

// Pass slot `slot` (0..7) of the device-side plan.  Launched unconditionally;
// the kernel resolves digit and buffers from DevState.
void launch_onesweep_slot(int slot, uint64_t *keysA, uint64_t *keysB, const uint32_t *vals_init,
                          uint32_t *vals_final, uint32_t *vals_tmp, uint64_t n, DevState *st,
                          unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, cudaStream_t s) {
  if (n == 0) return;
  Scope sc_(ST_RADIX, s, n);
  SlotPtrs sp{keysA, keysB, vals_init, vals_final, vals_tmp};
  if (radix_items(n) == kRadixItemsSmall)
    onesweep_launch<kRadixItemsSmall>(nullptr, nullptr, nullptr, nullptr, n, 0, nullptr, lb, tile_counter, epoch, st,
                                      slot, sp, s);
  else
    onesweep_launch<kRadixItems>(nullptr, nullptr, nullptr, nullptr, n, 0, nullptr, lb, tile_counter, epoch, st,
                                 slot, sp, s);
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
