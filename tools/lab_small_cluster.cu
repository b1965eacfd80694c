// LAB EXPERIMENT, NOT BUILT (measured slower): the whole sort of n <= 131072 strings in
// one launch of a 16-CTA thread-block cluster with DSMEM digit-count exchange.  Kept for reference.
// small.cu -- the whole hot path of a small input in ONE kernel launch: one
// thread-block cluster of 16 CTAs (distributed shared memory), no look-back.
//
// A sort of n <= 131072 strings moves ~3 MB: at HBM speed that is ~1 us, so
// the ~14 dependent launches of the regular path (encoder, histograms, pass
// slots, gather, classification, fix-ups) and each pass's decoupled look-back
// are what it costs (C1: 0.12 ms).  Here CTA c of the cluster owns positions
// [8192 c, 8192 (c + 1)) and the method's steps run back to back:
//   A1  encode its strings (Alg. 4, coders.cuh) straight
//       into registers; the cluster agrees on the alphabet of the code fields
//       (alphabet compression, R17), on the digits that vary (the
//       pass plan) and on input violations through distributed shared memory;
//   A2  per LSD pass: warp label-matching rank of its keys (as k_onesweep),
//       its 256 digit counts published in shared memory, every CTA reads the
//       16 CTAs' counts through DSMEM (the exclusive prefix over CTAs replaces
//       the look-back), exchange in smem, scatter to an L2-resident global
//       buffer, cluster barrier, reload;
//   A3  equal adjacent codes: exact order check (cmp_equal_code), run
//       statistics by a cluster-wide segmented max-scan;
//   A4  sorted offsets (scan of the lengths over the cluster) and the units.
// A dirty run (an equal-code pair out of order) or input the coder cannot
// order (bad offsets, off-domain units) sets DevState::small_status and the
// host runs the regular path instead (refinement, fix-ups, general cleanup).
#include <cooperative_groups.h>

#include "coders.cuh"
#include "husky_internal.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace husky {

constexpr int kSmallCL = 16;                          // CTAs per cluster (non-portable size)
constexpr int kSmallThreads = 1024, kSmallItems = 8;  // 8192 strings per CTA
constexpr int kSmallChunk = kSmallThreads * kSmallItems;
constexpr int kSmallWarps = kSmallThreads / 32;
static_assert((uint64_t)kSmallCL * kSmallChunk == kSmallMaxN, "kSmallMaxN");
// dynamic smem: keys u64 + payload u32 + rank u16 per string, per-warp u16 digit counters
constexpr int kSmallSmem = kSmallChunk * (8 + 4 + 2) + kSmallWarps * kBins * 2;

#ifdef HUSKY_SMALL_TIMING
// lab builds: %globaltimer of CTA 0 at each phase (start, encode, cluster agreement,
// passes, runs, gather)
__device__ unsigned long long g_small_t[64];
#define STIME(i) do { if (c == 0 && threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_small_t[i] = t_; } } while (0)
#else
#define STIME(i) do { } while (0)
#endif

template <int CODER>
__global__ void __launch_bounds__(kSmallThreads, 1)
    k_small(const void *__restrict__ units, const int64_t *__restrict__ offsets, uint64_t n, uint64_t *kA,
            uint64_t *kB, uint32_t *vA, uint32_t *vB, uint32_t *perm, void *sorted_units, int64_t *sorted_offsets,
            DevState *st) {
  using T = CoderTraits<CODER>;
  constexpr int W = T::kUnitBytes;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t *xk = reinterpret_cast<uint64_t *>(smem);
  uint32_t *xv = reinterpret_cast<uint32_t *>(smem + kSmallChunk * 8);
  uint16_t *rk = reinterpret_cast<uint16_t *>(smem + kSmallChunk * 12);
  uint16_t *cnt = reinterpret_cast<uint16_t *>(smem + kSmallChunk * 14);
  __shared__ uint32_t s_cnt[kBins];         // this CTA's digit counts (read by the cluster)
  __shared__ uint32_t s_local_start[kBins], s_gbase[kBins];
  __shared__ uint32_t s_wt[kSmallWarps + 1];
  __shared__ unsigned long long s_wt64[kSmallWarps + 1];
  __shared__ uint8_t s_pres[128];
  __shared__ uint32_t s_red[8];             // violations, alphabet words [1..4], ...
  __shared__ unsigned long long s_kor, s_kand, s_tot64, s_maxstart;
  __shared__ uint8_t s_rank[128];
  __shared__ uint32_t s_plan[9];            // np, digits

  const uint32_t c = cluster.block_rank();
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const uint64_t base_c = (uint64_t)c * kSmallChunk;
  const uint32_t nvalid = n > base_c ? (uint32_t)((n - base_c) < (uint64_t)kSmallChunk ? (n - base_c) : kSmallChunk) : 0u;
  const uint32_t slot0 = warp * (kSmallItems * 32) + lane;

  STIME(0);
  if (tid < 128) s_pres[tid] = 0;
  if (tid < 8) s_red[tid] = 0;
  if (tid == 0) { s_kor = 0; s_kand = ~0ull; }
  __syncthreads();

  // ---------------------------------------------------------------- A1 encode
  const uintptr_t ub = (uintptr_t)units;
  const int64_t ofirst = __ldg(offsets), olast = __ldg(offsets + n);
  const bool any_units = olast > ofirst;
  const uintptr_t lo_word = (ub + (uintptr_t)(ofirst * W)) & ~(uintptr_t)7;
  const uintptr_t hi_word = any_units ? ((ub + (uintptr_t)(olast * W) - 1) & ~(uintptr_t)7) : lo_word;
  uint32_t viol = 0;
  uint64_t k[kSmallItems];
  uint32_t v[kSmallItems];
#pragma unroll
  for (int r = 0; r < kSmallItems; ++r) {
    const uint32_t sl = slot0 + r * 32;
    const uint64_t i = base_c + sl;
    k[r] = 0;
    v[r] = (uint32_t)i;
    if (sl < nvalid) {
      const int64_t o0 = __ldg(offsets + i), o1 = __ldg(offsets + i + 1);
      uint64_t w0 = 0, w1 = 0, w2 = 0;
      const uintptr_t a = ub + (uintptr_t)(o0 * W);
      const int sh = (int)(a & 7);
      if (any_units) {
        uintptr_t aw = a & ~(uintptr_t)7;
        aw = aw < lo_word ? lo_word : (aw > hi_word ? hi_word : aw);
        const uintptr_t aw1 = aw + 8 > hi_word ? hi_word : aw + 8;
        const uintptr_t aw2 = aw1 + 8 > hi_word ? hi_word : aw1 + 8;
        w0 = __ldg((const uint64_t *)aw);
        w1 = __ldg((const uint64_t *)aw1);
        if (CODER == HUSKY_CODER_ENGLISH5 || CODER == HUSKY_CODER_ENGLISH6) w2 = __ldg((const uint64_t *)aw2);
      }
      k[r] = encode_words<CODER>(w0, w1, w2, sh, o1 - o0, viol);
      if (CODER == HUSKY_CODER_ASCII) {
#pragma unroll
        for (int f = 0; f < 9; ++f) s_pres[(uint32_t)(k[r] >> (7 * (8 - f))) & 0x7Fu] = 1;
      }
    }
  }
  viol = __reduce_or_sync(0xFFFFFFFFu, viol);
  if (lane == 0 && viol) atomicOr(&s_red[0], viol);
  __syncthreads();
  STIME(1);
  if (CODER == HUSKY_CODER_ASCII && tid < 128) {
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, s_pres[tid] != 0);
    if (lane == 0) s_red[1 + (tid >> 5)] = m;
  }
  cluster.sync();  // every CTA's violations and alphabet words are published
  uint32_t allv = 0, a4[4] = {0, 0, 0, 0};
  for (uint32_t q = 0; q < kSmallCL; ++q) {
    const uint32_t *r = cluster.map_shared_rank(s_red, q);
    allv |= r[0];
    a4[0] |= r[1];
    a4[1] |= r[2];
    a4[2] |= r[3];
    a4[3] |= r[4];
  }
  cluster.sync();  // no CTA leaves (or rewrites s_red) while another still reads it
  // input the coder cannot order exactly here: the regular path takes over
  // (host_common.h domain_violation, restated for the device)
  const bool off_domain = (CODER == HUSKY_CODER_ASCII || CODER == HUSKY_CODER_ENGLISH6) ? (allv & kDomainBad) != 0
                          : CODER == HUSKY_CODER_ENGLISH5 ? ((allv & kNotLower) && (allv & kNotUpper))
                                                          : false;
  if ((allv & kOffsetsBad) || off_domain) {
    if (c == 0 && tid == 0) { st->small_status = 2; st->violations |= allv; }
    return;
  }
  uint32_t cbits = 7;
  bool cmp = false;
  if (CODER == HUSKY_CODER_ASCII) {
    cbits = alpha_bits(a4);
    cmp = cbits <= 6;
    if (tid < 128) s_rank[tid] = (uint8_t)alpha_rank(a4, tid);
  }
  __syncthreads();
  unsigned long long kor = 0, kand = ~0ull;
#pragma unroll
  for (int r = 0; r < kSmallItems; ++r) {
    if (slot0 + r * 32 >= nvalid) continue;
    if (cmp) {
      uint64_t x = 0;
#pragma unroll
      for (int f = 0; f < 9; ++f) x |= (uint64_t)s_rank[(uint32_t)(k[r] >> (7 * (8 - f))) & 0x7Fu] << (cbits * (8 - f));
      k[r] = x;
    }
    kor |= k[r];
    kand &= k[r];
  }
  kor = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)kor) | ((unsigned long long)__reduce_or_sync(0xFFFFFFFFu, (uint32_t)(kor >> 32)) << 32);
  kand = __reduce_and_sync(0xFFFFFFFFu, (uint32_t)kand) |
         ((unsigned long long)__reduce_and_sync(0xFFFFFFFFu, (uint32_t)(kand >> 32)) << 32);
  if (lane == 0) {
    atomicOr(&s_kor, kor);
    atomicAnd(&s_kand, kand);
  }
  cluster.sync();  // every CTA's key OR / AND
  if (tid == 0) {
    unsigned long long o = 0, a = ~0ull;
    for (uint32_t q = 0; q < kSmallCL; ++q) {
      o |= *cluster.map_shared_rank(&s_kor, q);
      a &= *cluster.map_shared_rank(&s_kand, q);
    }
    const unsigned long long vary = o ^ a;  // bits some keys differ in
    uint32_t np = 0, trivial = 0;
    for (int d = 0; d < 8; ++d) {
      if ((vary >> (8 * d)) & 0xFFull) s_plan[1 + np++] = d;
      else trivial |= 1u << d;
    }
    s_plan[0] = np;
    if (c == 0) {
      st->violations |= allv;
      st->np = np;
      st->trivial_mask = trivial;
      st->ccomp = cmp ? 1u : 0u;
      st->cbits = cbits;
      for (int q = 0; q < 4; ++q) st->alpha[q] = a4[q];
    }
  }
  __syncthreads();
  const uint32_t np = s_plan[0];
  STIME(2);
#pragma unroll
  for (int r = 0; r < kSmallItems; ++r)
    if (slot0 + r * 32 >= nvalid) k[r] = ~0ull;  // padding ranks last (digit 255), never stored

  // ---------------------------------------------------------------- A2 passes
  uint64_t *kin = kA, *kout = kB;
  uint32_t *vin = vA, *vout = vB;
  const uint32_t npad = kSmallChunk - nvalid;
  for (uint32_t p = 0; p < np; ++p) {
    const int shift = 8 * (int)s_plan[1 + p];
    for (int i = tid; i < kSmallWarps * kBins; i += kSmallThreads) cnt[i] = 0;
    __syncthreads();
    uint16_t *wc = cnt + warp * kBins;
#pragma unroll
    for (int r = 0; r < kSmallItems; ++r) {
      const uint32_t d = (uint32_t)(k[r] >> shift) & 0xFFu;
      const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d >> 5) & __match_any_sync(0xFFFFFFFFu, (d >> 2) & 7u) &
                             __match_any_sync(0xFFFFFFFFu, d & 3u);
      const uint32_t pre = wc[d];
      rk[slot0 + r * 32] = (uint16_t)(pre + __popc(peers & lanemask_lt()));
      __syncwarp();
      if (lane == 31 - __clz(peers)) wc[d] = (uint16_t)(pre + __popc(peers));
      __syncwarp();
    }
    __syncthreads();
    const bool is_dg = tid < kBins;
    const uint32_t dg = tid & (kBins - 1);
    uint32_t tot = 0;
    if (is_dg) {
      for (int w = 0; w < kSmallWarps; ++w) {
        const uint32_t x = cnt[w * kBins + dg];
        cnt[w * kBins + dg] = (uint16_t)tot;
        tot += x;
      }
      if (dg == 255) tot -= npad;  // padding keys
      s_cnt[dg] = tot;
    }
    uint32_t block_total;
    const uint32_t local_start = block_exclusive_scan<uint32_t, kSmallThreads>(is_dg ? tot : 0u, &block_total, s_wt);
    if (is_dg) s_local_start[dg] = local_start;
    cluster.sync();  // every CTA's digit counts are published
    uint32_t total = 0, before = 0;
    if (is_dg) {
      for (uint32_t q = 0; q < kSmallCL; ++q) {
        const uint32_t x = cluster.map_shared_rank(s_cnt, q)[dg];
        total += x;
        before += q < c ? x : 0u;
      }
    }
    uint32_t all;
    const uint32_t gstart = block_exclusive_scan<uint32_t, kSmallThreads>(is_dg ? total : 0u, &all, s_wt);
    if (is_dg) s_gbase[dg] = gstart + before - s_local_start[dg];  // modular; global = gbase + local position
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSmallItems; ++r) {
      const uint32_t d = (uint32_t)(k[r] >> shift) & 0xFFu;
      const uint32_t pos = s_local_start[d] + wc[d] + rk[slot0 + r * 32];
      xk[pos] = k[r];
      xv[pos] = v[r];
    }
    __syncthreads();
    for (uint32_t i = tid; i < nvalid; i += kSmallThreads) {
      const uint64_t key = xk[i];
      const uint32_t g = s_gbase[(uint32_t)(key >> shift) & 0xFFu] + i;
      kout[g] = key;
      vout[g] = xv[i];
    }
    cluster.sync();  // the pass is complete: every CTA reloads its positions
#pragma unroll
    for (int r = 0; r < kSmallItems; ++r) {
      const uint32_t sl = slot0 + r * 32;
      k[r] = sl < nvalid ? __ldcg(kout + base_c + sl) : ~0ull;
      v[r] = sl < nvalid ? __ldcg(vout + base_c + sl) : 0u;
    }
    STIME(3 + p);
    uint64_t *tk = kin; kin = kout; kout = tk;
    uint32_t *tv = vin; vin = vout; vout = tv;
  }

  // ------------------------------------------------- A3 runs + A4 gather
  // the chunk in position order: keys in xk, payload (original index) in xv
#pragma unroll
  for (int r = 0; r < kSmallItems; ++r) {
    xk[slot0 + r * 32] = k[r];
    xv[slot0 + r * 32] = v[r];
  }
  cluster.sync();  // every chunk is in place (the next chunk's first key is read below)
  const uint64_t next_key = (c + 1 < kSmallCL && nvalid == (uint32_t)kSmallChunk && base_c + kSmallChunk < n)
                                ? cluster.map_shared_rank(xk, c + 1)[0] : ~0ull;
  // blocked: thread t owns positions 8t .. 8t + 7 of the chunk
  const uint32_t b0 = tid * kSmallItems;
  uint32_t eq = 0;  // bit j: position b0 + j equals its successor
  uint32_t bad = 0, len[kSmallItems];
  unsigned long long lsum = 0;
  for (int j = 0; j < kSmallItems; ++j) {
    const uint32_t q = b0 + j;
    len[j] = 0;
    if (q >= nvalid) continue;
    const uint32_t idx = xv[q];
    len[j] = (uint32_t)(__ldg(offsets + idx + 1) - __ldg(offsets + idx));
    lsum += len[j];
    const uint64_t nk = q + 1 < nvalid ? xk[q + 1] : next_key;
    if (nk == xk[q]) {
      eq |= 1u << j;
      const uint32_t idx2 = q + 1 < nvalid ? xv[q + 1] : cluster.map_shared_rank(xv, c + 1)[0];
      // the comparator of the regular path: the byte coders share the ASCII
      // instantiation (S = PL = 9, conservative for the English coders)
      constexpr int KC = CODER == HUSKY_CODER_UNICODE ? HUSKY_CODER_UNICODE : HUSKY_CODER_ASCII;
      if (cmp_equal_code<KC>(units, offsets, idx, idx2, CoderTraits<KC>::kS) > 0) bad = 1;
    }
  }
  // run starts: position p starts a run (of any length) unless it equals its
  // predecessor; the predecessor of b0 is the previous thread's last position
  __shared__ uint32_t s_eq_last[kSmallThreads];
  s_eq_last[tid] = (eq >> (kSmallItems - 1)) & 1u;
  __syncthreads();
  uint32_t prev_of_first = 0;  // does position b0 equal b0 - 1?
  if (tid > 0) prev_of_first = s_eq_last[tid - 1];
  else if (c > 0 && n > base_c) {
    // the previous CTA's last position equals our first?
    const uint64_t *pk = cluster.map_shared_rank(xk, c - 1);
    prev_of_first = pk[kSmallChunk - 1] == xk[0];
  }
  unsigned long long my_start = 0;  // max start position (global) among my positions
  uint32_t in_runs = 0, runs = 0;
  for (int j = 0; j < kSmallItems; ++j) {
    const uint32_t q = b0 + j;
    if (q >= nvalid) break;
    const bool ep = j == 0 ? prev_of_first : ((eq >> (j - 1)) & 1u);
    const bool en = (eq >> j) & 1u;
    if (!ep) my_start = base_c + q;
    in_runs += (ep || en);
    runs += (!ep && en);
  }
  // segmented max-scan of run starts over the cluster -> start of each position's run
  // max-scan (exclusive) of my_start over threads
  {
    unsigned long long x = my_start;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= (uint32_t)o) x = y > x ? y : x;
    }
    if (lane == 31) s_wt64[warp] = x;
    __syncthreads();
    if (warp == 0) {
      unsigned long long wv = lane < kSmallWarps ? s_wt64[lane] : 0ull;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, wv, o);
        if (lane >= (uint32_t)o) wv = y > wv ? y : wv;
      }
      if (lane < kSmallWarps) s_wt64[lane] = wv;  // inclusive per warp
    }
    __syncthreads();
    const unsigned long long incl = x;
    unsigned long long excl_thr = __shfl_up_sync(0xFFFFFFFFu, incl, 1);
    if (lane == 0) excl_thr = 0;
    const unsigned long long warp_before = warp > 0 ? s_wt64[warp - 1] : 0ull;
    my_start = excl_thr > warp_before ? excl_thr : warp_before;  // start carried into my first position
    if (tid == kSmallThreads - 1) s_maxstart = incl > warp_before ? incl : warp_before;
  }
  __syncthreads();  // s_wt64 is reused by the next scan
  // the lengths: exclusive scan over the chunk, then over the CTAs
  unsigned long long ctatot;
  const unsigned long long lex = block_exclusive_scan<unsigned long long, kSmallThreads>(lsum, &ctatot, s_wt64);
  if (tid == 0) s_tot64 = ctatot;
  if (bad) atomicOr(&s_red[5], 1u);
  cluster.sync();  // chunk totals, run-start maxima and dirty flags are published
  unsigned long long ubase = 0, carry_start = 0;
  uint32_t any_bad = 0;
  for (uint32_t q = 0; q < kSmallCL; ++q) {
    if (q < c) {
      ubase += *cluster.map_shared_rank(&s_tot64, q);
      const unsigned long long ms = *cluster.map_shared_rank(&s_maxstart, q);
      carry_start = ms > carry_start ? ms : carry_start;
    }
    any_bad |= cluster.map_shared_rank(s_red, q)[5];
  }
  STIME(12);
  cluster.sync();  // the last reads of another CTA's shared memory: nobody exits before them
  if (any_bad) {  // an equal-code pair out of order: the regular path (fix-ups) takes over
    if (c == 0 && tid == 0) st->small_status = 1;
    return;
  }
  // run statistics: a run ends at position p when p equals p - 1 but not p + 1
  unsigned long long start = my_start > carry_start ? my_start : carry_start;
  uint32_t maxrun = 0;
  for (int j = 0; j < kSmallItems; ++j) {
    const uint32_t q = b0 + j;
    if (q >= nvalid) break;
    const bool ep = j == 0 ? prev_of_first : ((eq >> (j - 1)) & 1u);
    const bool en = (eq >> j) & 1u;
    if (!ep) start = base_c + q;
    if (ep && !en) {
      const uint32_t L = (uint32_t)(base_c + q - start + 1);
      maxrun = L > maxrun ? L : maxrun;
    }
  }
  in_runs = __reduce_add_sync(0xFFFFFFFFu, in_runs);
  runs = __reduce_add_sync(0xFFFFFFFFu, runs);
  maxrun = __reduce_max_sync(0xFFFFFFFFu, maxrun);
  if (lane == 0) {
    if (in_runs) atomicAdd(&st->n_in_runs, (unsigned long long)in_runs);
    if (runs) {
      atomicAdd(&st->runs_total, (unsigned long long)runs);
      atomicAdd(&st->runs_by_class[0], (unsigned long long)runs);
    }
    if (maxrun) atomicMax(&st->max_run, (unsigned long long)maxrun);
  }
  // A4: perm and sorted offsets; each string's source offset replaces its key
  // in xk (the keys are no longer read: every remote read came before the
  // last cluster barrier)
  unsigned long long d = lex;  // units before my first string, in this CTA's output
  for (int j = 0; j < kSmallItems; ++j) {
    const uint32_t q = b0 + j;
    if (q >= nvalid) break;
    const uint32_t idx = xv[q];
    perm[base_c + q] = idx;
    if (sorted_offsets) {
      sorted_offsets[base_c + q] = (int64_t)(ubase + d);
      xk[q] = (unsigned long long)__ldg(offsets + idx);
    }
    d += len[j];
  }
  if (sorted_offsets && base_c + nvalid == n && tid == kSmallThreads - 1) sorted_offsets[n] = (int64_t)(ubase + ctatot);
  STIME(13);
  if (!sorted_offsets) return;
  __syncthreads();
  // the units, window by window through shared memory (xv / rk / cnt are free
  // now): every thread copies the part of its strings inside the window with
  // independent 8-byte loads, then the CTA writes the window with aligned
  // 16-byte stores (a per-thread byte loop over global memory would be one
  // dependent round trip per byte)
  constexpr uint32_t kWin = kSmallChunk * 6 - 32;  // bytes of stage (xv + rk + cnt), read slack kept
  uint8_t *stage = smem + kSmallChunk * 8;
  const uint8_t *ub8 = (const uint8_t *)units;
  uint8_t *g0 = (uint8_t *)sorted_units + ubase * W;  // first output byte of this CTA
  const unsigned long long tbytes = ctatot * W;
  for (unsigned long long w0 = 0; w0 < tbytes; w0 += kWin) {
    const unsigned long long w1 = w0 + kWin < tbytes ? w0 + kWin : tbytes;
    unsigned long long x = lex * W;
    for (int j = 0; j < kSmallItems; ++j) {
      const uint32_t q = b0 + j;
      if (q >= nvalid) break;
      const unsigned long long nb = (unsigned long long)len[j] * W;
      const unsigned long long lo = x > w0 ? x : w0, hi = x + nb < w1 ? x + nb : w1;
      if (lo < hi) {
        const uint8_t *sp = ub8 + xk[q] * W + (lo - x);
        for (unsigned long long y = lo; y < hi; y += 8) {
          const int take = (int)(hi - y < 8 ? hi - y : 8);
          const uint64_t v8 = load8_unaligned(sp + (y - lo), take);
          for (int b = 0; b < take; ++b) stage[y - w0 + b] = (uint8_t)(v8 >> (8 * b));
        }
      }
      x += nb;
    }
    __syncthreads();
    // aligned 16-byte chunks of [g0 + w0, g0 + w1), edges byte by byte
    const uintptr_t a0 = (uintptr_t)(g0 + w0), a1 = (uintptr_t)(g0 + w1);
    const uintptr_t c0 = (a0 + 15) & ~(uintptr_t)15, c1 = a1 & ~(uintptr_t)15;
    if (c0 < c1) {
      for (uintptr_t a = c0 + (uintptr_t)tid * 16; a < c1; a += (uintptr_t)kSmallThreads * 16) {
        const uint32_t so_ = (uint32_t)(a - a0);
        uint4 o;
        o.x = (uint32_t)stage[so_] | ((uint32_t)stage[so_ + 1] << 8) | ((uint32_t)stage[so_ + 2] << 16) |
              ((uint32_t)stage[so_ + 3] << 24);
        o.y = (uint32_t)stage[so_ + 4] | ((uint32_t)stage[so_ + 5] << 8) | ((uint32_t)stage[so_ + 6] << 16) |
              ((uint32_t)stage[so_ + 7] << 24);
        o.z = (uint32_t)stage[so_ + 8] | ((uint32_t)stage[so_ + 9] << 8) | ((uint32_t)stage[so_ + 10] << 16) |
              ((uint32_t)stage[so_ + 11] << 24);
        o.w = (uint32_t)stage[so_ + 12] | ((uint32_t)stage[so_ + 13] << 8) | ((uint32_t)stage[so_ + 14] << 16) |
              ((uint32_t)stage[so_ + 15] << 24);
        *reinterpret_cast<uint4 *>(a) = o;
      }
      for (uintptr_t a = a0 + tid; a < c0; a += kSmallThreads) *(uint8_t *)a = stage[a - a0];
      for (uintptr_t a = c1 + tid; a < a1; a += kSmallThreads) *(uint8_t *)a = stage[a - a0];
    } else {
      for (uintptr_t a = a0 + tid; a < a1; a += kSmallThreads) *(uint8_t *)a = stage[a - a0];
    }
    __syncthreads();
  }
  STIME(14);
}

extern "C" int husky_debug_small_times(unsigned long long *out) {
#ifdef HUSKY_SMALL_TIMING
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_small_t, sizeof(g_small_t));
  return 64;
#else
  (void)out;
  return 0;
#endif
}

static int small_clusters_ok(int coder_k) {
  // whether a 16-CTA cluster with this footprint can be resident (one CTA per
  // SM on 16 SMs of one GPC); asked once per device
  static std::atomic<unsigned long long> asked{0}, ok{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (asked.load() & bit) return (ok.load() & bit) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kSmallCL);
  cfg.blockDim = dim3(kSmallThreads);
  cfg.dynamicSmemBytes = kSmallSmem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kSmallCL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&clusters, k_small<HUSKY_CODER_ASCII>, &cfg);
  (void)coder_k;
  cudaGetLastError();
  if (e == cudaSuccess && clusters >= 1) ok.fetch_or(bit);
  asked.fetch_or(bit);
  return (e == cudaSuccess && clusters >= 1) ? 1 : 0;
}

template <int CODER>
static cudaError_t small_launch(const void *units, const int64_t *offsets, uint64_t n, uint64_t *kA, uint64_t *kB,
                                uint32_t *vA, uint32_t *vB, uint32_t *perm, void *su, int64_t *so, DevState *st,
                                cudaStream_t s) {
  static SmemAttr attr_smem;
  static std::atomic<unsigned long long> np_done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(np_done.load() & (1ull << (dev & 63)))) {
    cudaFuncSetAttribute(k_small<CODER>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    np_done.fetch_or(1ull << (dev & 63));
  }
  attr_smem.ensure(k_small<CODER>, kSmallSmem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kSmallCL);
  cfg.blockDim = dim3(kSmallThreads);
  cfg.dynamicSmemBytes = kSmallSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kSmallCL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_small<CODER>, units, offsets, n, kA, kB, vA, vB, perm, su, so, st);
}

bool small_path_available() {
  static std::atomic<int> cached{-1};
  int v = cached.load();
  if (v < 0) {
    // make sure the attributes are set before the occupancy query
    cudaFuncSetAttribute(k_small<HUSKY_CODER_ASCII>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_small<HUSKY_CODER_ASCII>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmallSmem);
    v = small_clusters_ok(0);
    cached.store(v);
  }
  return v == 1;
}

cudaError_t launch_small(int coder, const void *units, const int64_t *offsets, uint64_t n, uint64_t *kA,
                         uint64_t *kB, uint32_t *vA, uint32_t *vB, uint32_t *perm, void *su, int64_t *so,
                         DevState *st, cudaStream_t s) {
  Scope sc_(ST_SMALL, s, n);
  switch (coder) {
    case HUSKY_CODER_ASCII:
      return small_launch<HUSKY_CODER_ASCII>(units, offsets, n, kA, kB, vA, vB, perm, su, so, st, s);
    case HUSKY_CODER_UNICODE:
      return small_launch<HUSKY_CODER_UNICODE>(units, offsets, n, kA, kB, vA, vB, perm, su, so, st, s);
    case HUSKY_CODER_ENGLISH5:
      return small_launch<HUSKY_CODER_ENGLISH5>(units, offsets, n, kA, kB, vA, vB, perm, su, so, st, s);
    default:
      return small_launch<HUSKY_CODER_ENGLISH6>(units, offsets, n, kA, kB, vA, vB, perm, su, so, st, s);
  }
}

}  // namespace husky
