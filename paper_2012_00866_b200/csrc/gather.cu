// gather.cu -- A4: sorted-string gather.
//
// The paper's co-swap moves object references with the keys;
// here the strings themselves are materialised in sorted order:
//   sorted_offsets = exclusive scan of len[perm[i]]  (single pass, look-back)
//   sorted_units   = concatenation of units[offsets[perm[i]] ..)
// A tile of kGatherTile = 1024 sorted positions (256 threads x 4): perm (coalesced) ->
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

#ifdef HUSKY_TIMING
// per-tile phase timestamps of the last gather (instrumented builds only)
constexpr int kGTimingTiles = 16384;
__device__ unsigned long long g_gather_times[kGTimingTiles][8];
__device__ __forceinline__ unsigned long long gt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define GT(tile, i) \
  do { if (threadIdx.x == 0 && (tile) < kGTimingTiles) g_gather_times[tile][i] = gt_now(); } while (0)
#else
#define GT(tile, i) do { } while (0)
#endif

// PACKED: perm holds index | min(len,15) << 28 (written by the encoder, carried
// through the radix as the payload).  Strings whose length is <= PL are then
// rebuilt from their sorted code (sequential reads only); perm is unpacked in
// place.  Only longer strings read offsets / units at random.
// CHECK (the main gather after the key sort) also does A3 in the same pass:
// run detection (equal adjacent codes; the k-th run start / end of the array
// belong to run k, ids from a second single-pass scan whose look-back runs in
// warp 1 next to the length scan's in warp 0) and the order check of every
// adjacent equal-code pair on the strings this tile just staged (pairs whose
// strings are not both in the stage compare the source strings).  A run with an
// out-of-order pair is marked dirty for the fix-up (A5).
struct GatherRuns {
  uint32_t *run_start, *run_end;
  uint8_t *dirty;
  unsigned long long *lb;  // look-back words of the run-count scan (one per tile)
  DevState *st;            // n_runs
};

// look-back words per lane and round trip (32 V predecessors per round);
// measured on C5 (2^30) gathers: V = 1 42.4 ms, 2 45.1, 4 46.4 -- the walk
// width is not what bounds the gather (C2: 252 / 262 / 277 us)
#ifndef HUSKY_GATHER_LBV
#define HUSKY_GATHER_LBV 1
#endif
constexpr int kGatherLbV = HUSKY_GATHER_LBV;

template <int CODER, bool PACKED, bool CHECK, bool PEER>
// L1 prefetch of the long strings' units: 0 = as soon as the offset is loaded
// (before the block scan), 1 = after the tile's aggregate is published, 2 = none
#ifndef HUSKY_GATHER_PF
#define HUSKY_GATHER_PF 1
#endif
// resident CTAs per SM: 5 for the packed instantiations (48 registers; C2
// 280 vs 289 us at 4), 4 for the others (64 registers, no spills: the C5 gather
// with slab records 50 -> 44 ms)
#ifndef HUSKY_GATHER_CPASYNC
#define HUSKY_GATHER_CPASYNC 1
#endif
#ifndef HUSKY_GATHER_MINB
#define HUSKY_GATHER_MINB (PACKED ? 5 : 4)
#endif
__global__ void __launch_bounds__(kGatherThreads, HUSKY_GATHER_MINB)
    k_gather(uint32_t *__restrict__ perm, uint64_t n, const void *__restrict__ units,
             const int64_t *__restrict__ offsets, void *__restrict__ sorted_units,
             int64_t *__restrict__ sorted_offsets, unsigned long long *lb, uint32_t *tile_counter,
             uint32_t epoch, const int64_t *base_ptr, int dbg, const uint64_t *__restrict__ codes,
             const DevState *st, GatherRuns runs, const PeerTable *peer, const uint4 *__restrict__ slab) {
  using T = CoderTraits<CODER>;
  constexpr int W = T::kUnitBytes;
  constexpr uint32_t PL = T::kPL;
  extern __shared__ __align__(16) uint8_t stage[];  // kGatherStage + 32 bytes (+ slab records, CHECK)
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_wt[kGatherThreads / 32 + 1];
  __shared__ unsigned long long s_base, s_rbase;
  // CHECK: each thread's last item (code, length, index, tile-local unit offset)
  __shared__ unsigned long long s_lcode[CHECK ? kGatherThreads : 1], s_loff[CHECK ? kGatherThreads : 1];
  __shared__ uint32_t s_llen[CHECK ? kGatherThreads : 1], s_lidx[CHECK ? kGatherThreads : 1];
  // PEER: the buckets' start positions / units in the partitioned order
  __shared__ unsigned long long s_sn[PEER ? kMaxPeers + 1 : 1], s_su[PEER ? kMaxPeers + 1 : 1];
  // alphabet-compressed ASCII codes: rank -> unit (the inverse of the re-packing)
  __shared__ uint8_t s_unrank[64];
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  pdl_wait();  // the main gather is a programmatic dependent of the key sort
  // the tile id first: its round trip overlaps the DevState reads below (a
  // CTA that then returns on invalid input returns with every other CTA)
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  uint32_t cbits = 0;
  bool ccomp = false;
  if (CODER == HUSKY_CODER_ASCII && (PACKED || CHECK) && st && st->ccomp) {
    ccomp = true;
    cbits = st->cbits;
    if (tid < 128) {
      const uint32_t a[4] = {st->alpha[0], st->alpha[1], st->alpha[2], st->alpha[3]};
      if (tid == 0 || ((a[tid >> 5] >> (tid & 31)) & 1u)) s_unrank[alpha_rank(a, tid)] = (uint8_t)tid;
    }
  }
  // unit byte b (< S) of a string rebuilt from its sorted code
  auto decb = [&](uint64_t code, int b) -> uint8_t {
    return ccomp ? decode_byte_c(code, b, cbits, s_unrank) : decode_byte<CODER>(code, b);
  };
  if (PEER) {
    for (uint32_t b = tid; b <= peer->world; b += kGatherThreads) {
      s_sn[b] = peer->start_n[b];
      s_su[b] = peer->start_u[b];
    }
  }
  const RunRule rule = run_rule<CODER>(CHECK ? st : nullptr);  // run detection rule (R6 / R19)
  if (st) {
    if (st->violations & kOffsetsBad) return;  // invalid input: reported by the caller
    if ((PACKED || CHECK) && codes == nullptr) codes = reinterpret_cast<const uint64_t *>(st->sorted_keys);
  }
  // re-gather of a span: output positions start at *base_ptr (unchanged by us)
  const unsigned long long gbase = base_ptr ? (unsigned long long)*base_ptr : 0ull;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t p0 = (uint64_t)tile * kGatherTile + (uint64_t)tid * kGatherItems;
  GT(tile, 0);
  if (CHECK && st && st->trivial_mask == 0xFFu && n > 1) {
    // every code is equal: the whole array is one run, which the fix-up or the
    // refinement (A6) reorders and gathers again -- gathering it here in code
    // order would be thrown away (C4).  Unpack perm, record the run as dirty.
    if (PACKED)
      for (int j = 0; j < kGatherItems; ++j)
        if (p0 + j < n) perm[p0 + j] &= 0x0FFFFFFFu;
    if (tile == 0 && tid == 0) {
      runs.run_start[0] = 0;
      runs.run_end[0] = (uint32_t)(n - 1);
      runs.dirty[0] = 1;
      runs.st->n_runs = 1;
      if (sorted_offsets) {  // the span's ends; the re-gather fills the inside
        sorted_offsets[0] = (int64_t)gbase;
        sorted_offsets[n] = (int64_t)gbase + (offsets[n] - offsets[0]);
      }
    }
    return;
  }

  // per item: len (units) and either the source offset or, for strings rebuilt
  // from their code, the code itself (bit j of `dec`); slab strings (bit j of
  // `slb`): units [0, S) from the code, the rest from the 16-byte slab record
  // in sl[j] -- one random read instead of offsets + units (encode.cu)
  uint32_t raw[kGatherItems];
#pragma unroll
  for (int j = 0; j < kGatherItems; ++j) raw[j] = p0 + j < n ? perm[p0 + j] : 0u;
#ifdef HUSKY_CHECKED
  if (st && !PEER)
    for (int j = 0; j < kGatherItems; ++j)
      if (p0 + j < n) HCHK(kChkGatherPerm, PACKED ? (raw[j] & 0x0FFFFFFFu) : raw[j], st->chk_n);
#endif
  uint64_t sv[kGatherItems], cc[kGatherItems];
  uint32_t len[kGatherItems], ix[kGatherItems];
  // slab records parked in shared memory ([item][thread]: conflict-free 16-B
  // accesses) until the staging, so they hold no registers across the scan
  uint4 *s_slab = reinterpret_cast<uint4 *>(stage + kGatherStage + 32);
  uint32_t dec = 0, slb = 0;
  unsigned long long mine = 0;
  // the main gather with slab records: every item's record goes straight to
  // its shared-memory park by cp.async (no register round trip, so the
  // records of all items are in flight at once; C5 gather 37.4 -> 36.0 ms)
  constexpr bool kRecAsync = HUSKY_GATHER_CPASYNC && CHECK;
  if (kRecAsync && slab != nullptr) {
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j)  // (packed: strings longer than PL only -- the others need no record)
      if (p0 + j < n && (!PACKED || (raw[j] >> 28) > PL))
        cp_async16(&s_slab[j * kGatherThreads + tid], slab + (PACKED ? (raw[j] & 0x0FFFFFFFu) : raw[j]));
    cp_async_commit();
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) cc[j] = p0 + j < n ? __ldg(codes + p0 + j) : 0ull;
    cp_async_wait_all();
  }
#pragma unroll
  for (int j = 0; j < kGatherItems; ++j) {
    if (!kRecAsync || slab == nullptr) cc[j] = 0;
    ix[j] = 0;
    if (p0 + j >= n) {
      sv[j] = 0;
      len[j] = 0;
    } else {
      uint32_t idx = raw[j], lc = 15;
      if (PACKED) {
        lc = idx >> 28;
        idx &= 0x0FFFFFFFu;
        perm[p0 + j] = idx;
      }
      ix[j] = idx;
      if (CHECK && !(kRecAsync && slab != nullptr)) cc[j] = __ldg(codes + p0 + j);
      uint4 rec = make_uint4(0xFFu, 0, 0, 0);
      if (PACKED && lc <= PL) {
        dec |= 1u << j;
        len[j] = lc;
        sv[j] = CHECK ? cc[j] : __ldg(codes + p0 + j);
      } else if (CHECK && slab != nullptr &&
                 (rec = kRecAsync ? s_slab[j * kGatherThreads + tid] : __ldg(slab + idx), (rec.x & 0xFFu) != 0xFFu)) {
        slb |= 1u << j;
        len[j] = rec.x & 0xFFu;
        sv[j] = cc[j];
        if (!kRecAsync) s_slab[j * kGatherThreads + tid] = rec;
      } else {
        const int64_t a = __ldg(offsets + idx);
        sv[j] = (uint64_t)a;
        // a packed length below 15 is exact: the scan need not wait for the
        // offsets load, whose value is first used by the staging
        if (PACKED && lc < 15) len[j] = lc;
        else len[j] = (uint32_t)(__ldg(offsets + idx + 1) - a);
#if HUSKY_GATHER_PF == 0
        // the staging reads these units after the block scan: start the fetch now
        if ((PEER || sorted_units) && len[j]) {
          const uint8_t *pa = (const uint8_t *)units + (uint64_t)a * W;
          asm volatile("prefetch.global.L1 [%0];" ::"l"(pa));
          if ((((uintptr_t)pa & 127) + (uint64_t)len[j] * W) > 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(pa + 127));
        }
#endif
      }
    }
    mine += len[j];
  }
  // CHECK: run flags.  eqp bit j: position p0+j equals its predecessor; eqn:
  // equals its successor (neighbours across lanes by shuffles, across warps and
  // tiles from global memory)
  uint32_t eqp = 0, eqn = 0, nstart = 0;
  if (CHECK) {
    unsigned long long prevc = __shfl_up_sync(0xFFFFFFFFu, cc[kGatherItems - 1], 1);
    unsigned long long nextc = __shfl_down_sync(0xFFFFFFFFu, cc[0], 1);
    if (lane == 0) prevc = p0 > 0 && p0 - 1 < n ? __ldg(codes + p0 - 1) : 0ull;
    if (lane == 31) nextc = p0 + kGatherItems < n ? __ldg(codes + p0 + kGatherItems) : 0ull;
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
      const uint64_t p = p0 + j;
      const unsigned long long pc = j == 0 ? prevc : cc[j - 1];
      const unsigned long long nc = j == kGatherItems - 1 ? nextc : cc[j + 1];
      const bool ep = p < n && p > 0 && ((cc[j] ^ pc) & rule.mask) == 0;
      const bool en = p + 1 < n && ((cc[j] ^ nc) & rule.mask) == 0;
      eqp |= (uint32_t)ep << j;
      eqn |= (uint32_t)en << j;
      nstart += (!ep && en);
    }
  }
  // CHECK, thread 0: the previous tile's last string when it has this tile's
  // first code (the tile-boundary pair is then checked); its dependent loads
  // issued here so they overlap the scan and the staging
  unsigned long long b_code = 0;
  uint32_t b_idx = 0, b_len = 0;
  if (CHECK && tid == 0 && (eqp & 1u)) {
    b_code = __ldg(codes + p0 - 1);
    b_idx = perm[p0 - 1] & (PACKED ? 0x0FFFFFFFu : 0xFFFFFFFFu);  // unpacked or not yet
    b_len = (uint32_t)(__ldg(offsets + b_idx + 1) - __ldg(offsets + b_idx));
  }
  // one scan for both: units in the low 48 bits, run starts above
  unsigned long long tile_total;
  unsigned long long excl_t = block_exclusive_scan<unsigned long long, kGatherThreads>(
      mine | ((unsigned long long)nstart << 48), &tile_total, s_wt);
  GT(tile, 1);
  const uint32_t excl_r = (uint32_t)(excl_t >> 48), tile_runs = (uint32_t)(tile_total >> 48);
  excl_t &= (1ull << 48) - 1;
  tile_total &= (1ull << 48) - 1;
  if (tid == 0) {
    st_relaxed_u64(lb + tile, make_flag(tile == 0 ? kFlagInc : kFlagAgg, epoch, tile_total));
    if (CHECK) st_relaxed_u64(runs.lb + tile, make_flag(tile == 0 ? kFlagInc : kFlagAgg, epoch, tile_runs));
  }

#if HUSKY_GATHER_PF == 1 || HUSKY_GATHER_PF == 3
  // the long strings' units, for the staging below (issued after the publish).
  // Main gather only: the re-gathers after a refinement (C4: every string long)
  // measured faster without it (C4 gather 526 vs 582 us; C2 276 vs 286 us with)
  if (CHECK && sorted_units) {
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
      if (p0 + j < n && !(((dec | slb) >> j) & 1) && len[j]) {
        const uint8_t *pa = (const uint8_t *)units + sv[j] * W;
#if HUSKY_GATHER_PF == 1
        asm volatile("prefetch.global.L1 [%0];" ::"l"(pa));
        if ((((uintptr_t)pa & 127) + (uint64_t)len[j] * W) > 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(pa + 127));
#else
        asm volatile("prefetch.global.L2 [%0];" ::"l"(pa));
        if ((((uintptr_t)pa & 127) + (uint64_t)len[j] * W) > 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(pa + 127));
#endif
      }
    }
  }
#endif
  const uint8_t *ub = (const uint8_t *)units;
  uint8_t *ob = (uint8_t *)sorted_units;
  const uint64_t tile_bytes = tile_total * W;
  const bool direct = !PEER && (dbg & 1) != 0;
  const bool want_units = PEER || sorted_units != nullptr;

  // stage tile-local output bytes [w0, w1) of this thread's strings at stage[x - w0]
  auto stage_window = [&](uint64_t w0, uint64_t w1) {
    uint64_t d = excl_t * W;
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
      const uint64_t nb = (uint64_t)len[j] * W;
      const uint64_t lo = d > w0 ? d : w0, hi = d + nb < w1 ? d + nb : w1;
      if (lo < hi) {
        if (PACKED && ((dec >> j) & 1)) {
          for (uint64_t x = lo; x < hi; ++x) stage[x - w0] = decb(sv[j], (int)(x - d));
        } else if (PACKED && CHECK && ((slb >> j) & 1)) {
          // (the packed instantiations keep the per-byte loop: the register
          // image below costs them spills -- C2 / C3 gathers 250 / 224 ->
          // 264 / 240 us)
          constexpr int SB = T::kS * W;
          const uint4 rec = s_slab[j * kGatherThreads + tid];
          for (uint64_t x = lo; x < hi; ++x) {
            const int b = (int)(x - d);
            stage[x - w0] = b < SB ? decb(sv[j], b) : slab_byte(rec, b - SB + 1);
          }
        } else if (!PACKED && CHECK && ((slb >> j) & 1)) {
          // the string's bytes assembled in three registers first -- units
          // [0, S) decoded from the code (independent table lookups), the
          // rest from the slab record -- then stored byte by byte with no
          // dependency between the stores (a per-byte decode loop measured
          // 10 us per C5 tile, half of the tile's time)
          constexpr int SB = T::kS * W;  // string bytes [0, SB) come from the code
          uint64_t img0 = 0, img1 = 0, img2 = 0;
#pragma unroll
          for (int b = 0; b < SB; ++b) {
            const uint64_t ch = decb(sv[j], b);
            if (b < 8) img0 |= ch << (8 * b);
            else img1 |= ch << (8 * (b - 8));
          }
          {
            const uint4 rec = s_slab[j * kGatherThreads + tid];
            const uint64_t r0 = (uint64_t)rec.x | ((uint64_t)rec.y << 32), r1 = (uint64_t)rec.z | ((uint64_t)rec.w << 32);
            const uint64_t t0 = (r0 >> 8) | (r1 << 56), t1 = r1 >> 8;  // record bytes 1..15
            if (SB == 9) {
              img1 |= t0 << 8;
              img2 = (t0 >> 56) | (t1 << 8);
            } else {  // SB == 6
              img0 |= t0 << 48;
              img1 = (t0 >> 16) | (t1 << 48);
              img2 = t1 >> 16;
            }
          }
          // bytes up to a 4-byte boundary of the stage, then whole 32-bit
          // words (funnel-shifted out of the image), then the tail
          auto img_byte = [&](uint32_t b) -> uint32_t {
            const uint64_t wv = b < 8 ? img0 : (b < 16 ? img1 : img2);
            return (uint32_t)(wv >> (8 * (b & 7))) & 0xFFu;
          };
          uint64_t x = lo;
          for (; x < hi && ((x - w0) & 3); ++x) stage[x - w0] = (uint8_t)img_byte((uint32_t)(x - d));
          for (; x + 4 <= hi; x += 4) {
            const uint32_t b = (uint32_t)(x - d), sh = (b & 7) * 8;
            const uint64_t lo64 = b < 8 ? img0 : (b < 16 ? img1 : img2), hi64 = b < 8 ? img1 : (b < 16 ? img2 : 0ull);
            const uint64_t v = sh ? ((lo64 >> sh) | (hi64 << (64 - sh))) : lo64;
            *reinterpret_cast<uint32_t *>(stage + (x - w0)) = (uint32_t)v;
          }
          for (; x < hi; ++x) stage[x - w0] = (uint8_t)img_byte((uint32_t)(x - d));
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
  // write tile-local bytes [lo, hi) of the window staged from w0 (byte x at
  // stage[x - w0]) to g0 + x
  auto write_range = [&](uint8_t *g0, uint64_t w0, uint64_t lo_x, uint64_t hi_x) {
    const uint32_t align = (uint32_t)((uintptr_t)g0 & 15);
    uint8_t *a0 = g0 - align;  // 16-aligned; tile byte x lives at a0 + align + x
    const uint64_t lo_b = align + lo_x, hi_b = align + hi_x, st_b = align + w0;  // st_b: address of stage[0]
    const uint64_t c0 = lo_b / 16, c1 = (hi_b + 15) / 16;
    const uint32_t *sw = reinterpret_cast<const uint32_t *>(stage);
    for (uint64_t ch = c0 + tid; ch < c1; ch += kGatherThreads) {
      uint64_t lo = ch * 16, hi = lo + 16;
      if (lo >= lo_b && hi <= hi_b) {
        uint32_t so = (uint32_t)(lo - st_b);  // stage offset of the chunk
        uint32_t wi = so >> 2, sh = (so & 3) * 8;
        uint32_t x0 = sw[wi], x1 = sw[wi + 1], x2 = sw[wi + 2], x3 = sw[wi + 3], x4 = sw[wi + 4];
        uint4 o;
        o.x = __funnelshift_r(x0, x1, sh);
        o.y = __funnelshift_r(x1, x2, sh);
        o.z = __funnelshift_r(x2, x3, sh);
        o.w = __funnelshift_r(x3, x4, sh);
        *reinterpret_cast<uint4 *>(a0 + lo) = o;
      } else {
        for (uint64_t b = (lo > lo_b ? lo : lo_b); b < (hi < hi_b ? hi : hi_b); ++b) a0[b] = stage[b - st_b];
      }
    }
  };
  // PEER: the window's bytes bucket by bucket, each to its destination
  auto write_window = [&](uint8_t *g0, uint64_t w0, uint64_t w1) {
    if (!PEER) {
      write_range(g0, w0, w0, w1);
      return;
    }
    const uint64_t v0 = s_base * W;  // virtual byte of tile byte 0 (s_base: units before the tile)
    uint32_t b = 0;
    while (b + 1 < peer->world && s_su[b + 1] * W <= v0 + w0) ++b;
    for (; b < peer->world && s_su[b] * W < v0 + w1; ++b) {
      const uint64_t blo = s_su[b] * W, bhi = s_su[b + 1] * W;
      const uint64_t lo = blo > v0 + w0 ? blo - v0 : w0, hi = bhi < v0 + w1 ? bhi - v0 : w1;
      if (lo < hi) write_range(reinterpret_cast<uint8_t *>(peer->units[b] + v0), w0, lo, hi);
    }
  };

  const uint64_t first_w1 = tile_bytes < (uint64_t)kGatherStage ? tile_bytes : (uint64_t)kGatherStage;
  if (want_units && !direct) stage_window(0, first_w1);  // overlaps the look-back
  GT(tile, 2);

  if (CHECK) {
    s_lcode[tid] = cc[kGatherItems - 1];
    s_llen[tid] = len[kGatherItems - 1];
    s_lidx[tid] = ix[kGatherItems - 1];
    s_loff[tid] = excl_t + mine - len[kGatherItems - 1];
  }
  // CHECK: the order check needs the stage and the neighbours' last items but
  // no look-back.  Warps 0 / 1 (the look-back warps) only signal that their
  // strings are staged (bar.arrive) and start walking at once; warps 2.. wait
  // for every warp's stage (bar.sync on the same named barrier) and compare
  // meanwhile; warps 0 / 1 compare after their walks
  uint32_t bad = 0;
  if (CHECK) {
    static_assert(kGatherThreads == 256, "named-barrier thread counts");
    if (warp < 2) {
      asm volatile("bar.arrive 1, 256;" ::: "memory");
      asm volatile("bar.sync 2, 64;" ::: "memory");  // warp 1's first pair reads warp 0's last string
    } else {
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
  }
  if (warp == 0) {
    unsigned long long ex =
        tile == 0 ? 0ull : ((dbg & 2) ? lookback(lb, tile, 1, epoch) : warp_lookback<kGatherLbV>(lb, tile, epoch));
    if (lane == 0) {
      if (tile != 0) st_relaxed_u64(lb + tile, make_flag(kFlagInc, epoch, ex + tile_total));
      s_base = ex;
      if (!PEER && (uint64_t)(tile + 1) * kGatherTile >= n) sorted_offsets[n] = (int64_t)(gbase + ex + tile_total);
    }
  } else if (CHECK && warp == 1) {  // the run-count scan's look-back, next to warp 0's
    unsigned long long ex = tile == 0 ? 0ull : warp_lookback<kGatherLbV>(runs.lb, tile, epoch);
    if (lane == 0) {
      if (tile != 0) st_relaxed_u64(runs.lb + tile, make_flag(kFlagInc, epoch, ex + tile_runs));
      s_rbase = ex;
      if ((uint64_t)(tile + 1) * kGatherTile >= n) runs.st->n_runs = (uint32_t)(ex + tile_runs);
    }
  }
  if (CHECK) {
    // adjacent pairs (p-1, p) with equal codes, p = my items
    const uint64_t win_units = first_w1 / W;  // units [0, win_units) of the tile are staged
    unsigned long long pc, po;
    uint32_t pl, pi;
    if (tid > 0) {
      pc = s_lcode[tid - 1]; pl = s_llen[tid - 1]; pi = s_lidx[tid - 1]; po = s_loff[tid - 1];
    } else if (p0 > 0) {  // the previous tile's last string (loaded above): from the source
      pc = b_code;
      pi = b_idx;
      pl = b_len;
      po = ~0ull;  // not staged
    } else {
      pc = ~cc[0]; pl = 0; pi = 0; po = ~0ull;  // position 0: no pair
    }
    unsigned long long d = excl_t;
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
      if ((eqp >> j) & 1) {
        int c;
        if (pl <= rule.PL || len[j] <= rule.PL) {
          c = pl < len[j] ? -1 : (pl > len[j] ? 1 : 0);  // short rule (R6)
        } else if (sorted_units && !direct && po != ~0ull && po + pl <= win_units && d + len[j] <= win_units) {
          c = 0;  // both staged: compare units [S, min) in shared memory, 8 bytes at a time
          const uint32_t m = (pl < len[j] ? pl : len[j]) * W;  // bytes
          for (uint32_t k = rule.S * W; k < m && c == 0; k += 8) {
            uint64_t x = stage_load8(stage, (uint32_t)(po * W) + k), y = stage_load8(stage, (uint32_t)(d * W) + k);
            const uint32_t take = m - k < 8 ? m - k : 8;
            if (take < 8) {
              const uint64_t msk = (1ull << (8 * take)) - 1;
              x &= msk;
              y &= msk;
            }
            const uint64_t df = x ^ y;
            if (df) {
              const int sh = ((__ffsll((long long)df) - 1) / (8 * W)) * (8 * W);  // first differing unit
              const uint64_t um = W == 1 ? 0xFFull : 0xFFFFull;
              c = ((x >> sh) & um) < ((y >> sh) & um) ? -1 : 1;
            }
          }
          if (c == 0) c = pl < len[j] ? -1 : (pl > len[j] ? 1 : 0);
        } else {
          c = cmp_units_from<CODER>(units, __ldg(offsets + pi), pl, __ldg(offsets + ix[j]), len[j], rule.S);
        }
        if (c > 0 || (c == 0 && pi > ix[j])) bad |= 1u << j;
      }
      pc = cc[j]; pl = len[j]; pi = ix[j]; po = d;
      d += len[j];
    }
  }
  __syncthreads();
  GT(tile, 3);
  const unsigned long long tbase = gbase + s_base;  // units before this tile
  if (!PEER) {
    unsigned long long d = tbase + excl_t;
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
      if (p0 + j < n) sorted_offsets[p0 + j] = (int64_t)d;
      d += len[j];
    }
  } else if (p0 < n) {
    // length and global index of each string, into its destination's arrays
    uint32_t b = 0;
    while (b + 1 < peer->world && s_sn[b + 1] <= p0) ++b;
#pragma unroll
    for (int j = 0; j < kGatherItems; ++j) {
      const uint64_t p = p0 + j;
      if (p < n) {
        while (s_sn[b + 1] <= p) ++b;
        reinterpret_cast<uint32_t *>(peer->lens[b])[p] = len[j];
        reinterpret_cast<uint32_t *>(peer->gidx[b])[p] = peer->gbase + ix[j];
      }
    }
  }
  if (CHECK) {
    // runs: the k-th start and the k-th end of the array belong to run k
    if (eqp | eqn) {
      uint32_t rid = (uint32_t)s_rbase + excl_r - 1;
#pragma unroll
      for (int j = 0; j < kGatherItems; ++j) {
        const bool ep = (eqp >> j) & 1, en = (eqn >> j) & 1;
        const uint32_t p = (uint32_t)(p0 + j);
        if (!ep && en) {
          HCHK(kChkGatherRuns, rid + 1, n);
          runs.run_start[++rid] = p;
        }
        if (ep && !en) runs.run_end[rid] = p;
        if ((bad >> j) & 1) runs.dirty[rid] = 1;
      }
    }
  }
  GT(tile, 4);
  if (!want_units) return;

  uint8_t *g0 = ob + tbase * W;  // first output byte of the tile
#ifdef HUSKY_CHECKED
  if (st && !PEER && tid == 0) HCHK(kChkGatherUnits, (tbase + tile_total) * W, st->chk_units + 1);
#endif
  if (!direct) {
    write_window(g0, 0, first_w1);
    for (uint64_t w0 = first_w1; w0 < tile_bytes; w0 += kGatherStage) {  // large tiles: more windows
      const uint64_t w1 = w0 + kGatherStage < tile_bytes ? w0 + kGatherStage : tile_bytes;
      __syncthreads();
      stage_window(w0, w1);
      __syncthreads();
      write_window(g0, w0, w1);
    }
    GT(tile, 5);
    if (PEER) {
      // The peer stores (units, lengths, global indices into the destination
      // ranks' NCCL windows over NVLink) are made visible at system scope
      // before this CTA retires: the CTA barrier gathers every thread's
      // stores, the system-scope fence is cumulative over them.  The host
      // then enqueues a 1-element ncclAllReduce on the same stream, which no
      // rank completes before every rank's gather kernel has completed, and
      // only after it do the ranks read their windows (multi.cu: exec) -- the
      // stores happen-before the reads across ranks.
      __syncthreads();
      if (tid == 0) __threadfence_system();
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
        if (CHECK && ((__shfl_sync(0xFFFFFFFFu, slb, t) >> j) & 1)) {
          const uint4 r = s_slab[j * kGatherThreads + (warp * 32 + t)];
          constexpr int SB = T::kS * W;
          for (uint64_t b = lane; b < nb; b += 32)
            ob[d * W + b] = b < SB ? decb(s, (int)b) : slab_byte(r, (int)b - SB + 1);
        } else if (PACKED && ((dt >> j) & 1)) {
          for (uint64_t b = lane; b < nb; b += 32) ob[d * W + b] = decb(s, (int)b);
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
                   bool packed, const uint64_t *packed_codes, const DevState *st, const GatherRunsOut *runs_out,
                   const uint4 *slab) {
  if (n == 0) return;
  Scope sc_(ST_GATHER, s, n);
  dim3 g((unsigned)gather_tiles(n)), b(kGatherThreads);
  // HUSKY_DEBUG_GATHER: bit 0 forces the unstaged copy, bit 1 the serial look-back
  static const int dbg = [] {
    const char *v = getenv("HUSKY_DEBUG_GATHER");
    return v ? atoi(v) : 0;
  }();
  GatherRuns runs{};
  if (runs_out) runs = GatherRuns{runs_out->run_start, runs_out->run_end, runs_out->dirty, runs_out->lb, runs_out->st};
  const bool chk = runs_out != nullptr;
  if (!chk) slab = nullptr;  // slab records are read by the main (CHECK) gather only
#define G_LAUNCH(C, P, K)                                                                                         \
  do {                                                                                                            \
    const int kSmem = kGatherStage + 32 + (K && slab ? kGatherTile * 16 : 0);                                     \
    static SmemAttr attr;                                                                                         \
    attr.ensure(k_gather<C, P, K, false>, kGatherStage + 32 + (K ? kGatherTile * 16 : 0));                        \
    launch_pdl(k_gather<C, P, K, false>, g, b, kSmem, s, perm, n, units, offsets, sorted_units, sorted_offsets, lb, \
               tile_counter, epoch, base_ptr, dbg, packed_codes, st, runs, (const PeerTable *)nullptr, slab);     \
  } while (0)
  if (coder == HUSKY_CODER_ASCII) {
    if (packed) {
      if (chk) G_LAUNCH(HUSKY_CODER_ASCII, true, true);
      else G_LAUNCH(HUSKY_CODER_ASCII, true, false);
    } else {
      if (chk) G_LAUNCH(HUSKY_CODER_ASCII, false, true);
      else G_LAUNCH(HUSKY_CODER_ASCII, false, false);
    }
  } else {
    if (packed) {
      if (chk) G_LAUNCH(HUSKY_CODER_UNICODE, true, true);
      else G_LAUNCH(HUSKY_CODER_UNICODE, true, false);
    } else {
      if (chk) G_LAUNCH(HUSKY_CODER_UNICODE, false, true);
      else G_LAUNCH(HUSKY_CODER_UNICODE, false, false);
    }
  }
#undef G_LAUNCH
}

void launch_gather_peer(int coder, const uint32_t *perm, uint64_t n, const void *units, const int64_t *offsets,
                        unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, const PeerTable *d_table,
                        cudaStream_t s) {
  if (n == 0) return;
  constexpr int kSmem = kGatherStage + 32;
  Scope sc_(ST_MULTI, s, n);
  dim3 g((unsigned)gather_tiles(n)), b(kGatherThreads);
  uint32_t *pm = const_cast<uint32_t *>(perm);  // read only (PACKED = false)
  if (coder == HUSKY_CODER_ASCII) {
    static SmemAttr attr;
    attr.ensure(k_gather<HUSKY_CODER_ASCII, false, false, true>, kSmem);
    k_gather<HUSKY_CODER_ASCII, false, false, true><<<g, b, kSmem, s>>>(
        pm, n, units, offsets, nullptr, nullptr, lb, tile_counter, epoch, nullptr, 0, nullptr, nullptr, GatherRuns{},
        d_table, nullptr);
  } else {
    static SmemAttr attr;
    attr.ensure(k_gather<HUSKY_CODER_UNICODE, false, false, true>, kSmem);
    k_gather<HUSKY_CODER_UNICODE, false, false, true><<<g, b, kSmem, s>>>(
        pm, n, units, offsets, nullptr, nullptr, lb, tile_counter, epoch, nullptr, 0, nullptr, nullptr, GatherRuns{},
        d_table, nullptr);
  }
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
// are unchanged; only the order inside moves).  Small runs: a lane each when
// they hold <= kTinyMax strings, else a warp (lane per string); medium runs:
// a CTA each.  (One CTA per two-string run left 255 of 256 threads idle: 7.3 ms
// for the ~10^6 such runs of a 2^30 partial key sort.)  skip_staged (the main
// pass): runs fix_tiny already wrote back and medium runs k_fix_staged sorted
// in place are skipped.

template <int CODER>
__global__ void __launch_bounds__(256)
    k_regather_runs(const uint2 *__restrict__ list, uint64_t cap, const DevState *st,
                    const uint32_t *__restrict__ perm, const void *__restrict__ units,
                    const int64_t *__restrict__ offsets, void *__restrict__ sorted_units,
                    int64_t *__restrict__ sorted_offsets, uint32_t first_small, uint32_t first_medium,
                    int skip_staged) {
  constexpr int W = CoderTraits<CODER>::kUnitBytes;
  __shared__ unsigned long long s_wt[256 / 32 + 1];
  pdl_wait();
  if (st->violations & kOffsetsBad) return;
  // entries [first_small, n_small) of the small list, then [first_medium, n_medium) of the medium list
  const uint32_t ns = st->n_small - first_small, nm = st->n_medium - first_medium;
  const uint8_t *ub = (const uint8_t *)units;
  uint8_t *ob = (uint8_t *)sorted_units;
  const uint32_t lane = lane_id();
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t b = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; b < ns; b += nw * 32) {
    const uint2 mine = b + lane < ns ? list[first_small + b + lane] : make_uint2(0, 0);
    if (mine.y <= kTinyMax && !skip_staged) {  // (main pass: fix_tiny wrote them)
      uint64_t d = mine.y ? (uint64_t)sorted_offsets[mine.x] : 0;
      for (uint32_t k = 0; k < mine.y; ++k) {
        const uint32_t i = perm[mine.x + k];
        const int64_t o = offsets[i];
        const uint64_t L = (uint64_t)(offsets[i + 1] - o);
        sorted_offsets[mine.x + k] = (int64_t)d;
        HCHK(kChkRegather, (d + L) * W, st->chk_units + 1);
        copy_units<W>(ub, o, ob, d, L);
        d += L;
      }
    }
    uint32_t big = __ballot_sync(0xFFFFFFFFu, mine.y > kTinyMax);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const uint32_t start = __shfl_sync(0xFFFFFFFFu, mine.x, src), len = __shfl_sync(0xFFFFFFFFu, mine.y, src);
      const bool valid = lane < len;
      const uint32_t i = valid ? perm[start + lane] : 0u;
      const int64_t o = valid ? offsets[i] : 0;
      const uint64_t L = valid ? (uint64_t)(offsets[i + 1] - o) : 0ull;
      uint64_t ex = L;  // inclusive warp scan of the lengths
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint64_t t = __shfl_up_sync(0xFFFFFFFFu, ex, off);
        if (lane >= (uint32_t)off) ex += t;
      }
      const uint64_t base = (uint64_t)sorted_offsets[start];  // read by every lane before any write
      __syncwarp();
      if (valid) {
        const uint64_t d = base + ex - L;
        sorted_offsets[start + lane] = (int64_t)d;
        copy_units<W>(ub, o, ob, d, L);
      }
      __syncwarp();
    }
  }
  for (uint32_t e = blockIdx.x; e < nm; e += gridDim.x) {
    uint2 ent = list[cap - 1 - (first_medium + e)];
    const uint32_t start = ent.x, len = ent.y & ~kRunDone;
    // medium runs k_fix_staged sorted and wrote back in place (fixup.cu)
    if (skip_staged && st->trivial_mask != 0xFFu &&
        (uint64_t)(sorted_offsets[start + len] - sorted_offsets[start]) * W <= (uint64_t)kFixStageBytes)
      continue;
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
        copy_units<W>(ub, o, ob, d, L);
      }
      running += tot;
      __syncthreads();
    }
  }
}

void launch_regather_runs(int coder, const uint2 *list_sm, uint64_t cap_sm, const DevState *st,
                          const uint32_t *perm, const void *units, const int64_t *offsets,
                          void *sorted_units, int64_t *sorted_offsets, int num_sms, cudaStream_t s,
                          uint32_t first_small, uint32_t first_medium, bool skip_staged) {
  Scope sc_(ST_FIX_SMALL, s, 0);
  dim3 g(num_sms * 4), b(256);
  if (coder == HUSKY_CODER_ASCII)
    launch_pdl(k_regather_runs<HUSKY_CODER_ASCII>, g, b, 0, s, list_sm, cap_sm, st, (const uint32_t *)perm, units,
               offsets, sorted_units, sorted_offsets, first_small, first_medium, skip_staged ? 1 : 0);
  else
    launch_pdl(k_regather_runs<HUSKY_CODER_UNICODE>, g, b, 0, s, list_sm, cap_sm, st, (const uint32_t *)perm, units,
               offsets, sorted_units, sorted_offsets, first_small, first_medium, skip_staged ? 1 : 0);
}

}  // namespace husky

extern "C" int husky_debug_gather_times(unsigned long long *out, int max_tiles) {
#ifdef HUSKY_TIMING
  int k = max_tiles < husky::kGTimingTiles ? max_tiles : husky::kGTimingTiles;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, husky::g_gather_times, (size_t)k * 8 * sizeof(unsigned long long));
  return k;
#else
  (void)out;
  (void)max_tiles;
  return 0;
#endif
}
