// runs.cu -- A3: equal-code run detection + order check, and run classification.
//
// After the stable key sort, code(a) < code(b) implies a < b (the husky-code
// contract, holds with p = 0 for the built-in coders on their
// domain: DESIGN.md R6), so every remaining inversion lies inside a contiguous
// run of equal codes.  "After the first pass ... we can easily determine
// whether our encoding was perfect": here that check is done
// per adjacent pair inside runs, with the exact comparator, in one flat
// data-parallel pass; a run is "dirty" iff one of its adjacent pairs is out of
// order (Timsort's natural-run idea).  Only dirty runs reach
// the fix-up (A5) -- the analogue of Alg. 1's cleanup pass.
//
// k_runs_scan is a single-pass scan (decoupled look-back over tiles of 4096
// positions) of the "nontrivial run starts here" flags; the k-th start and the
// k-th end belong to run k.  With sorted outputs the main path does this inside
// the gather (gather.cu, CHECK); this kernel serves the perm-only mode (MODE 0:
// strings through perm -> offsets -> units) and the refinement (MODE 1).
#include "husky_internal.cuh"
#include "kernels.cuh"

namespace husky {

template <int CODER, int MODE>
__global__ void __launch_bounds__(kScanThreads)
    k_runs_scan(const uint64_t *__restrict__ keys, uint64_t n, const uint32_t *__restrict__ perm,
                const void *__restrict__ units, const int64_t *__restrict__ offsets, uint32_t base,
                uint32_t *__restrict__ run_start, uint32_t *__restrict__ run_end, uint8_t *__restrict__ dirty,
                DevState *st, unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch,
                unsigned long long refmask) {
  using T = CoderTraits<CODER>;
  // Tile staging of the keys in smem (coalesced async copies).  Each thread then
  // works on kScanItems consecutive positions; the array is padded (one pad
  // element every 8 u64) so that blocked per-thread reads do not bank-conflict.
  extern __shared__ __align__(16) uint8_t dsm[];  // kScanKP * 8 bytes
  uint64_t *s_keys = reinterpret_cast<uint64_t *>(dsm);  // keys[tile_base - 1 + i]
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_wt[kScanThreads / 32 + 1];
  __shared__ unsigned long long s_excl;
  const uint32_t tid = threadIdx.x;
  if (st->violations & kOffsetsBad) return;  // invalid input: reported by the caller
  if (keys == nullptr) keys = reinterpret_cast<const uint64_t *>(st->sorted_keys);  // device-planned radix
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t tb = (uint64_t)tile * kScanTile;
  const uint64_t p0 = tb + (uint64_t)tid * kScanItems;
  for (uint32_t i = tid; i < kScanTile + 2; i += kScanThreads) {
    int64_t p = (int64_t)tb + (int64_t)i - 1;
    if (p >= 0 && (uint64_t)p < n) cp_async8(&s_keys[i + i / 8], keys + p);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();

  // keys at p0-1 .. p0+kScanItems (MODE 0: under the run rule's mask, R19)
  const RunRule rule = run_rule<CODER>(st);
  // MODE 1: a refinement that left the tag and the window's last units unsorted
  // compares keys under refmask, and every equal pair under it is unresolved
  const unsigned long long km = MODE == 0 ? rule.mask : refmask;
  uint64_t c[kScanItems + 2];
#pragma unroll
  for (int j = 0; j < kScanItems + 2; ++j) {
    int64_t p = (int64_t)p0 + j - 1;
    uint32_t i = tid * kScanItems + j;
    c[j] = (p >= 0 && (uint64_t)p < n) ? (s_keys[i + i / 8] & km) : 0ull;
  }
  uint32_t eqp = 0, eqn = 0, cnt = 0;  // bit j: eq_prev / eq_next of position p0+j
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    uint64_t p = p0 + j;
    bool ep = p < n && p > 0 && c[j + 1] == c[j];
    bool en = p + 1 < n && c[j + 1] == c[j + 2];
    eqp |= (uint32_t)ep << j;
    eqn |= (uint32_t)en << j;
    cnt += (!ep && en);
  }
  uint32_t tile_total;
  uint32_t excl_t = block_exclusive_scan<uint32_t, kScanThreads>(cnt, &tile_total, s_wt);
  if (tid == 0) st_relaxed_u64(lb + tile, make_flag(tile == 0 ? kFlagInc : kFlagAgg, epoch, tile_total));

  // order check of the adjacent pairs inside runs (independent of the look-back)
  uint32_t badm = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    uint64_t p = p0 + j;
    if ((eqn >> j) & 1) {
      bool bad;
      if (MODE == 0) {
        bad = cmp_equal_code<CODER>(units, offsets, __ldg(perm + p), __ldg(perm + p + 1), rule.S, rule.PL) > 0;
      } else {
        constexpr uint64_t tagmask = CODER == HUSKY_CODER_ASCII ? 0xFFull : 0xFFFFull;
        bad = refmask != ~0ull || (c[j + 1] & tagmask) == (uint64_t)(16 + T::kTagCap);
      }
      badm |= (uint32_t)bad << j;
    }
  }

  if ((tid >> 5) == 0) {  // warp-wide look-back: 32 predecessor tiles per round trip
    unsigned long long ex = tile == 0 ? 0ull : warp_lookback(lb, tile, epoch);
    if (lane_id() == 0) {
      if (tile != 0) st_relaxed_u64(lb + tile, make_flag(kFlagInc, epoch, ex + tile_total));
      s_excl = ex;
      if ((uint64_t)(tile + 1) * kScanTile >= n) st->n_runs = (uint32_t)(ex + tile_total);
    }
  }
  __syncthreads();
  if ((eqp | eqn) == 0) return;

  // run id of position p = (# nontrivial starts at or before p) - 1
  uint32_t rid = (uint32_t)s_excl + excl_t - 1;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    bool ep = (eqp >> j) & 1, en = (eqn >> j) & 1;
    uint64_t p = p0 + j;
    if (!ep && en) {
      ++rid;
      run_start[rid] = base + (uint32_t)p;
    }
    if (ep && !en) run_end[rid] = base + (uint32_t)p;
    if ((badm >> j) & 1) dirty[rid] = 1;
  }
}

void launch_runs_scan(int coder, int mode, const uint64_t *keys, uint64_t n, const uint32_t *perm,
                      const void *units, const int64_t *offsets, uint32_t base, uint32_t *run_start,
                      uint32_t *run_end, uint8_t *dirty, DevState *st, unsigned long long *lb,
                      uint32_t *tile_counter, uint32_t epoch, cudaStream_t s, unsigned long long refmask) {
  if (n == 0) return;
  constexpr int kSmem0 = kScanKP * 8;  // the padded key staging
  static SmemAttr a0, a1, a2, a3;
  a0.ensure(k_runs_scan<HUSKY_CODER_ASCII, 0>, kSmem0);
  a1.ensure(k_runs_scan<HUSKY_CODER_ASCII, 1>, kSmem0);
  a2.ensure(k_runs_scan<HUSKY_CODER_UNICODE, 0>, kSmem0);
  a3.ensure(k_runs_scan<HUSKY_CODER_UNICODE, 1>, kSmem0);
  Scope sc_(ST_RUNS_SCAN, s, n);
  dim3 g((unsigned)scan_tiles(n)), b(kScanThreads);
#define RS_ARGS keys, n, perm, units, offsets, base, run_start, run_end, dirty, st, lb, tile_counter, epoch, refmask
  if (coder == HUSKY_CODER_ASCII) {
    if (mode == 0) k_runs_scan<HUSKY_CODER_ASCII, 0><<<g, b, kSmem0, s>>>(RS_ARGS);
    else k_runs_scan<HUSKY_CODER_ASCII, 1><<<g, b, kSmem0, s>>>(RS_ARGS);
  } else {
    if (mode == 0) k_runs_scan<HUSKY_CODER_UNICODE, 0><<<g, b, kSmem0, s>>>(RS_ARGS);
    else k_runs_scan<HUSKY_CODER_UNICODE, 1><<<g, b, kSmem0, s>>>(RS_ARGS);
  }
#undef RS_ARGS
}

// Classification of the runs found by the last scan: statistics, and dirty runs
// appended to the small (front of list_sm), medium (back of list_sm) and giant
// (list_g) lists.  Grid-stride over st->n_runs (read on device, no host sync).
__global__ void __launch_bounds__(256)
    k_runs_classify(const uint32_t *__restrict__ run_start, const uint32_t *__restrict__ run_end,
                    const uint8_t *__restrict__ dirty, DevState *st, uint2 *list_sm, uint64_t cap_sm,
                    uint2 *list_g, int count_stats) {
  __shared__ unsigned long long s_sum[4], s_in, s_max;
  pdl_wait();
  if (threadIdx.x < 4) s_sum[threadIdx.x] = 0;
  if (threadIdx.x == 0) { s_in = 0; s_max = 0; }
  __syncthreads();
  const uint32_t nr = st->n_runs;
  unsigned long long in = 0, mx = 0, cls[4] = {0, 0, 0, 0};
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
    uint32_t s = run_start[r];
    uint32_t len = run_end[r] - s + 1;
    in += len;
    mx = len > mx ? len : mx;
    if (!dirty[r]) { cls[0]++; continue; }
    if (len <= (uint32_t)kSmallMax) {
      cls[1]++;
      uint32_t i = atomicAdd(&st->n_small, 1u);
      list_sm[i] = make_uint2(s, len);
    } else if (len <= (uint32_t)kMediumMax) {
      cls[2]++;
      uint32_t i = atomicAdd(&st->n_medium, 1u);
      list_sm[cap_sm - 1 - i] = make_uint2(s, len);
    } else {
      cls[3]++;
      uint32_t i = atomicAdd(&st->n_giant, 1u);
      list_g[i] = make_uint2(s, len);
    }
  }
  // block-aggregate the statistics, one atomic per block
  for (int o = 16; o > 0; o >>= 1) {
    in += __shfl_xor_sync(0xFFFFFFFFu, in, o);
    unsigned long long m2 = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
    mx = m2 > mx ? m2 : mx;
#pragma unroll
    for (int c = 0; c < 4; ++c) cls[c] += __shfl_xor_sync(0xFFFFFFFFu, cls[c], o);
  }
  if (lane_id() == 0) {
    atomicAdd(&s_in, in);
    atomicMax(&s_max, mx);
    for (int c = 0; c < 4; ++c) atomicAdd(&s_sum[c], cls[c]);
  }
  __syncthreads();
  if (threadIdx.x == 0 && count_stats) {
    if (blockIdx.x == 0) st->runs_total = nr;
    for (int c = 0; c < 4; ++c)
      if (s_sum[c]) atomicAdd(&st->runs_by_class[c], s_sum[c]);
    {
      if (s_in) atomicAdd(&st->n_in_runs, s_in);
      if (s_max) atomicMax(&st->max_run, s_max);
    }
  }
}

void launch_runs_classify(const uint32_t *run_start, const uint32_t *run_end, const uint8_t *dirty,
                          DevState *st, uint2 *list_sm, uint64_t cap_sm, uint2 *list_g,
                          bool count_stats, int num_sms, cudaStream_t s) {
  Scope sc_(ST_CLASSIFY, s, 0);
  launch_pdl(k_runs_classify, dim3(num_sms * 2), dim3(256), 0, s, run_start, run_end, dirty, st, list_sm, cap_sm,
             list_g, count_stats ? 1 : 0);
}

}  // namespace husky
