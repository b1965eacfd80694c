// multi.cu -- E: the hot path sharded as a sample sort over P GPUs (one process
// per GPU, NCCL over NVLink 5 / NVSwitch), plus a single-GPU "loopback" driver
// that runs P virtual ranks through the very same phases with device-to-device
// copies as the transport (used to test the sharded path on one GPU).
//
// Not in the paper (single-threaded Java).  Splitters are
// STRINGS (composite splitters): a splitter is
// the prefix (<= kPrefixUnits units) of a sampled string, and bucket(x) =
// #splitters <= x in the sort order itself (code first -- the code is a
// function of the prefix, PAPER.md:195-211 -- then the units).  Equal-code runs
// may therefore straddle ranks (an all-colliding input like C4 spreads over all
// GPUs), while equal STRINGS never do, and the concatenation of the locally
// sorted buckets is the global order.  Phases:
//   1. encode the local strings (A1); take s regular samples: code + prefix;
//      all-gather the P*s samples (+ each rank's input-violation word);
//   2. every rank sorts the gathered sample prefixes on the GPU (husky_sort of
//      the samples) and picks the same P-1 splitters (the rule of
//      husky_select_splitters); bucket(x) = #splitters <= x (binary search,
//      strings compared only on code ties); per-destination string/unit
//      counts; all-gather of the P x P count matrix;
//   3. stable partition by bucket = one onesweep pass on the bucket digit, then
//      the exchange, one of:
//      * peer stores (default, NEXT-2): the A4 gather writes every string's
//        units, length and global index straight into its destination rank's
//        receive window -- an NCCL symmetric window (ncclMemAlloc +
//        ncclCommWindowRegister) whose peer mappings (ncclGetPeerPointer) are
//        NVLink / NVSwitch load-store addresses -- at the rank's displacement
//        in that window (from the count matrix); one 4-byte all-reduce then
//        orders the stores before any rank reads its window;
//      * HUSKY_EXCHANGE=nccl (or a failed window registration): the gather
//        builds send buffers, then grouped ncclSend/ncclRecv of the three arrays;
//   4. lengths -> offsets scan, the single-GPU husky_sort on the received bucket
//      (received order = ascending global index, so the index tie-break holds),
//      perm remapped to global indices.
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cstdio>
#include <cstring>
#include <vector>

#include "host_common.h"

namespace husky {

constexpr int kSamplesPerRank = 4096;
constexpr int kMaxWorld = 256;  // bucket ids must fit one radix digit
constexpr int kSampleStride = kSamplesPerRank + 1;  // + the rank's violation word
// A sample / splitter string: its code, its length capped at kPrefixUnits and
// the first kPrefixUnits units (zero-filled).  Equal prefixes cannot be split,
// so only strings sharing a 32-unit prefix are kept on one rank.
constexpr int kPrefixUnits = 32;
struct SampleRec {
  uint64_t code;
  uint32_t len;  // min(length, kPrefixUnits); 0xFFFFFFFF: no sample (empty rank)
  uint32_t pad;
  uint8_t u[kPrefixUnits * 2];
};
static_assert(sizeof(SampleRec) == 80, "SampleRec layout");

#define HCHECK(expr)                                                                               \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) return fail(HUSKY_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_));   \
  } while (0)
#define NCHECK(expr)                                                                               \
  do {                                                                                             \
    ncclResult_t r_ = (expr);                                                                      \
    if (r_ != ncclSuccess) return fail(HUSKY_ERR_NCCL, "%s: %s", #expr, ncclGetErrorString(r_));   \
  } while (0)

// ------------------------------------------------------------------ kernels
__global__ void k_sample(const uint64_t *__restrict__ codes, uint64_t n, uint64_t *__restrict__ out,
                         const DevState *st) {
  for (int i = threadIdx.x; i < kSamplesPerRank; i += blockDim.x)
    out[i] = n ? codes[(uint64_t)i * n / kSamplesPerRank] : ~0ull;  // ~0: "no sample" (codes < 2^63)
  if (threadIdx.x == 0) out[kSamplesPerRank] = st->violations;
}

// the sample records of one rank: s regular samples (positions i*n/s)
template <int W>
__global__ void k_sample_str(const uint64_t *__restrict__ codes, uint64_t n, const void *__restrict__ units,
                             const int64_t *__restrict__ offsets, SampleRec *__restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kSamplesPerRank; i += gridDim.x * blockDim.x) {
    SampleRec r;
    memset(&r, 0, sizeof r);
    if (n == 0) {
      r.len = 0xFFFFFFFFu;
    } else {
      const uint64_t p = (uint64_t)i * n / kSamplesPerRank;
      const int64_t o = offsets[p], L = offsets[p + 1] - o;
      const uint32_t m = (uint32_t)(L < kPrefixUnits ? L : kPrefixUnits);
      r.code = codes[p];
      r.len = m;
      const uint8_t *src = (const uint8_t *)units + o * W;
      for (uint32_t b = 0; b < m * W; ++b) r.u[b] = src[b];
    }
    out[i] = r;
  }
}

// gathered records of the non-empty ranks -> a string array (units + offsets)
// for the GPU sort of the samples: lengths first (scanned by k_lens_to_offsets),
// then the units at their offsets
__device__ __forceinline__ const SampleRec &sample_rec(const SampleRec *recs, const int *ranks, uint64_t i) {
  return recs[(uint64_t)ranks[i / kSamplesPerRank] * kSamplesPerRank + i % kSamplesPerRank];
}
__global__ void k_sample_lens(const SampleRec *__restrict__ recs, const int *__restrict__ ranks, uint64_t m,
                              uint32_t *__restrict__ lens) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    lens[i] = sample_rec(recs, ranks, i).len;
}
template <int W>
__global__ void k_sample_units(const SampleRec *__restrict__ recs, const int *__restrict__ ranks, uint64_t m,
                               const int64_t *__restrict__ so, uint8_t *__restrict__ su) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const SampleRec &r = sample_rec(recs, ranks, i);
    for (uint32_t b = 0; b < r.len * W; ++b) su[so[i] * W + b] = r.u[b];
  }
}

// splitter k (1..P-1) = the sample at sorted position floor(k*m/P)
__global__ void k_pick_splitters(const SampleRec *__restrict__ recs, const int *__restrict__ ranks, uint64_t m,
                                 const uint32_t *__restrict__ sorted, int world, SampleRec *__restrict__ split) {
  for (int k = 1 + threadIdx.x; k < world; k += blockDim.x) {
    split[k - 1] = sample_rec(recs, ranks, sorted[(uint64_t)((unsigned __int128)k * m / world)]);
  }
}

// x (code c, units xs[0..xl)) >= splitter?  Code first; on a code tie the units
// (unsigned, position by position), then the shorter string first.
template <int W>
__device__ __forceinline__ bool ge_splitter(uint64_t c, const uint8_t *xs, int64_t xl, const SampleRec &sp,
                                            bool general) {
  if (!general && c != sp.code) return c > sp.code;
  const int64_t m = xl < (int64_t)sp.len ? xl : (int64_t)sp.len;
  for (int64_t k = 0; k < m; ++k) {
    uint32_t a, b;
    if (W == 1) { a = xs[k]; b = sp.u[k]; }
    else { a = ((const uint16_t *)xs)[k]; b = ((const uint16_t *)sp.u)[k]; }
    if (a != b) return a > b;
  }
  return xl >= (int64_t)sp.len;
}

template <int W>
__global__ void __launch_bounds__(256)
    k_bucket(const uint64_t *__restrict__ codes, uint64_t n, const SampleRec *__restrict__ splitters,
             int nsplit, int world, const void *__restrict__ units, const int64_t *__restrict__ offsets,
             uint64_t *__restrict__ keys, DevState *st, unsigned long long *counts, int general) {
  __shared__ SampleRec s_split[kMaxWorld - 1];
  __shared__ unsigned long long s_cnt[kMaxWorld], s_units[kMaxWorld];
  for (int i = threadIdx.x; i < nsplit; i += blockDim.x) s_split[i] = splitters[i];
  for (int i = threadIdx.x; i < kMaxWorld; i += blockDim.x) {
    s_cnt[i] = 0;
    s_units[i] = 0;
  }
  __syncthreads();
  // counts are aggregated per warp when the warp's strings share one bucket
  // (P = 1, sorted or skewed input): per-lane atomics on one shared address
  // serialise (0.9 ms for 1e7 strings at P = 1)
  const uint32_t lane = lane_id();
  // kBucketIT strings per thread per round, their loads issued together (one
  // string per thread per round left the kernel latency-bound: 87 us for 1e7)
  constexpr int kBucketIT = 4;
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x * kBucketIT;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * kBucketIT; base < n; base += step) {
    uint64_t cc[kBucketIT];
    int64_t oo[kBucketIT], oe[kBucketIT];
#pragma unroll
    for (int k = 0; k < kBucketIT; ++k) {
      const uint64_t i = base + threadIdx.x + (uint64_t)k * blockDim.x;
      cc[k] = i < n ? codes[i] : 0ull;
      oo[k] = i < n ? offsets[i] : 0;
      oe[k] = i < n ? offsets[i + 1] : 0;
    }
#pragma unroll
    for (int k = 0; k < kBucketIT; ++k) {
      const uint64_t i = base + threadIdx.x + (uint64_t)k * blockDim.x;
      const bool valid = i < n;
      uint32_t b = 0xFFFFFFFFu;
      const unsigned long long L = valid ? (unsigned long long)(oe[k] - oo[k]) : 0ull;
      if (valid) {
        const uint8_t *xs = (const uint8_t *)units + oo[k] * W;
        int lo = 0, hi = nsplit;  // number of splitters <= x
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (ge_splitter<W>(cc[k], xs, (int64_t)L, s_split[mid], general != 0)) lo = mid + 1;
          else hi = mid;
        }
        b = (uint32_t)lo;
        keys[i] = (uint64_t)lo;
      }
      const uint32_t b0 = __shfl_sync(0xFFFFFFFFu, b, 0);
      if (__all_sync(0xFFFFFFFFu, b == b0 || !valid)) {
        unsigned long long sum = L;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
        const uint32_t nv = __popc(__ballot_sync(0xFFFFFFFFu, valid));
        if (lane == 0 && nv) {
          atomicAdd(&s_cnt[b0], (unsigned long long)nv);
          atomicAdd(&s_units[b0], sum);
        }
      } else if (valid) {  // several buckets: few lanes share an address
        atomicAdd(&s_cnt[b], 1ull);
        atomicAdd(&s_units[b], L);
      }
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < world; b += blockDim.x) {
    if (s_cnt[b]) {
      atomicAdd(&counts[2 * b], s_cnt[b]);
      atomicAdd(&counts[2 * b + 1], s_units[b]);
      atomicAdd(&st->hist[0][b], (uint32_t)s_cnt[b]);
    }
  }
}

__global__ void k_send_meta(const uint32_t *__restrict__ send_perm, uint64_t n, const int64_t *__restrict__ offsets,
                            uint32_t gbase, uint32_t *__restrict__ gidx, uint32_t *__restrict__ lens) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t p = send_perm[j];
    gidx[j] = gbase + p;
    lens[j] = (uint32_t)(offsets[p + 1] - offsets[p]);
  }
}

// exclusive scan of u32 lengths -> int64 offsets[n+1] (single pass, look-back)
__global__ void __launch_bounds__(kScanThreads)
    k_lens_to_offsets(const uint32_t *__restrict__ lens, uint64_t n, int64_t *__restrict__ offsets,
                      unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, int64_t add) {
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_wt[kScanThreads / 32 + 1];
  __shared__ unsigned long long s_base;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t p0 = (uint64_t)tile * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  unsigned long long v[kScanItems], sum = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    v[j] = p0 + j < n ? lens[p0 + j] : 0;
    sum += v[j];
  }
  unsigned long long tot;
  unsigned long long ex = block_exclusive_scan<unsigned long long, kScanThreads>(sum, &tot, s_wt);
  if (threadIdx.x == 0) st_relaxed_u64(lb + tile, make_flag(tile == 0 ? kFlagInc : kFlagAgg, epoch, tot));
  if (threadIdx.x < 32) {  // warp-wide look-back: 32 predecessors per round trip
    const unsigned long long b = tile == 0 ? 0ull : warp_lookback(lb, tile, epoch);
    if (threadIdx.x == 0) {
      if (tile != 0) st_relaxed_u64(lb + tile, make_flag(kFlagInc, epoch, b + tot));
      s_base = b;
      if ((uint64_t)(tile + 1) * kScanTile >= n) offsets[n] = (int64_t)(b + tot) + add;
    }
  }
  __syncthreads();
  unsigned long long d = s_base + ex;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    if (p0 + j < n) offsets[p0 + j] = (int64_t)d + add;
    d += v[j];
  }
}

__global__ void k_remap(uint32_t *perm, uint64_t n, const uint32_t *__restrict__ gidx) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    perm[i] = gidx[perm[i]];
}

__global__ void k_add_base(int64_t *o, uint64_t n, int64_t add) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    o[i] += add;
}

// peer base addresses of a symmetric window (NVLink load/store mappings)
__global__ void k_win_ptrs(ncclWindow_t w, int world, unsigned long long *out) {
  for (int p = threadIdx.x; p < world; p += blockDim.x) out[p] = (unsigned long long)ncclGetPeerPointer(w, 0, p);
}

static unsigned grid_for(uint64_t n) {
  uint64_t b = (n + 255) / 256;
  return (unsigned)(b < 1 ? 1 : (b > 4096 ? 4096 : b));
}

// ------------------------------------------------------------------ host side
// HUSKY_MULTI_TIMING=1: synchronise after each phase and print its wall time
// (diagnostics only; changes the overlap it measures)
struct PhaseClock {
  cudaStream_t s;
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit PhaseClock(cudaStream_t st) : s(st) {
    const char *v = getenv("HUSKY_MULTI_TIMING");
    on = v && v[0] == '1';
    if (on) { cudaStreamSynchronize(s); t = std::chrono::steady_clock::now(); }
  }
  void mark(const char *name) {
    if (!on) return;
    cudaStreamSynchronize(s);
    auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[husky multi] %-24s %8.1f us\n", name, std::chrono::duration<double, std::micro>(n - t).count());
    t = n;
  }
};
static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Comm {
  ncclComm_t nccl = nullptr;
  int rank = 0, world = 1;
  // receive window for the peer-store exchange (grown collectively on demand)
  void *win_buf = nullptr;
  size_t win_bytes = 0;
  ncclWindow_t win = nullptr;
  bool win_failed = false;                // registration failed on some rank: NCCL send/recv
  std::vector<unsigned long long> peer;   // peer base address of the window, per rank
  unsigned long long *d_tmp = nullptr;    // world words (peer addresses, barrier word)
  bool aborted = false;                   // ncclCommAbort ran: every later call fails fast
};

// Waits for `s` while watching the communicator: an asynchronous NCCL error
// (a peer died, a network fault) or no progress within HUSKY_NCCL_TIMEOUT_S
// seconds (default 600) aborts the communicator and returns HUSKY_ERR_NCCL
// instead of hanging every rank (failure detection).
// c == NULL (loopback driver): a plain synchronisation.
static double nccl_timeout_s() {
  static const double t = [] {
    const char *v = getenv("HUSKY_NCCL_TIMEOUT_S");
    return v ? atof(v) : 600.0;
  }();
  return t;
}

static husky_status comm_sync(Comm *c, cudaStream_t s) {
  if (!c) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(HUSKY_ERR_CUDA, "cudaStreamSynchronize: %s", cudaGetErrorString(e));
    return HUSKY_OK;
  }
  if (c->aborted) return fail(HUSKY_ERR_NCCL, "communicator was aborted by an earlier failure");
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t it = 0;; ++it) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) return HUSKY_OK;
    if (e != cudaErrorNotReady) return fail(HUSKY_ERR_CUDA, "stream: %s", cudaGetErrorString(e));
    ncclResult_t ae = ncclSuccess;
    ncclCommGetAsyncError(c->nccl, &ae);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if ((ae != ncclSuccess && ae != ncclInProgress) || el > nccl_timeout_s()) {
      ncclCommAbort(c->nccl);
      c->aborted = true;
      if (ae != ncclSuccess && ae != ncclInProgress)
        return fail(HUSKY_ERR_NCCL, "NCCL asynchronous error: %s (communicator aborted)", ncclGetErrorString(ae));
      return fail(HUSKY_ERR_NCCL, "no progress for %.0f s (HUSKY_NCCL_TIMEOUT_S): communicator aborted", el);
    }
    if (it > 2000) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// Where a rank receives: units at 0, lengths and global indices after them.
// Window offsets are the same on every rank (sized by the largest shard).
struct WinLayout {
  size_t units = 0, lens = 0, gidx = 0, total = 0;
};
static WinLayout make_win_layout(size_t w, uint64_t cap_n, uint64_t cap_u) {
  WinLayout W;
  W.units = 0;
  W.lens = align_up(cap_u * w + 16, 256);
  W.gidx = W.lens + align_up(cap_n * 4 + 4, 256);
  W.total = W.gidx + align_up(cap_n * 4 + 4, 256);
  return W;
}

static bool exchange_by_nccl() {
  const char *v = getenv("HUSKY_EXCHANGE");
  return v && (v[0] == 'n' || v[0] == 'c');  // "nccl" / "copy" (loopback)
}

struct MultiLayout {
  Layout L;  // state, keysA (= codes), keysB, vals, lb_radix, lb_scan used by the Sorter
  size_t send_perm = 0, samples = 0, splitters = 0, counts = 0, rcounts = 0, send_units = 0,
         send_offsets = 0, send_gidx = 0, send_lens = 0, peer_table = 0, total = 0;
  // composite splitters: gathered sample records, their packed strings, the
  // GPU sort of the samples (perm + workspace), the non-empty rank list
  size_t recs = 0, smp_units = 0, smp_offsets = 0, smp_lens = 0, smp_lb = 0, smp_perm = 0, smp_ws = 0, ranks = 0;
};

static MultiLayout make_multi_layout(int coder, uint64_t n, uint64_t units, int world) {
  MultiLayout M;
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off = align_up(off + b, 256); return o; };
  size_t w = coder_unit_bytes(coder);
  Layout &L = M.L;
  L.n = n;
  L.tiles_r = radix_tiles(n);
  L.tiles_s = std::max(scan_tiles(n), gather_tiles(n));
  L.state = take(sizeof(DevState));
  L.keysA = take(n * 8 + 8);
  L.keysB = take(n * 8 + 8);
  L.vals = take(n * 4 + 4);
  L.lb_radix_words = radix_lb_words(n);
  L.lb_radix = take(L.lb_radix_words * 8);
  L.lb_scan = take(L.tiles_s * 16 + 8);  // Sorter::reset_lookback clears two arrays
  M.send_perm = take(n * 4 + 4);
  M.samples = take((size_t)world * kSampleStride * 8);
  M.splitters = take((size_t)world * sizeof(SampleRec));
  const uint64_t ms = (uint64_t)world * kSamplesPerRank;
  M.recs = take(ms * sizeof(SampleRec));
  M.smp_units = take(ms * kPrefixUnits * w + 16);
  M.smp_offsets = take((ms + 1) * 8);
  M.smp_lens = take(ms * 4);
  M.smp_lb = take(scan_tiles(ms) * 8 + 8);
  M.smp_perm = take(ms * 4 + 4);
  M.smp_ws = take(make_layout(ms).total);
  M.ranks = take((size_t)world * 4);
  M.counts = take((size_t)world * 16);
  M.rcounts = take((size_t)world * world * 16);  // the all-gathered count matrix [src][dst]
  M.peer_table = take(sizeof(PeerTable));
  M.send_units = take(units * w + 16);
  M.send_offsets = take((n + 1) * 8);
  M.send_gidx = take(n * 4 + 4);
  M.send_lens = take(n * 4 + 4);
  M.total = off;
  L.total = off;
  return M;
}

struct RecvLayout {
  size_t units = 0, offsets = 0, lens = 0, gidx = 0, lb = 0, sort_ws = 0, total = 0;
};
// data = false: the received arrays live in the peer-store window instead
static RecvLayout make_recv_layout(int coder, uint64_t n_out, uint64_t units_out, bool data = true) {
  RecvLayout R;
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off = align_up(off + b, 256); return o; };
  size_t w = coder_unit_bytes(coder);
  R.units = take(data ? units_out * w + 16 : 0);
  R.offsets = take((n_out + 1) * 8);
  R.lens = take(data ? n_out * 4 + 4 : 0);
  R.gidx = take(data ? n_out * 4 + 4 : 0);
  R.lb = take(scan_tiles(n_out) * 8 + 8);
  R.sort_ws = take(make_layout(n_out).total);
  R.total = off;
  return R;
}

// One rank's state across the phases (a plan).
struct Plan {
  Comm *comm = nullptr;  // null in loopback mode
  int coder = 0, rank = 0, world = 1;
  const void *units = nullptr;
  const int64_t *offsets = nullptr;
  uint64_t n = 0, gbase = 0, local_units = 0;
  uint8_t *ws = nullptr;
  MultiLayout M;
  cudaStream_t s = nullptr;
  Sorter S;
  std::vector<uint64_t> send_cnt, send_u, recv_cnt, recv_u;  // per peer
  std::vector<uint64_t> disp_n, disp_u;  // this rank's offset in each destination's received arrays
  uint64_t n_out = 0, units_out = 0;
  uint64_t cap_n = 0, cap_u = 0;  // the largest shard (strings, units): sizes the receive windows
  bool general = false;  // some rank saw off-domain units (readings R5, R15)
  bool peer = false;     // exchange by peer stores into the receive windows (NEXT-2)
  PeerTable table;

  template <typename T> T *at(size_t o) const { return reinterpret_cast<T *>(ws + o); }
  DevState *st() const { return at<DevState>(M.L.state); }
  size_t w() const { return coder_unit_bytes(coder); }

  void init_sorter() {
    S.coder = coder;
    S.units = units;
    S.offsets = offsets;
    S.n = n;
    S.ws = ws;
    S.L = M.L;
    S.s = s;
    S.sms = device_sm_count();
    S.st = st();
    S.perm = at<uint32_t>(M.send_perm);
  }

  // phase 1: encode + regular sample (+ violation word) into samples[rank]
  husky_status phase1() {
    init_sorter();
    HCHECK(cudaMemsetAsync(st(), 0, sizeof(DevState), s));
    HCHECK(S.reset_lookback());
    launch_encode(coder, units, offsets, n, at<uint64_t>(M.L.keysA), &st()->violations, S.sms, s);
    HUSKY_SCOPE(ST_MULTI, s, 0);
    k_sample<<<1, 256, 0, s>>>(at<uint64_t>(M.L.keysA), n, at<uint64_t>(M.samples) + (size_t)rank * kSampleStride,
                               st());
    SampleRec *mine = at<SampleRec>(M.recs) + (size_t)rank * kSamplesPerRank;
    if (w() == 1) k_sample_str<1><<<16, 256, 0, s>>>(at<uint64_t>(M.L.keysA), n, units, offsets, mine);
    else k_sample_str<2><<<16, 256, 0, s>>>(at<uint64_t>(M.L.keysA), n, units, offsets, mine);
    HCHECK(cudaGetLastError());
    return HUSKY_OK;
  }

  // after the samples are gathered: splitters, then bucket + counts (phase 2)
  husky_status choose_splitters() {
    std::vector<uint64_t> all((size_t)world * kSampleStride);
    HCHECK(cudaMemcpyAsync(all.data(), at<uint64_t>(M.samples), all.size() * 8, cudaMemcpyDeviceToHost, s));
    if (husky_status e = comm_sync(comm, s)) return e;
    uint32_t viol = 0;
    std::vector<int> ranks;  // ranks with strings (a rank's samples are all valid or all absent)
    for (int r = 0; r < world; ++r) {
      viol |= (uint32_t)all[(size_t)r * kSampleStride + kSamplesPerRank];
      if (all[(size_t)r * kSampleStride] != ~0ull) ranks.push_back(r);
    }
    if (viol & kOffsetsBad) return fail(HUSKY_ERR_INVALID_ARG, "offsets are not non-decreasing (some rank)");
    // off-domain input somewhere: codes are not monotone, so buckets compare the
    // strings alone (and every rank's local sort runs the general cleanup)
    general = domain_violation(coder, viol);
    if (world == 1) return HUSKY_OK;
    SampleRec *split = at<SampleRec>(M.splitters);
    const uint64_t m = (uint64_t)ranks.size() * kSamplesPerRank;
    if (m == 0) {  // no strings anywhere: any splitters
      HCHECK(cudaMemsetAsync(split, 0, (size_t)(world - 1) * sizeof(SampleRec), s));
      return HUSKY_OK;
    }
    // the same rule as husky_select_splitters, on the GPU: sort the gathered
    // sample prefixes (index order = rank-major, the host rule's input order)
    // and take positions floor(k*m/P)
    HCHECK(cudaMemcpyAsync(at<int>(M.ranks), ranks.data(), ranks.size() * 4, cudaMemcpyHostToDevice, s));
    const SampleRec *recs = at<SampleRec>(M.recs);
    const int *rk = at<int>(M.ranks);
    const unsigned g = grid_for(m);
    {
      HUSKY_SCOPE(ST_MULTI, s, 0);
      k_sample_lens<<<g, 256, 0, s>>>(recs, rk, m, at<uint32_t>(M.smp_lens));
      HCHECK(cudaMemsetAsync(at<uint8_t>(M.smp_lb), 0, scan_tiles(m) * 8 + 8, s));
      HCHECK(cudaMemsetAsync(&st()->tile_counter[61], 0, 4, s));
      k_lens_to_offsets<<<(unsigned)scan_tiles(m), kScanThreads, 0, s>>>(
          at<uint32_t>(M.smp_lens), m, at<int64_t>(M.smp_offsets), at<unsigned long long>(M.smp_lb),
          &st()->tile_counter[61], 1, 0);
      if (w() == 1)
        k_sample_units<1><<<g, 256, 0, s>>>(recs, rk, m, at<int64_t>(M.smp_offsets), at<uint8_t>(M.smp_units));
      else
        k_sample_units<2><<<g, 256, 0, s>>>(recs, rk, m, at<int64_t>(M.smp_offsets), at<uint8_t>(M.smp_units));
      HCHECK(cudaGetLastError());
    }
    if (husky_status e = sort_impl(coder, at<void>(M.smp_units), at<int64_t>(M.smp_offsets), m,
                                   at<uint32_t>(M.smp_perm), nullptr, nullptr, at<void>(M.smp_ws),
                                   make_layout(m).total, nullptr, s, false))
      return e;
    HUSKY_SCOPE(ST_MULTI, s, 0);
    k_pick_splitters<<<1, 256, 0, s>>>(recs, rk, m, at<uint32_t>(M.smp_perm), world, split);
    HCHECK(cudaGetLastError());
    return HUSKY_OK;
  }

  husky_status phase2() {
    HCHECK(cudaMemsetAsync(at<uint8_t>(M.counts), 0, (size_t)world * 16, s));
    HCHECK(cudaMemsetAsync(st()->hist, 0, sizeof(st()->hist), s));
    if (n) {
      unsigned blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)S.sms * 4);
      HUSKY_SCOPE(ST_MULTI, s, 0);
      if (w() == 1)
        k_bucket<1><<<blocks, 256, 0, s>>>(at<uint64_t>(M.L.keysA), n, at<SampleRec>(M.splitters), world - 1, world,
                                           units, offsets, at<uint64_t>(M.L.keysB), st(),
                                           at<unsigned long long>(M.counts), general ? 1 : 0);
      else
        k_bucket<2><<<blocks, 256, 0, s>>>(at<uint64_t>(M.L.keysA), n, at<SampleRec>(M.splitters), world - 1, world,
                                           units, offsets, at<uint64_t>(M.L.keysB), st(),
                                           at<unsigned long long>(M.counts), general ? 1 : 0);
      launch_hist_scan(n, st(), s);
      HCHECK(cudaGetLastError());
    }
    return HUSKY_OK;
  }

  // counts[p] = (strings, units) this rank sends to p; rcounts = the all-gathered
  // matrix, row q = rank q's counts
  husky_status read_counts() {
    std::vector<uint64_t> c((size_t)world * 2), mat((size_t)world * world * 2);
    HCHECK(cudaMemcpyAsync(c.data(), at<uint64_t>(M.counts), c.size() * 8, cudaMemcpyDeviceToHost, s));
    HCHECK(cudaMemcpyAsync(mat.data(), at<uint64_t>(M.rcounts), mat.size() * 8, cudaMemcpyDeviceToHost, s));
    if (husky_status e = comm_sync(comm, s)) return e;
    send_cnt.assign(world, 0); send_u.assign(world, 0); recv_cnt.assign(world, 0); recv_u.assign(world, 0);
    disp_n.assign(world, 0); disp_u.assign(world, 0);
    n_out = units_out = cap_n = cap_u = 0;
    auto m = [&](int q, int p, int k) { return mat[((size_t)q * world + p) * 2 + k]; };
    for (int p = 0; p < world; ++p) {
      send_cnt[p] = c[2 * p]; send_u[p] = c[2 * p + 1];
      recv_cnt[p] = m(p, rank, 0); recv_u[p] = m(p, rank, 1);
      n_out += recv_cnt[p];
      units_out += recv_u[p];
      uint64_t tn = 0, tu = 0;
      for (int q = 0; q < world; ++q) {
        if (q == rank) { disp_n[p] = tn; disp_u[p] = tu; }
        tn += m(q, p, 0);
        tu += m(q, p, 1);
      }
      cap_n = std::max(cap_n, tn);
      cap_u = std::max(cap_u, tu);
    }
    return HUSKY_OK;
  }

  // phase 3a: stable partition by bucket (one onesweep pass on the bucket digit)
  husky_status partition() {
    if (n == 0) return HUSKY_OK;
    // every string to one destination: the stable partition is the identity
    if (std::count_if(send_cnt.begin(), send_cnt.end(), [](uint64_t c) { return c != 0; }) <= 1) {
      launch_iota(at<uint32_t>(M.send_perm), n, s);
      HCHECK(cudaGetLastError());
      return HUSKY_OK;
    }
    uint64_t *sorted_keys = nullptr;
    // bucket ids only occupy digit 0
    return S.radix(at<uint64_t>(M.L.keysB), nullptr, n, 0xFEu, at<uint32_t>(M.send_perm), at<uint32_t>(M.L.vals),
                   &sorted_keys);
  }

  // phase 3b (NCCL exchange): send buffers -- units, lengths, global indices
  husky_status build_send() {
    if (n == 0) return HUSKY_OK;
    HUSKY_SCOPE(ST_MULTI, s, 0);
    k_send_meta<<<grid_for(n), 256, 0, s>>>(at<uint32_t>(M.send_perm), n, offsets, (uint32_t)gbase,
                                            at<uint32_t>(M.send_gidx), at<uint32_t>(M.send_lens));
    launch_gather(kernel_coder(coder), at<uint32_t>(M.send_perm), n, units, offsets, at<void>(M.send_units),
                  at<int64_t>(M.send_offsets), S.lb_scan(), S.next_counter(), S.next_epoch(), s);
    HCHECK(cudaGetLastError());
    return HUSKY_OK;
  }

  // phase 3b (peer stores): the gather writes each bucket straight into its
  // destination's window; du / dl / dg [p] = addresses of rank p's received
  // units / lengths / global indices (its NVLink mapping, or a loopback region)
  husky_status scatter_peer(const std::vector<unsigned long long> &du, const std::vector<unsigned long long> &dl,
                            const std::vector<unsigned long long> &dg) {
    if (n == 0) return HUSKY_OK;
    table.world = (uint32_t)world;
    table.gbase = (uint32_t)gbase;
    table.start_n[0] = table.start_u[0] = 0;
    for (int p = 0; p < world; ++p) {
      table.start_n[p + 1] = table.start_n[p] + send_cnt[p];
      table.start_u[p + 1] = table.start_u[p] + send_u[p];
      // modular address arithmetic: base + (displacement - bucket start) * size
      table.units[p] = du[p] + (disp_u[p] - table.start_u[p]) * w();
      table.lens[p] = dl[p] + (disp_n[p] - table.start_n[p]) * 4;
      table.gidx[p] = dg[p] + (disp_n[p] - table.start_n[p]) * 4;
    }
    HCHECK(cudaMemcpyAsync(at<PeerTable>(M.peer_table), &table, sizeof table, cudaMemcpyHostToDevice, s));
    launch_gather_peer(kernel_coder(coder), at<uint32_t>(M.send_perm), n, units, offsets, S.lb_scan(),
                       S.next_counter(), S.next_epoch(), at<PeerTable>(M.peer_table), s);
    HCHECK(cudaGetLastError());
    return HUSKY_OK;
  }

  // phase 4 on the received bucket (recv buffers already filled)
  // r_units / r_lens / r_gidx: the received arrays (receive workspace or window)
  husky_status phase4(const uint8_t *r_units, const uint32_t *r_lens, const uint32_t *r_gidx, uint8_t *rws,
                      const RecvLayout &R, uint32_t *d_perm_out, void *d_sorted_units_out,
                      int64_t *d_sorted_offsets_out, husky_outcome *h_out) {
    if (n_out == 0) {
      if (h_out) { memset(h_out, 0, sizeof *h_out); h_out->perfect = 1; h_out->domain_ok = 1; }
      if (d_sorted_offsets_out) HCHECK(cudaMemsetAsync(d_sorted_offsets_out, 0, 8, s));
      return HUSKY_OK;
    }
    HCHECK(cudaMemsetAsync(rws + R.lb, 0, scan_tiles(n_out) * 8 + 8, s));
    HCHECK(cudaMemsetAsync(&st()->tile_counter[63], 0, 4, s));
    HUSKY_SCOPE(ST_MULTI, s, 0);
    k_lens_to_offsets<<<(unsigned)scan_tiles(n_out), kScanThreads, 0, s>>>(
        r_lens, n_out, (int64_t *)(rws + R.offsets), (unsigned long long *)(rws + R.lb),
        &st()->tile_counter[63], 1, 0);
    HCHECK(cudaGetLastError());
    if (debug_sync()) {
      int64_t ends[2] = {-1, -1};
      uint32_t l0[4] = {0, 0, 0, 0};
      HCHECK(cudaStreamSynchronize(s));
      HCHECK(cudaMemcpy(&ends[0], rws + R.offsets, 8, cudaMemcpyDeviceToHost));
      HCHECK(cudaMemcpy(&ends[1], (int64_t *)(rws + R.offsets) + n_out, 8, cudaMemcpyDeviceToHost));
      HCHECK(cudaMemcpy(l0, r_lens, 16, cudaMemcpyDeviceToHost));
      fprintf(stderr, "[husky] rank %d recv n=%llu units=%llu offsets[0]=%lld offsets[n]=%lld lens %u %u %u %u\n",
              rank, (unsigned long long)n_out, (unsigned long long)units_out, (long long)ends[0],
              (long long)ends[1], l0[0], l0[1], l0[2], l0[3]);
    }
    husky_status e = sort_impl(coder, r_units, (const int64_t *)(rws + R.offsets), n_out, d_perm_out,
                               d_sorted_units_out, d_sorted_offsets_out, rws + R.sort_ws,
                               make_layout(n_out).total, h_out, s, false);
    if (e) return e;
    HUSKY_SCOPE(ST_MULTI, s, 0);
    k_remap<<<grid_for(n_out), 256, 0, s>>>(d_perm_out, n_out, r_gidx);
    HCHECK(cudaGetLastError());
    return HUSKY_OK;
  }
};

// exchange over NCCL: counts (phase 2) and data (phase 3)
static husky_status nccl_allgather_samples(Plan &P) {
  uint64_t *buf = P.at<uint64_t>(P.M.samples);
  SampleRec *recs = P.at<SampleRec>(P.M.recs);
  NCHECK(ncclGroupStart());
  NCHECK(ncclAllGather(buf + (size_t)P.rank * kSampleStride, buf, kSampleStride, ncclUint64, P.comm->nccl, P.s));
  NCHECK(ncclAllGather(recs + (size_t)P.rank * kSamplesPerRank, recs, kSamplesPerRank * sizeof(SampleRec), ncclUint8,
                       P.comm->nccl, P.s));
  NCHECK(ncclGroupEnd());
  return HUSKY_OK;
}

// every rank gets the whole P x P count matrix (its displacements in the
// destinations' windows and the window size need the other ranks' rows)
static husky_status nccl_allgather_counts(Plan &P) {
  NCHECK(ncclAllGather(P.at<uint64_t>(P.M.counts), P.at<uint64_t>(P.M.rcounts), (size_t)P.world * 2, ncclUint64,
                       P.comm->nccl, P.s));
  return HUSKY_OK;
}

// AND of a flag over the ranks (synchronous)
static husky_status all_ranks_ok(Comm *c, cudaStream_t s, bool mine, bool *all) {
  unsigned long long v = mine ? 1ull : 0ull;
  HCHECK(cudaMemcpyAsync(c->d_tmp + c->world, &v, 8, cudaMemcpyHostToDevice, s));
  NCHECK(ncclAllReduce(c->d_tmp + c->world, c->d_tmp + c->world, 1, ncclUint64, ncclMin, c->nccl, s));
  HCHECK(cudaMemcpyAsync(&v, c->d_tmp + c->world, 8, cudaMemcpyDeviceToHost, s));
  if (husky_status e = comm_sync(c, s)) return e;
  *all = v != 0;
  return HUSKY_OK;
}

static void release_window(Comm *c) {
  if (c->win) ncclCommWindowDeregister(c->nccl, c->win);
  if (c->win_buf) ncclMemFree(c->win_buf);
  c->win = nullptr;
  c->win_buf = nullptr;
  c->win_bytes = 0;
}

// Make the receive window hold `need` bytes on every rank.  Collective: all
// ranks see the same count matrix, hence the same `need`, and take the same
// branches.  A failure anywhere turns the exchange into NCCL send/recv for the
// communicator's lifetime (*ok = false on every rank).
static husky_status ensure_window(Comm *c, size_t need, cudaStream_t s, bool *ok) {
  *ok = false;
  if (c->win_failed) return HUSKY_OK;
  if (c->win && c->win_bytes >= need) { *ok = true; return HUSKY_OK; }
  HCHECK(cudaStreamSynchronize(s));
  release_window(c);
  const size_t bytes = align_up(need + need / 4 + 4096, (size_t)2 << 20);  // headroom for the next call
  bool mine = ncclMemAlloc(&c->win_buf, bytes) == ncclSuccess, all = false;
  if (!mine) c->win_buf = nullptr;
  if (husky_status e = all_ranks_ok(c, s, mine, &all)) return e;
  if (all) {
    mine = ncclCommWindowRegister(c->nccl, c->win_buf, bytes, &c->win, NCCL_WIN_COLL_SYMMETRIC) == ncclSuccess;
    if (!mine) c->win = nullptr;
    if (husky_status e = all_ranks_ok(c, s, mine, &all)) return e;
  }
  if (!all) {
    release_window(c);
    c->win_failed = true;
    fprintf(stderr, "[husky] symmetric window registration failed: exchanging by NCCL send/recv\n");
    return HUSKY_OK;
  }
  c->win_bytes = bytes;
  k_win_ptrs<<<1, 256, 0, s>>>(c->win, c->world, c->d_tmp);
  c->peer.assign(c->world, 0);
  HCHECK(cudaMemcpyAsync(c->peer.data(), c->d_tmp, (size_t)c->world * 8, cudaMemcpyDeviceToHost, s));
  HCHECK(cudaStreamSynchronize(s));
  // every peer must be load/store reachable (one NVLink / NVSwitch domain)
  mine = std::all_of(c->peer.begin(), c->peer.end(), [](unsigned long long a) { return a != 0; });
  if (husky_status e = all_ranks_ok(c, s, mine, &all)) return e;
  if (!all) {
    release_window(c);
    c->win_failed = true;
    fprintf(stderr, "[husky] a peer window is not load/store reachable: exchanging by NCCL send/recv\n");
    return HUSKY_OK;
  }
  *ok = true;
  return HUSKY_OK;
}

static husky_status nccl_exchange(Plan &P, uint8_t *rws, const RecvLayout &R) {
  const size_t w = P.w();
  uint64_t so = 0, su = 0, ro = 0, ru = 0;
  NCHECK(ncclGroupStart());
  for (int p = 0; p < P.world; ++p) {
    if (P.send_cnt[p]) {
      NCHECK(ncclSend(P.at<uint8_t>(P.M.send_units) + su * w, P.send_u[p] * w, ncclUint8, p, P.comm->nccl, P.s));
      NCHECK(ncclSend(P.at<uint32_t>(P.M.send_lens) + so, P.send_cnt[p], ncclUint32, p, P.comm->nccl, P.s));
      NCHECK(ncclSend(P.at<uint32_t>(P.M.send_gidx) + so, P.send_cnt[p], ncclUint32, p, P.comm->nccl, P.s));
    }
    if (P.recv_cnt[p]) {
      NCHECK(ncclRecv(rws + R.units + ru * w, P.recv_u[p] * w, ncclUint8, p, P.comm->nccl, P.s));
      NCHECK(ncclRecv((uint32_t *)(rws + R.lens) + ro, P.recv_cnt[p], ncclUint32, p, P.comm->nccl, P.s));
      NCHECK(ncclRecv((uint32_t *)(rws + R.gidx) + ro, P.recv_cnt[p], ncclUint32, p, P.comm->nccl, P.s));
    }
    so += P.send_cnt[p]; su += P.send_u[p]; ro += P.recv_cnt[p]; ru += P.recv_u[p];
  }
  NCHECK(ncclGroupEnd());
  return HUSKY_OK;
}


}  // namespace husky

using namespace husky;

extern "C" {

husky_status husky_select_splitters(int coder, const void *h_units, const int64_t *h_offsets, uint64_t m,
                                    int world, uint64_t *h_idx) {
  if (!valid_coder(coder)) return fail(HUSKY_ERR_INVALID_ARG, "unknown coder %d", coder);
  if (world < 1 || world > kMaxWorld) return fail(HUSKY_ERR_INVALID_ARG, "world %d out of range", world);
  if (world == 1 || m == 0) return HUSKY_OK;
  if (!h_idx || !h_offsets || !h_units) return fail(HUSKY_ERR_INVALID_ARG, "null pointer");
  const size_t w = coder_unit_bytes(coder);
  auto unit = [&](int64_t p) -> uint32_t {
    return w == 1 ? ((const uint8_t *)h_units)[p] : ((const uint16_t *)h_units)[p];
  };
  std::vector<uint64_t> idx(m);
  for (uint64_t i = 0; i < m; ++i) idx[i] = i;
  // the sort order (units unsigned, shorter first), ties by index
  std::stable_sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
    const int64_t oa = h_offsets[a], la = h_offsets[a + 1] - oa, ob = h_offsets[b], lb = h_offsets[b + 1] - ob;
    const int64_t k = la < lb ? la : lb;
    for (int64_t t = 0; t < k; ++t) {
      const uint32_t x = unit(oa + t), y = unit(ob + t);
      if (x != y) return x < y;
    }
    return la < lb;
  });
  for (int k = 1; k < world; ++k) h_idx[k - 1] = idx[(size_t)((unsigned __int128)k * m / world)];
  return HUSKY_OK;
}

husky_status husky_comm_unique_id(uint8_t id[128]) {
  if (!id) return fail(HUSKY_ERR_INVALID_ARG, "id is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  NCHECK(ncclGetUniqueId(&u));
  memcpy(id, &u, 128);
  return HUSKY_OK;
}

husky_status husky_comm_create(int rank, int world, const uint8_t id[128], void **comm) {
  if (!id || !comm || world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
    return fail(HUSKY_ERR_INVALID_ARG, "bad comm arguments (rank %d, world %d)", rank, world);
  ncclUniqueId u;
  memcpy(&u, id, 128);
  Comm *c = new Comm;
  c->rank = rank;
  c->world = world;
  ncclResult_t r = ncclCommInitRank(&c->nccl, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(HUSKY_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  if (cudaMalloc(&c->d_tmp, ((size_t)world + 1) * 8) != cudaSuccess) {
    ncclCommDestroy(c->nccl);
    delete c;
    return fail(HUSKY_ERR_CUDA, "cudaMalloc of the communicator scratch failed");
  }
  *comm = c;
  return HUSKY_OK;
}

husky_status husky_comm_world(void *comm, int *world) {
  if (!comm || !world) return fail(HUSKY_ERR_INVALID_ARG, "null pointer");
  *world = ((Comm *)comm)->world;
  return HUSKY_OK;
}

husky_status husky_comm_destroy(void *comm) {
  if (!comm) return HUSKY_OK;
  Comm *c = (Comm *)comm;
  if (c->aborted) {  // ncclCommAbort already released the NCCL resources
    if (c->d_tmp) cudaFree(c->d_tmp);
    delete c;
    return HUSKY_OK;
  }
  release_window(c);
  if (c->d_tmp) cudaFree(c->d_tmp);
  ncclResult_t r = ncclCommDestroy(c->nccl);
  delete c;
  if (r != ncclSuccess) return fail(HUSKY_ERR_NCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return HUSKY_OK;
}

husky_status husky_sort_multi_workspace(int coder, uint64_t n_local, uint64_t local_units, int world,
                                        size_t *bytes) {
  if (!valid_coder(coder) || !bytes || world < 1 || world > kMaxWorld)
    return fail(HUSKY_ERR_INVALID_ARG, "bad arguments");
  *bytes = make_multi_layout(coder, n_local, local_units, world).total;
  return HUSKY_OK;
}

husky_status husky_sort_multi_plan(void *comm, int coder, const void *d_units, const int64_t *d_offsets,
                                   uint64_t n_local, uint64_t global_base, void *d_ws, size_t ws_bytes,
                                   void **plan, uint64_t *h_n_out, uint64_t *h_units_out, void *stream) {
  if (!comm || !valid_coder(coder) || !plan || !d_offsets || !d_ws || (n_local && !d_units))
    return fail(HUSKY_ERR_INVALID_ARG, "null required pointer or unknown coder");
  if (global_base + n_local >= 0xFFFFFFFFull) return fail(HUSKY_ERR_INVALID_ARG, "global index >= 2^32 - 1");
  if ((uintptr_t)d_ws % 256) return fail(HUSKY_ERR_INVALID_ARG, "workspace not 256-byte aligned");
  Comm *c = (Comm *)comm;
  if (c->aborted) return fail(HUSKY_ERR_NCCL, "communicator was aborted by an earlier failure");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t o[2] = {0, 0};
  if (n_local) {
    HCHECK(cudaMemcpyAsync(&o[0], d_offsets, 8, cudaMemcpyDeviceToHost, s));
    HCHECK(cudaMemcpyAsync(&o[1], d_offsets + n_local, 8, cudaMemcpyDeviceToHost, s));
    HCHECK(cudaStreamSynchronize(s));
  }
  Plan *P = new Plan;
  P->comm = c;
  P->coder = coder;
  P->rank = c->rank;
  P->world = c->world;
  P->units = d_units;
  P->offsets = d_offsets;
  P->n = n_local;
  P->gbase = global_base;
  P->local_units = (uint64_t)(o[1] - o[0]);
  P->ws = (uint8_t *)d_ws;
  P->s = s;
  P->M = make_multi_layout(coder, n_local, P->local_units, c->world);
  husky_status e = HUSKY_OK;
  PhaseClock pc(s);
  if (ws_bytes < P->M.total) e = fail(HUSKY_ERR_WORKSPACE, "workspace %zu < required %zu", ws_bytes, P->M.total);
  if (!e) e = P->phase1();
  pc.mark("encode+sample");
  if (!e) e = nccl_allgather_samples(*P);
  pc.mark("allgather samples");
  if (!e) e = P->choose_splitters();
  pc.mark("splitters");
  if (!e) e = P->phase2();
  pc.mark("bucket");
  if (!e) e = nccl_allgather_counts(*P);
  if (!e) e = P->read_counts();
  pc.mark("counts");
  // exchange mode: peer stores into the receive windows unless disabled / failed
  if (!e && !exchange_by_nccl()) {
    bool ok = false;
    e = ensure_window(c, make_win_layout(P->w(), P->cap_n, P->cap_u).total, s, &ok);
    P->peer = ok;
  }
  pc.mark("window");
  if (e) { delete P; return e; }
  if (h_n_out) *h_n_out = P->n_out;
  if (h_units_out) *h_units_out = P->units_out;
  *plan = P;
  return HUSKY_OK;
}

husky_status husky_sort_multi_recv_workspace(void *plan, size_t *bytes) {
  if (!plan || !bytes) return fail(HUSKY_ERR_INVALID_ARG, "null pointer");
  Plan *P = (Plan *)plan;
  *bytes = make_recv_layout(P->coder, P->n_out, P->units_out, !P->peer).total;
  return HUSKY_OK;
}

husky_status husky_sort_multi_exec(void *plan, uint32_t *d_perm_out, void *d_sorted_units_out,
                                   int64_t *d_sorted_offsets_out, void *d_recv_ws, size_t recv_ws_bytes,
                                   husky_outcome *h_out, void *stream) {
  if (!plan || (!d_perm_out && ((Plan *)plan)->n_out) || !d_recv_ws)
    return fail(HUSKY_ERR_INVALID_ARG, "null required pointer");
  if ((d_sorted_units_out == nullptr) != (d_sorted_offsets_out == nullptr))
    return fail(HUSKY_ERR_INVALID_ARG, "sorted units/offsets must both be set or both NULL");
  Plan *P = (Plan *)plan;
  P->s = (cudaStream_t)stream;
  P->S.s = P->s;
  RecvLayout R = make_recv_layout(P->coder, P->n_out, P->units_out, !P->peer);
  if (recv_ws_bytes < R.total) return fail(HUSKY_ERR_WORKSPACE, "recv workspace %zu < %zu", recv_ws_bytes, R.total);
  if ((uintptr_t)d_recv_ws % 256) return fail(HUSKY_ERR_INVALID_ARG, "workspace not 256-byte aligned");
  uint8_t *rws = (uint8_t *)d_recv_ws;
  Comm *c = P->comm;
  PhaseClock pc(P->s);
  if (husky_status e = P->partition()) return e;
  pc.mark("partition");
  const uint8_t *r_units = rws + R.units;
  const uint32_t *r_lens = (const uint32_t *)(rws + R.lens), *r_gidx = (const uint32_t *)(rws + R.gidx);
  if (P->peer) {
    const WinLayout WL = make_win_layout(P->w(), P->cap_n, P->cap_u);
    std::vector<unsigned long long> du(P->world), dl(P->world), dg(P->world);
    for (int q = 0; q < P->world; ++q) {
      du[q] = c->peer[q] + WL.units;
      dl[q] = c->peer[q] + WL.lens;
      dg[q] = c->peer[q] + WL.gidx;
    }
    if (husky_status e = P->scatter_peer(du, dl, dg)) return e;
    pc.mark("scatter to peers");
    // every rank's stores are done before any rank reads its window
    NCHECK(ncclAllReduce(c->d_tmp + c->world, c->d_tmp + c->world, 1, ncclUint64, ncclSum, c->nccl, P->s));
    pc.mark("barrier");
    const uint8_t *wb = (const uint8_t *)c->win_buf;
    r_units = wb + WL.units;
    r_lens = (const uint32_t *)(wb + WL.lens);
    r_gidx = (const uint32_t *)(wb + WL.gidx);
  } else {
    if (husky_status e = P->build_send()) return e;
    pc.mark("send buffers");
    if (husky_status e = nccl_exchange(*P, rws, R)) return e;
    pc.mark("exchange");
  }
  if (husky_status e = P->phase4(r_units, r_lens, r_gidx, rws, R, d_perm_out, d_sorted_units_out,
                                 d_sorted_offsets_out, h_out))
    return e;
  if (h_out) {
    h_out->exchange = P->peer ? HUSKY_EXCHANGE_PEER : HUSKY_EXCHANGE_NCCL;
    uint64_t to = 0, from = 0;
    for (int q = 0; q < P->world; ++q) {
      if (q == P->rank) continue;
      to += P->send_u[q] * P->w() + 8 * P->send_cnt[q];
      from += P->recv_u[q] * P->w() + 8 * P->recv_cnt[q];
    }
    h_out->bytes_to_peers = to;
    h_out->bytes_from_peers = from;
  }
  pc.mark("local sort");
  if (husky_status e = comm_sync(c, P->s)) return e;
  return checked_result(HUSKY_OK, "husky_sort_multi_exec");
}

husky_status husky_plan_destroy(void *plan) {
  delete (Plan *)plan;
  return HUSKY_OK;
}

husky_status husky_sort_multi(void *comm, int coder, const void *d_units, const int64_t *d_offsets,
                              uint64_t n_local, uint64_t global_base, uint32_t *d_perm_out,
                              void *d_sorted_units_out, int64_t *d_sorted_offsets_out, uint64_t cap_n,
                              uint64_t cap_units, uint64_t *h_n_out, uint64_t *h_units_out, void *d_ws,
                              size_t ws_bytes, husky_outcome *h_out, void *stream) {
  // d_ws holds the plan workspace followed by the receive workspace
  if (!d_ws) return fail(HUSKY_ERR_INVALID_ARG, "null workspace");
  if (!comm || !valid_coder(coder)) return fail(HUSKY_ERR_INVALID_ARG, "null comm or unknown coder");
  Comm *c = (Comm *)comm;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t o[2] = {0, 0};
  if (n_local) {
    HCHECK(cudaMemcpyAsync(&o[0], d_offsets, 8, cudaMemcpyDeviceToHost, s));
    HCHECK(cudaMemcpyAsync(&o[1], d_offsets + n_local, 8, cudaMemcpyDeviceToHost, s));
    HCHECK(cudaStreamSynchronize(s));
  }
  size_t plan_bytes = make_multi_layout(coder, n_local, (uint64_t)(o[1] - o[0]), c->world).total;
  if (ws_bytes < plan_bytes) return fail(HUSKY_ERR_WORKSPACE, "workspace %zu < plan %zu", ws_bytes, plan_bytes);
  void *plan = nullptr;
  uint64_t n_out = 0, u_out = 0;
  if (husky_status e = husky_sort_multi_plan(comm, coder, d_units, d_offsets, n_local, global_base, d_ws,
                                             plan_bytes, &plan, &n_out, &u_out, stream))
    return e;
  if (h_n_out) *h_n_out = n_out;
  if (h_units_out) *h_units_out = u_out;
  size_t rb = 0;
  husky_sort_multi_recv_workspace(plan, &rb);
  // every rank must reach the exchange or none: the capacity / workspace
  // checks are agreed on across the ranks first (a rank that failed alone
  // would leave its peers blocked in the exchange)
  const bool cap_ok = n_out <= cap_n && u_out <= cap_units;
  const bool ws_ok = ws_bytes >= align_up(plan_bytes, 256) + rb;
  bool all_cap = true, all_ws = true;
  husky_status e = all_ranks_ok(c, s, cap_ok, &all_cap);
  if (!e) e = all_ranks_ok(c, s, ws_ok, &all_ws);
  if (!e && !all_cap)
    e = fail(HUSKY_ERR_CAPACITY, cap_ok ? "another rank's shard exceeds its capacity"
                                        : "shard needs %llu strings / %llu units",
             (unsigned long long)n_out, (unsigned long long)u_out);
  else if (!e && !all_ws)
    e = fail(HUSKY_ERR_WORKSPACE, ws_ok ? "another rank's workspace is too small for its receive buffers"
                                        : "workspace too small for the receive buffers");
  else if (!e)
    e = husky_sort_multi_exec(plan, d_perm_out, d_sorted_units_out, d_sorted_offsets_out,
                              (uint8_t *)d_ws + align_up(plan_bytes, 256), ws_bytes - align_up(plan_bytes, 256),
                              h_out, stream);
  husky_plan_destroy(plan);
  return e;
}

// ------------------------------------------------------------ loopback driver
// Sorts n strings as if block-distributed over `world` virtual ranks of ONE GPU,
// running exactly the sample-sort phases above with device-to-device copies as
// the transport.  Output = the rank-order concatenation (global perm, sorted
// units, global sorted offsets).  h_shard_n (nullable, world entries) receives
// the shard sizes.  Test hook for the sharded path; declared in husky.h.
static uint64_t lb_base(uint64_t n, int world, int r) { return (uint64_t)((unsigned __int128)n * r / world); }

husky_status husky_sort_multi_loopback_workspace(int coder, int world, uint64_t n, uint64_t total_units,
                                                 size_t *bytes) {
  if (!valid_coder(coder) || !bytes || world < 1 || world > kMaxWorld) return fail(HUSKY_ERR_INVALID_ARG, "bad args");
  size_t tot = 0;
  for (int r = 0; r < world; ++r) {
    uint64_t nr = lb_base(n, world, r + 1) - lb_base(n, world, r);
    tot += align_up(make_multi_layout(coder, nr, total_units, world).total, 256);  // units bound per rank
  }
  tot += align_up(make_recv_layout(coder, n, total_units).total, 256);  // shared recv + sort ws (worst case)
  // peer-store mode: every virtual rank's receive window (sum of the shards)
  tot += align_up(total_units * coder_unit_bytes(coder) + n * 8 + (size_t)world * 1024, 256);
  tot += align_up((size_t)world * 256, 256) * world;
  *bytes = tot;
  return HUSKY_OK;
}

husky_status husky_sort_multi_loopback(int coder, int world, const void *d_units, const int64_t *d_offsets,
                                       uint64_t n, uint32_t *d_perm, void *d_sorted_units,
                                       int64_t *d_sorted_offsets, void *d_ws, size_t ws_bytes,
                                       uint64_t *h_shard_n, husky_outcome *h_out, void *stream) {
  if (!valid_coder(coder) || world < 1 || world > kMaxWorld || !d_offsets || !d_ws || (n && (!d_units || !d_perm)))
    return fail(HUSKY_ERR_INVALID_ARG, "bad arguments");
  if ((d_sorted_units == nullptr) != (d_sorted_offsets == nullptr))
    return fail(HUSKY_ERR_INVALID_ARG, "sorted units/offsets must both be set or both NULL");
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<int64_t> bo(world + 1);
  for (int r = 0; r <= world; ++r)
    HCHECK(cudaMemcpyAsync(&bo[r], d_offsets + lb_base(n, world, r), 8, cudaMemcpyDeviceToHost, s));
  HCHECK(cudaStreamSynchronize(s));
  uint64_t total_units = (uint64_t)(bo[world] - bo[0]);
  size_t need = 0;
  husky_sort_multi_loopback_workspace(coder, world, n, total_units, &need);
  if (ws_bytes < need) return fail(HUSKY_ERR_WORKSPACE, "workspace %zu < required %zu", ws_bytes, need);
  uint8_t *ws = (uint8_t *)d_ws;
  size_t off = 0;
  std::vector<Plan> P(world);
  for (int r = 0; r < world; ++r) {
    Plan &p = P[r];
    p.coder = coder; p.rank = r; p.world = world; p.units = d_units;
    p.offsets = d_offsets + lb_base(n, world, r);
    p.n = lb_base(n, world, r + 1) - lb_base(n, world, r);
    p.gbase = lb_base(n, world, r);
    p.local_units = (uint64_t)(bo[r + 1] - bo[r]);
    p.s = s;
    p.M = make_multi_layout(coder, p.n, p.local_units, world);
    p.ws = ws + off;
    off += align_up(make_multi_layout(coder, p.n, total_units, world).total, 256);
  }
  uint8_t *rws_all = ws + off;
  // phase 1 + "all-gather" of the samples
  for (auto &p : P) if (husky_status e = p.phase1()) return e;
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < world; ++q)
      if (q != r)
      {
        HCHECK(cudaMemcpyAsync(P[r].at<uint64_t>(P[r].M.samples) + (size_t)q * kSampleStride,
                               P[q].at<uint64_t>(P[q].M.samples) + (size_t)q * kSampleStride, kSampleStride * 8,
                               cudaMemcpyDeviceToDevice, s));
        HCHECK(cudaMemcpyAsync(P[r].at<SampleRec>(P[r].M.recs) + (size_t)q * kSamplesPerRank,
                               P[q].at<SampleRec>(P[q].M.recs) + (size_t)q * kSamplesPerRank,
                               kSamplesPerRank * sizeof(SampleRec), cudaMemcpyDeviceToDevice, s));
      }
  for (auto &p : P) if (husky_status e = p.choose_splitters()) return e;
  for (auto &p : P) if (husky_status e = p.phase2()) return e;
  // "all-gather" of the counts: row q of every rank's matrix = rank q's counts
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < world; ++q)
      HCHECK(cudaMemcpyAsync(P[r].at<uint64_t>(P[r].M.rcounts) + (size_t)q * world * 2, P[q].at<uint64_t>(P[q].M.counts),
                             (size_t)world * 16, cudaMemcpyDeviceToDevice, s));
  for (auto &p : P) if (husky_status e = p.read_counts()) return e;
  for (auto &p : P) if (husky_status e = p.partition()) return e;
  const size_t w = coder_unit_bytes(coder);
  // peer-store mode (default): the gather of every virtual rank writes straight
  // into the destinations' windows (regions of this workspace), exactly as the
  // NCCL path writes into the NVLink mappings; HUSKY_EXCHANGE=copy: send
  // buffers + device-to-device copies
  const bool peer = !exchange_by_nccl();
  uint8_t *win_all = rws_all + align_up(make_recv_layout(coder, n, total_units).total, 256);
  std::vector<size_t> win_off(world);
  std::vector<WinLayout> WLs(world);
  {
    size_t o = 0;
    for (int r = 0; r < world; ++r) {
      WLs[r] = make_win_layout(w, P[r].n_out, P[r].units_out);
      win_off[r] = o;
      o += WLs[r].total;
    }
  }
  if (peer) {
    std::vector<unsigned long long> du(world), dl(world), dg(world);
    for (int r = 0; r < world; ++r) {
      const unsigned long long base = (unsigned long long)(uintptr_t)(win_all + win_off[r]);
      du[r] = base + WLs[r].units;
      dl[r] = base + WLs[r].lens;
      dg[r] = base + WLs[r].gidx;
    }
    for (auto &p : P) if (husky_status e = p.scatter_peer(du, dl, dg)) return e;
  } else {
    for (auto &p : P) if (husky_status e = p.build_send()) return e;
  }
  // data exchange (copy mode) + local sorts, one destination rank at a time (shared recv ws)
  uint64_t out_n = 0, out_u = 0;
  husky_outcome agg;
  memset(&agg, 0, sizeof agg);
  agg.perfect = 1; agg.domain_ok = 1;
  for (int r = 0; r < world; ++r) {
    Plan &dst = P[r];
    RecvLayout R = make_recv_layout(coder, dst.n_out, dst.units_out, !peer);
    const uint8_t *r_units = rws_all + R.units;
    const uint32_t *r_lens = (const uint32_t *)(rws_all + R.lens), *r_gidx = (const uint32_t *)(rws_all + R.gidx);
    if (peer) {
      uint8_t *wb = win_all + win_off[r];
      r_units = wb + WLs[r].units;
      r_lens = (const uint32_t *)(wb + WLs[r].lens);
      r_gidx = (const uint32_t *)(wb + WLs[r].gidx);
    }
    uint64_t ro = 0, ru = 0;
    for (int q = 0; q < world && !peer; ++q) {
      Plan &src = P[q];
      uint64_t so = 0, su = 0;
      for (int k = 0; k < r; ++k) { so += src.send_cnt[k]; su += src.send_u[k]; }
      uint64_t cnt = src.send_cnt[r], u = src.send_u[r];
      if (cnt) {
        HCHECK(cudaMemcpyAsync(rws_all + R.units + ru * w, src.at<uint8_t>(src.M.send_units) + su * w, u * w,
                               cudaMemcpyDeviceToDevice, s));
        HCHECK(cudaMemcpyAsync((uint32_t *)(rws_all + R.lens) + ro, src.at<uint32_t>(src.M.send_lens) + so, cnt * 4,
                               cudaMemcpyDeviceToDevice, s));
        HCHECK(cudaMemcpyAsync((uint32_t *)(rws_all + R.gidx) + ro, src.at<uint32_t>(src.M.send_gidx) + so, cnt * 4,
                               cudaMemcpyDeviceToDevice, s));
      }
      ro += cnt; ru += u;
    }
    husky_outcome o;
    // empty shards write nothing (their offsets slot belongs to the previous shard)
    void *su_out = (d_sorted_units && dst.n_out) ? (uint8_t *)d_sorted_units + out_u * w : nullptr;
    int64_t *so_out = (d_sorted_offsets && dst.n_out) ? d_sorted_offsets + out_n : nullptr;
    // offsets slot out_n is shared with the previous shard's end: write it first
    if (husky_status e = dst.phase4(r_units, r_lens, r_gidx, rws_all, R, d_perm + out_n, su_out, so_out, &o))
      return e;
    if (so_out && out_u && dst.n_out) {
      HUSKY_SCOPE(ST_MULTI, s, 0);
      k_add_base<<<grid_for(dst.n_out + 1), 256, 0, s>>>(so_out, dst.n_out + 1, (int64_t)out_u);
    }
    if (h_shard_n) h_shard_n[r] = dst.n_out;
    agg.perfect &= o.perfect; agg.domain_ok &= o.domain_ok;
    agg.n_runs += o.n_runs; agg.n_in_runs += o.n_in_runs;
    agg.max_run = std::max(agg.max_run, o.max_run);
    for (int c = 0; c < 4; ++c) agg.runs_by_class[c] += o.runs_by_class[c];
    agg.refine_rounds += o.refine_rounds; agg.radix_passes += o.radix_passes;
    agg.keys_partitioned += o.keys_partitioned;
    out_n += dst.n_out; out_u += dst.units_out;
  }
  if (n == 0 && d_sorted_offsets) HCHECK(cudaMemsetAsync(d_sorted_offsets, 0, 8, s));
  HCHECK(cudaStreamSynchronize(s));
  HCHECK(cudaGetLastError());
  agg.exchange = peer ? HUSKY_EXCHANGE_LOOPBACK_PEER : HUSKY_EXCHANGE_LOOPBACK_COPY;
  if (h_out) *h_out = agg;
  return checked_result(HUSKY_OK, "husky_sort_multi_loopback");
}

}  // extern "C"
