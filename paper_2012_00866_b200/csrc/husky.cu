// husky.cu -- host orchestration and the C ABI of libhusky (single GPU).
//
// husky_sort = Alg. 1 re-expressed for one B200:
//   encode (A1, Alg. 2-4)  ->  onesweep LSD radix of (code, index) (A2, Alg. 1
//   line 3)  ->  run detection + pairwise order check (A3, "we can easily
//   determine whether our encoding was perfect")  ->  fix-up
//   of dirty runs (A5, the cleanup of Alg. 1 line 5 restricted to where
//   inversions can be) with giant-run refinement (A6)  ->  gather (A4).
// Host<->device synchronisation: ONE per sort on the common path (the outcome,
// read after the re-gather); the radix pass plan is made on device and input
// violations turn later kernels into no-ops.  Only inputs with giant dirty runs
// (A6) add one synchronisation per refinement round.
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <atomic>
#include <thread>
#include <utility>
#include <vector>

#include "husky_internal.cuh"
#include "kernels.cuh"
#include "host_common.h"

namespace husky {

thread_local std::string g_last_error;

Profiler &profiler() {
  static Profiler *p = new Profiler;  // never destroyed: events may outlive static teardown
  return *p;
}

husky_status fail(husky_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#ifdef HUSKY_CHECKED
static std::vector<ChkReader> &chk_readers() {
  static std::vector<ChkReader> *v = new std::vector<ChkReader>;
  return *v;
}
int checked_register(ChkReader r) {
  chk_readers().push_back(r);
  return 1;
}
unsigned long long checked_take(unsigned long long *first) {
  cudaDeviceSynchronize();
  unsigned long long total = 0;
  for (ChkReader r : chk_readers()) total += r(first);
  return total;
}
#endif

#ifdef HUSKY_CHECKED
// shrink (HUSKY_CHK_SELFTEST=1): bounds one short, so that a correct sort
// must report violations -- the check that the checks fire
__global__ void k_chk_init(DevState *st, const int64_t *offsets, uint64_t n, uint32_t w, uint32_t shrink) {
  st->chk_n = n - shrink;
  st->chk_units = (unsigned long long)offsets[n] * w - shrink;
}
static uint32_t chk_shrink() {
  static const uint32_t v = [] {
    const char *e = getenv("HUSKY_CHK_SELFTEST");
    return (e && atoi(e) == 1) ? 1u : 0u;
  }();
  return v;
}
#endif

// checked builds: the violations counted by the kernels of the call that just
// returned (synchronises the device); always HUSKY_OK otherwise
husky_status checked_result(husky_status st, const char *what) {
#ifdef HUSKY_CHECKED
  unsigned long long first = 0, v = checked_take(&first);
  if (st == HUSKY_OK && v)
    return fail(HUSKY_ERR_CUDA, "checked build: %s: %llu out-of-bounds indices (first: site %llu index %llu)", what,
                v, first >> 48, first & 0xFFFFFFFFFFFFull);
#else
  (void)what;
#endif
  return st;
}

int device_sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

Layout make_layout(uint64_t n) {
  Layout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  L.n = n;
  L.tiles_r = radix_tiles(n);
  L.tiles_s = scan_tiles(n) > gather_tiles(n) ? scan_tiles(n) : gather_tiles(n);
  L.cap_sm = n / 2 + 1;
  L.cap_g = n / (kMediumMax + 1) + 1;
  L.state = take(sizeof(DevState));
  L.keysA = take(n * 8);
  L.keysB = take(n * 8);
  L.vals = take(n * 4);
  // packed initial payload (index | min(len, 15) << 28), only when n <= 2^28
  L.vals2 = take(n <= kPackMaxN ? n * 4 : 0);
  // string slab records for the main gather (16 B per string, encode.cu)
  L.slab = take(n * 16);
  L.lb_radix_words = radix_lb_words(n);
  L.lb_radix = take(L.lb_radix_words * 8);
  L.lb_scan = take(L.tiles_s * 16);  // two look-back arrays (lengths, run counts)
  L.run_start = take(L.cap_sm * 4);
  L.run_end = take(L.cap_sm * 4);
  L.dirty = take(L.cap_sm);
  L.list_sm = take(L.cap_sm * 8);
  L.list_g = take(L.cap_g * 8);
  L.total = off;
  return L;
}

// HUSKY_DEBUG_SYNC only: verify that perm[0..n) is a permutation (bitmap count)
__global__ void k_debug_perm(const uint32_t *perm, uint64_t n, uint32_t *bitmap, unsigned long long *bad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = perm[i];
    if (v >= n) { atomicAdd(bad, 1ull); continue; }
    uint32_t old = atomicOr(&bitmap[v >> 5], 1u << (v & 31));
    if (old & (1u << (v & 31))) atomicAdd(bad, 1ull);
  }
}

static void debug_check_perm(const uint32_t *perm, uint64_t n, const char *tag, cudaStream_t s) {
  if (!debug_sync()) return;
  uint32_t *bm = nullptr;
  unsigned long long *bad = nullptr, hb = 0;
  cudaStreamSynchronize(s);
  cudaMalloc(&bm, (n / 32 + 1) * 4);
  cudaMalloc(&bad, 8);
  cudaMemset(bm, 0, (n / 32 + 1) * 4);
  cudaMemset(bad, 0, 8);
  k_debug_perm<<<1024, 256>>>(perm, n, bm, bad);
  cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
  if (hb) fprintf(stderr, "[husky] perm check after %s: %llu bad entries (n=%llu)\n", tag, hb, (unsigned long long)n);
  cudaFree(bm);
  cudaFree(bad);
}

struct HostSnap {  // small prefix of DevState read back at sync points
  uint32_t trivial_mask, violations;
};

static husky_status cuda_check(const char *where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HUSKY_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
  return HUSKY_OK;
}

#define HCHECK(expr)                                                                          \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) return fail(HUSKY_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

static husky_status refine_giants(Sorter &S, const DevState &hs0, void *d_sorted_units, int64_t *d_sorted_offsets,
                                  DevState *out, bool general);

// HUSKY_SLAB=1 forces the slab records at any size (tests), 0 disables them
// (read per sort: a getenv, so tests can switch it within one process)
static int slab_env() {
  const char *e = getenv("HUSKY_SLAB");
  return e ? atoi(e) : -1;
}

static int skip_env() {
  const char *e = getenv("HUSKY_SKIP");
  return e ? atoi(e) : 1;
}

static bool alpha_env() {
  const char *e = getenv("HUSKY_ALPHA");
  return !(e && e[0] == '0');
}

// What one sort enqueues before its single synchronisation (decided on the
// host from the arguments and the environment; part of the graph cache key).
// from this many strings the host waits for the device-side pass plan and
// launches only the planned pass slots (enqueue_main); below, all 8 slots are
// enqueued without a synchronisation (and the sequence may be a cached graph)
constexpr uint64_t kHostPlanMinN = 1ull << 26;

struct MainFlags {
  int coder = 0, kc = 0;
  bool packed = false, compress = false, slab = false, pdl = true;
  int skip = 0;  // leave the lowest varying digit unsorted (R19): 0 never, 1 entropy rule, 2 always
};

// Everything from the DevState reset to the copy of DevState into h_state
// (pinned when captured into a graph): encode, histograms + plan, the 8 pass
// slots, the gather with run detection, classification and the small / medium
// fix-ups.  Enqueued on S.s; no host synchronisation inside.
static husky_status enqueue_main(Sorter &S, const MainFlags &F, void *d_sorted_units, int64_t *d_sorted_offsets,
                                 DevState *h_state) {
  const Layout &L = S.L;
  DevState *st = S.st;
  cudaStream_t s = S.s;
  const uint64_t n = S.n;
  const int coder = F.coder, kc = F.kc;
  const void *d_units = S.units;
  const int64_t *d_offsets = S.offsets;
  uint32_t *d_perm = S.perm;
  HCHECK(cudaMemsetAsync(st, 0, sizeof(DevState), s));
#ifdef HUSKY_CHECKED
  k_chk_init<<<1, 1, 0, s>>>(st, d_offsets, n, (uint32_t)husky_unit_bytes(coder), chk_shrink());
#endif
  HCHECK(S.reset_lookback());
  // the dirty-run flags the main gather sets (cleared here, not between the key
  // sort and the gather, so the gather stays a programmatic dependent)
  HCHECK(cudaMemsetAsync(S.at<uint8_t>(L.dirty), 0, L.cap_sm, s));

  // ---- A1 encode (+ flags, alphabet, slab records) and the digit histograms
  // n <= 2^28: the payload carries min(len, 15) in its top 4 bits, so the
  // gather rebuilds strings of length <= PL from their code (no random reads)
  uint32_t *packed_payload = F.packed ? S.at<uint32_t>(L.vals2) : nullptr;
  uint4 *slab = F.slab ? S.at<uint4>(L.slab) : nullptr;
  uint64_t *keysA = S.keysA(), *keysB = S.keysB();
  uint32_t *vals_tmp = S.at<uint32_t>(L.vals);
  {
    GroupScope grp(ST_ENCODE, s);
    launch_encode(coder, d_units, d_offsets, n, S.keysA(), &st->violations, S.sms, s, packed_payload, slab,
                  !F.packed, F.compress ? st->alpha : nullptr);
  }
  launch_hist_plan(keysA, n, st, keysA, keysB, S.sms, s, F.compress, F.skip,
                   kc == HUSKY_CODER_UNICODE ? CoderTraits<HUSKY_CODER_UNICODE>::kS : CoderTraits<HUSKY_CODER_ASCII>::kS,
                   kc == HUSKY_CODER_UNICODE ? CoderTraits<HUSKY_CODER_UNICODE>::kPL : CoderTraits<HUSKY_CODER_ASCII>::kPL,
                   kc == HUSKY_CODER_UNICODE);

  // ---- A2 key sort, LSD onesweep: (code, index) -> sorted codes, perm.  The
  // pass plan (which digits are not shared by all keys) is made on device, so
  // the host enqueues all 8 pass slots without waiting; slots beyond the plan
  // exit at once.  Input violations (bad offsets, ASCII domain) make every
  // later kernel a no-op and are reported at the single synchronisation.
  {
    // large inputs: the host reads the plan's pass count and launches only
    // those slots -- an unused slot still launches (and retires) one CTA per
    // tile, ~0.2 ms each at 2^30, against ~20 us for this synchronisation
    // (such sorts are never captured into a graph, see sort_impl)
    int slots = 8;
    if (n >= kHostPlanMinN) {
      uint32_t np = 8;
      HCHECK(cudaMemcpyAsync(&np, &st->np, 4, cudaMemcpyDeviceToHost, s));
      HCHECK(cudaStreamSynchronize(s));
      slots = (int)std::min<uint32_t>(np, 8u);
    }
    GroupScope grp(ST_RADIX, s);  // profiler mode 2: the pass slots as one timed group
    for (int slot = 0; slot < slots; ++slot)
      launch_onesweep_slot(slot, keysA, keysB, packed_payload, d_perm, vals_tmp, n, st, S.lb_radix(),
                           S.next_counter(), S.next_epoch(), s);
  }
  launch_radix_finalize(st, packed_payload, d_perm, n, s);
  if (F.packed && !d_sorted_units) launch_unpack_perm(d_perm, n, s);  // the gather unpacks otherwise

  // ---- A4 gather in (code, index) order.  Done BEFORE the fix-up: the order
  // check below then reads every run's strings contiguously instead of through
  // a second random perm -> offsets -> units walk; only spans the fix-up
  // reorders are gathered again (rare outside all-colliding inputs).
  // A3 is fused into this gather: run detection and the order check of every
  // adjacent equal-code pair on the strings it stages (perm-only mode runs the
  // separate run scan below instead).
  uint32_t *run_start = S.at<uint32_t>(L.run_start), *run_end = S.at<uint32_t>(L.run_end);
  uint8_t *dirty = S.at<uint8_t>(L.dirty);
  if (d_sorted_units) {
    GroupScope grp(ST_GATHER, s);
    GatherRunsOut ro{run_start, run_end, dirty, S.lb_scan2(), st};
    launch_gather(kc, d_perm, n, d_units, d_offsets, d_sorted_units, d_sorted_offsets, S.lb_scan(),
                  S.next_counter(), S.next_epoch(), s, nullptr, F.packed, nullptr, st, &ro, slab);
  }
  debug_check_perm(d_perm, n, "key sort", s);

  // ---- A3 run detection + order check (keys: DevState::sorted_keys), classification
  uint2 *list_sm = S.at<uint2>(L.list_sm), *list_g = S.at<uint2>(L.list_g);
  if (!d_sorted_units)
    launch_runs_scan(kc, 0, nullptr, n, d_perm, d_units, d_offsets, 0, run_start, run_end, dirty, st,
                     S.lb_scan(), S.next_counter(), S.next_epoch(), s);
  launch_runs_classify(run_start, run_end, dirty, st, list_sm, L.cap_sm, list_g, true, S.sms, s);

  // ---- A5 fix-up of small / medium dirty runs (counts read on device), then
  // A4 again for the spans it reordered.  Enqueued optimistically before the
  // host knows whether there are giant runs: giant runs are disjoint from the
  // small/medium ones, so their refinement only appends list entries.
  // with sorted strings, runs whose units fit the stage are sorted in shared
  // memory and written back in place (k_fix_staged); the others (and perm-only
  // mode) take the global-memory kernels and the re-gather
  launch_fix_staged(kc, list_sm, L.cap_sm, st, d_perm, d_sorted_units, d_sorted_units ? d_sorted_offsets : nullptr,
                    S.sms, s, d_units, d_offsets);
  launch_fix_small(kc, list_sm, st, d_perm, d_units, d_offsets, S.sms, s, 0, d_sorted_units, d_sorted_offsets);
  launch_fix_medium(kc, list_sm, L.cap_sm, st, d_perm, d_units, d_offsets, S.sms, s, 0, d_sorted_offsets);
  if (d_sorted_units)
    launch_regather_runs(kc, list_sm, L.cap_sm, st, d_perm, d_units, d_offsets, d_sorted_units,
                         d_sorted_offsets, S.sms, s, 0, 0, true);
  HCHECK(cudaMemcpyAsync(h_state, st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  return HUSKY_OK;
}

// ------------------------------------------------------------- CUDA graphs
// A sort's launch sequence up to its synchronisation depends only on the
// arguments (buffers, n, coder, flags), so it is captured once into a CUDA
// graph and replayed when the same call repeats: one cudaGraphLaunch instead
// of ~15 launches and memsets (small sorts are launch-bound: C1's 1e5 strings
// move ~26 MB, 4 us at HBM speed).  Captured on a library stream, launched on
// the caller's; the DevState copy lands in a pinned buffer of the entry.
// Off while profiling (per-launch events), with HUSKY_DEBUG_SYNC, and with
// HUSKY_GRAPH=0.  LRU of kGraphCache entries per process.
struct GraphKey {
  int dev, coder, packed, compress, slab, pdl, skip;
  const void *units, *offsets, *perm, *su, *so, *ws;
  uint64_t n;
  size_t ws_bytes;
  bool operator==(const GraphKey &o) const { return memcmp(this, &o, sizeof *this) == 0; }
};
struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec = nullptr;
  DevState *h_state = nullptr;  // pinned
  uint32_t epoch = 0, slot = 0;
  uint64_t launches = 0, last_use = 0;
};
constexpr int kGraphCache = 16;
static std::mutex g_graph_mu;
static std::vector<GraphEntry> g_graphs;
static uint64_t g_graph_clock = 0;

static bool graphs_enabled() {
  const char *e = getenv("HUSKY_GRAPH");
  return !(e && e[0] == '0');
}

static cudaStream_t capture_stream(int dev) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  std::lock_guard<std::mutex> g(mu);
  if (!streams[dev & 63]) cudaStreamCreateWithFlags(&streams[dev & 63], cudaStreamNonBlocking);
  return streams[dev & 63];
}

static void free_entry(GraphEntry &e) {
  if (e.exec) cudaGraphExecDestroy(e.exec);
  if (e.h_state) cudaFreeHost(e.h_state);
  e.exec = nullptr;
  e.h_state = nullptr;
}

// the cached entry for `key`, captured now if absent (nullptr on failure:
// the caller falls back to direct launches)
static GraphEntry *graph_for(const GraphKey &key, Sorter &S, const MainFlags &F, void *su, int64_t *so) {
  std::lock_guard<std::mutex> g(g_graph_mu);
  for (auto &e : g_graphs)
    if (e.key == key) {
      e.last_use = ++g_graph_clock;
      return &e;
    }
  GraphEntry e;
  e.key = key;
  if (cudaMallocHost(&e.h_state, sizeof(DevState)) != cudaSuccess) return nullptr;
  cudaStream_t cs = capture_stream(key.dev);
  Sorter C = S;  // capture with a copy: the epoch / slot bookkeeping it ends with is the entry's
  C.s = cs;
  Profiler &P = profiler();
  uint64_t l0;
  {
    std::lock_guard<std::mutex> pg(P.mu);
    l0 = P.total_launches;
  }
  cudaGraph_t graph = nullptr;
  bool ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed) == cudaSuccess;
  husky_status st = ok ? enqueue_main(C, F, su, so, e.h_state) : HUSKY_ERR_CUDA;
  const bool ended = ok && cudaStreamEndCapture(cs, &graph) == cudaSuccess;
  ok = ok && st == HUSKY_OK && ended && graph && C.err == cudaSuccess &&
       cudaGraphInstantiate(&e.exec, graph, 0) == cudaSuccess;
  if (graph) cudaGraphDestroy(graph);
  cudaGetLastError();  // a failed capture leaves no sticky error; clear the last one
  {
    std::lock_guard<std::mutex> pg(P.mu);
    e.launches = P.total_launches - l0;
    P.total_launches = l0;  // counted again per replay
  }
  if (!ok) {
    free_entry(e);
    return nullptr;
  }
  e.epoch = C.epoch;
  e.slot = C.slot;
  e.last_use = ++g_graph_clock;
  if ((int)g_graphs.size() >= kGraphCache) {
    auto victim = std::min_element(g_graphs.begin(), g_graphs.end(),
                                   [](const GraphEntry &a, const GraphEntry &b) { return a.last_use < b.last_use; });
    free_entry(*victim);
    *victim = e;
    return &*victim;
  }
  g_graphs.push_back(e);
  return &g_graphs.back();
}

husky_status sort_impl(int coder, const void *d_units, const int64_t *d_offsets, uint64_t n,
                       uint32_t *d_perm, void *d_sorted_units, int64_t *d_sorted_offsets, void *d_ws,
                       size_t ws_bytes, husky_outcome *h_out, cudaStream_t s, bool allow_graph) {
  if (h_out) memset(h_out, 0, sizeof *h_out);
  if (!valid_coder(coder)) return fail(HUSKY_ERR_INVALID_ARG, "unknown coder %d", coder);
  if (n >= 0xFFFFFFFFull) return fail(HUSKY_ERR_INVALID_ARG, "n = %llu >= 2^32 - 1", (unsigned long long)n);
  if ((d_sorted_units == nullptr) != (d_sorted_offsets == nullptr))
    return fail(HUSKY_ERR_INVALID_ARG, "d_sorted_units and d_sorted_offsets must both be set or both NULL");
  if (n == 0) {
    if (h_out) { h_out->perfect = 1; h_out->domain_ok = 1; }
    if (d_sorted_offsets) HCHECK(cudaMemsetAsync(d_sorted_offsets, 0, 8, s));
    HCHECK(cudaStreamSynchronize(s));
    return HUSKY_OK;
  }
  if (!d_units || !d_offsets || !d_perm || !d_ws)
    return fail(HUSKY_ERR_INVALID_ARG, "null required pointer");
  if ((uintptr_t)d_ws % 256) return fail(HUSKY_ERR_INVALID_ARG, "workspace not 256-byte aligned");
  Layout L = make_layout(n);
  if (ws_bytes < L.total)
    return fail(HUSKY_ERR_WORKSPACE, "workspace %zu < required %zu", ws_bytes, L.total);

  Sorter S;
  // byte coders share the ASCII instantiation of every kernel but the encoder
  S.coder = kernel_coder(coder);
  S.units = d_units;
  S.offsets = d_offsets;
  S.n = n;
  S.perm = d_perm;
  S.ws = (uint8_t *)d_ws;
  S.L = L;
  S.s = s;
  S.sms = device_sm_count();
  S.st = S.at<DevState>(L.state);
  DevState *st = S.st;

  MainFlags F;
  F.coder = coder;
  F.kc = kernel_coder(coder);
  // the gather rebuilds short strings from ASCII / UNICODE codes only
  F.packed = n <= kPackMaxN && (coder == HUSKY_CODER_ASCII || coder == HUSKY_CODER_UNICODE);
  // alphabet compression of the sort's private keys (ASCII; HUSKY_ALPHA=0 off)
  F.compress = coder == HUSKY_CODER_ASCII && alpha_env();
  // slab records (ASCII / UNICODE) when sorted strings are produced and the
  // gather's random reads would miss L2: n > kSlabMinN strings (the offsets
  // alone then span >= 2x the 126 MB L2).  Every string's record when n > 2^28
  // (no packed lengths), else only the long strings'.  Below the threshold the
  // random reads mostly hit L2 and the records cost more than they save (C2:
  // encode 76 -> 119 us, gather 276 -> 332 us with them).  HUSKY_SLAB=1 / 0
  // forces them on / off (tests).
  F.slab = d_sorted_units && (coder == HUSKY_CODER_ASCII || coder == HUSKY_CODER_UNICODE) &&
           ((n > kSlabMinN && slab_env() != 0) || slab_env() == 1);
  F.pdl = pdl_enabled();
  // partial key sort (R19, ASCII codes only; HUSKY_SKIP=0 never, =2 always)
  // (the English coders share the ASCII kernels but not its field layout)
  F.skip = (coder == HUSKY_CODER_ASCII || coder == HUSKY_CODER_UNICODE) ? skip_env() : 0;

  DevState hs_local;
  const DevState *hs_src = &hs_local;
  GraphEntry *ge = nullptr;
  if (allow_graph && n < kHostPlanMinN && graphs_enabled() && !debug_sync() && profiler().on == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    GraphKey key;
    memset(&key, 0, sizeof key);
    key.dev = dev;
    key.coder = coder;
    key.packed = F.packed;
    key.compress = F.compress;
    key.slab = F.slab;
    key.pdl = F.pdl;
    key.skip = F.skip;
    key.units = d_units;
    key.offsets = d_offsets;
    key.perm = d_perm;
    key.su = d_sorted_units;
    key.so = d_sorted_offsets;
    key.ws = d_ws;
    key.n = n;
    key.ws_bytes = ws_bytes;
    ge = graph_for(key, S, F, d_sorted_units, d_sorted_offsets);
  }
  if (ge) {
    HCHECK(cudaGraphLaunch(ge->exec, s));
    S.epoch = ge->epoch;
    S.slot = ge->slot;
    {
      Profiler &P = profiler();
      std::lock_guard<std::mutex> pg(P.mu);
      P.total_launches += ge->launches;
    }
    hs_src = ge->h_state;
  } else {
    if (husky_status e = enqueue_main(S, F, d_sorted_units, d_sorted_offsets, &hs_local)) return e;
  }
  HCHECK(cudaStreamSynchronize(s));
  if (husky_status e = cuda_check("sort")) return e;
  HCHECK(S.err);
  DevState hs = *hs_src;
  if (hs.violations & kOffsetsBad) return fail(HUSKY_ERR_INVALID_ARG, "offsets are not non-decreasing");
  S.radix_passes = hs.np;
  debug_check_perm(d_perm, n, "fix-up", s);

  // ---- Off-domain input (a unit the coder masks inside a code window: the
  // code is not monotone there, readings R5 / R15): the general cleanup
  // (NEXT-4) -- Alg. 1's "cleanup repairs everything" restored by refining the
  // WHOLE array as one segment from unit 0 (an exact MSD string radix over
  // 7-unit windows, A6's machinery with whole-string comparisons).  Equal
  // strings have equal codes, so the stable code sort left them in index order.
  const bool general = domain_violation(coder, hs.violations);
  if (general) HCHECK(cudaMemsetAsync(&st->general, 1, 1, s));

  // ---- A6 giant-run refinement (rare: runs > 4096 strings with an inversion)
  const uint32_t n_giant = hs.n_giant;
  if (n_giant || general) {
    if (husky_status e = refine_giants(S, hs, d_sorted_units, d_sorted_offsets, &hs, general)) return e;
  }
  if (h_out) {
    h_out->perfect = !(hs.violations & kNotPerfect);
    h_out->domain_ok = !domain_violation(coder, hs.violations);
    h_out->n_in_runs = hs.n_in_runs;
    h_out->max_run = hs.max_run;
    for (int c = 0; c < 4; ++c) h_out->runs_by_class[c] = hs.runs_by_class[c];
    h_out->n_runs = hs.runs_total;
    h_out->refine_rounds = S.refine_rounds;
    h_out->radix_passes = S.radix_passes;
    h_out->keys_partitioned = (uint64_t)hs.np * n;
    h_out->exchange = HUSKY_EXCHANGE_NONE;
  }
  return HUSKY_OK;
}

// A6: refine the giant dirty runs found by the main scan (host-driven loop, one
// synchronisation per round), fix the small/medium sub-runs it appends to the
// lists, and re-gather the affected spans.  hs: DevState after the main pass;
// *out: DevState at the end.
static husky_status refine_giants(Sorter &S, const DevState &hs0, void *d_sorted_units, int64_t *d_sorted_offsets,
                                  DevState *out, bool general) {
  const int coder = S.coder;
  const Layout &L = S.L;
  DevState *st = S.st;
  cudaStream_t s = S.s;
  const void *d_units = S.units;
  const int64_t *d_offsets = S.offsets;
  uint32_t *d_perm = S.perm;
  const uint64_t n = S.n;
  uint32_t *run_start = S.at<uint32_t>(L.run_start), *run_end = S.at<uint32_t>(L.run_end);
  uint8_t *dirty = S.at<uint8_t>(L.dirty);
  uint2 *list_sm = S.at<uint2>(L.list_sm), *list_g = S.at<uint2>(L.list_g);
  // small/medium entries already fixed (and re-gathered) by the main pass
  const uint32_t s0 = hs0.n_small, m0 = hs0.n_medium;
  uint32_t n_giant = hs0.n_giant;
  HostSnap snap;

  struct Seg { uint32_t start, len, from; };
  std::vector<Seg> queue;
  std::vector<uint2> giant_spans;  // top-level giant runs: re-gathered at the end
  if (general) {  // the whole array, nothing known in common
    queue.push_back({0u, (uint32_t)n, 0u});
    giant_spans.push_back(make_uint2(0u, (uint32_t)n));
  } else {
    std::vector<uint2> g(n_giant);
    HCHECK(cudaMemcpy(g.data(), list_g, n_giant * sizeof(uint2), cudaMemcpyDeviceToHost));
    // units fixed by equal codes: the sort's run rule (R6 / R19)
    const uint32_t s0 = hs0.seq_units ? hs0.seq_units : (uint32_t)(coder == HUSKY_CODER_ASCII ? 9 : 3);
    for (auto &x : g) queue.push_back({x.x, x.y, s0});
    giant_spans = g;
  }
  const uint32_t win = coder == HUSKY_CODER_ASCII ? 7 : 3;
  for (size_t qi = 0; qi < queue.size(); ++qi) {
    Seg seg = queue[qi];
    S.refine_rounds++;
    uint32_t *perm_seg = d_perm + seg.start;
    // reset histogram + segment scratch
    HCHECK(cudaMemsetAsync(st->hist, 0, sizeof(st->hist), s));
    HCHECK(cudaMemsetAsync(&st->trivial_mask, 0, 4, s));
    HCHECK(cudaMemsetAsync(&st->seg_L, 0xFF, 4, s));
    HCHECK(cudaMemsetAsync(&st->seg_has_short, 0, 4, s));
    launch_seg_prep(coder, perm_seg, seg.len, d_units, d_offsets, seg.from, st, s);
    launch_seg_key2(coder, perm_seg, seg.len, d_units, d_offsets, seg.from, S.keysA(), st, S.sms, s);
    launch_hist_scan(seg.len, st, s);
    uint32_t info[2];
    HCHECK(cudaMemcpyAsync(&snap, &st->trivial_mask, sizeof snap, cudaMemcpyDeviceToHost, s));
    HCHECK(cudaMemcpyAsync(info, &st->seg_L, 8, cudaMemcpyDeviceToHost, s));
    HCHECK(cudaStreamSynchronize(s));
    uint32_t Lcur = info[1] ? seg.from : info[0];
    // R19 inside the refinement (ASCII windows): leave the tag and the window's
    // last two units (digits 0..2) unsorted when the sorted units' entropy makes
    // the extra equal pairs rare; every pair equal under the mask is then
    // resolved by the fix-ups (or the next round, from two units earlier)
    uint32_t trivial = snap.trivial_mask, adv = win;
    unsigned long long refmask = ~0ull;
    if (coder == HUSKY_CODER_ASCII && skip_env() != 0 && seg.len >= 4096) {
      std::vector<uint32_t> hh(8 * kBins);
      HCHECK(cudaMemcpy(hh.data(), st->hist, hh.size() * 4, cudaMemcpyDeviceToHost));
      double H = 0.0;
      for (int d = 3; d < 8; ++d)
        for (int b = 0; b < kBins; ++b) {
          const double p = (double)hh[d * kBins + b] / (double)seg.len;
          if (p > 0.0) H -= p * std::log2(p);
        }
      const double extra = 0.5 * (double)seg.len * (double)seg.len * std::exp2(-H);
      // (by the rule only, never forced: a degenerate segment -- identical
      // strings, H = 0 -- must keep the tag, or its rounds would not end)
      if (extra < 1e-2 * (double)seg.len) {
        trivial |= 0x07u;
        refmask = ~0xFFFFFFull;
        adv = win - 2;
      }
    }
    uint64_t *sorted_key2 = nullptr;
    // payload: the segment's perm entries; sorted back into perm_seg
    if (husky_status e = S.radix(S.keysA(), perm_seg, seg.len, trivial, perm_seg, S.at<uint32_t>(L.vals),
                                 &sorted_key2))
      return e;
    debug_check_perm(d_perm, n, "refine radix", s);
    // sub-runs of equal key with tag == cap are still ambiguous
    HCHECK(cudaMemsetAsync(dirty, 0, seg.len / 2 + 1, s));
    HCHECK(cudaMemsetAsync(&st->n_giant, 0, 4, s));
    launch_runs_scan(coder, 1, sorted_key2, seg.len, perm_seg, d_units, d_offsets, seg.start, run_start,
                     run_end, dirty, st, S.lb_scan(), S.next_counter(), S.next_epoch(), s, refmask);
    launch_runs_classify(run_start, run_end, dirty, st, list_sm, L.cap_sm, list_g, false, S.sms, s);
    HCHECK(cudaMemcpyAsync(&n_giant, &st->n_giant, 4, cudaMemcpyDeviceToHost, s));
    HCHECK(cudaStreamSynchronize(s));
    if (husky_status e = cuda_check("refine")) return e;
    if (n_giant) {
      std::vector<uint2> g(n_giant);
      HCHECK(cudaMemcpy(g.data(), list_g, n_giant * sizeof(uint2), cudaMemcpyDeviceToHost));
      for (auto &x : g) queue.push_back({x.x, x.y, Lcur + adv});
    }
  }

  // ---- A5 fix-up of the small / medium sub-runs the refinement appended
  launch_fix_small(coder, list_sm, st, d_perm, d_units, d_offsets, S.sms, s, s0);
  launch_fix_staged(coder, list_sm, L.cap_sm, st, d_perm, nullptr, nullptr, S.sms, s, d_units, d_offsets, m0);
  launch_fix_medium(coder, list_sm, L.cap_sm, st, d_perm, d_units, d_offsets, S.sms, s, m0);
  debug_check_perm(d_perm, n, "refine fix-up", s);

  // ---- A4 (again) for the spans whose order the fix-up changed
  if (d_sorted_units) {
    auto dbg_so = [&](const char *tag) {
      if (!debug_sync()) return;
      int64_t v[2] = {0, 0};
      cudaStreamSynchronize(s);
      cudaMemcpy(v, d_sorted_offsets, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(v + 1, d_sorted_offsets + n, 8, cudaMemcpyDeviceToHost);
      fprintf(stderr, "[husky] %s: sorted_offsets[0]=%lld [n]=%lld giants=%zu first=(%u,%u)\n", tag, (long long)v[0],
              (long long)v[1], giant_spans.size(), giant_spans.empty() ? 0u : giant_spans[0].x,
              giant_spans.empty() ? 0u : giant_spans[0].y);
    };
    // Giant spans first: the refinement reordered them wholesale, so the
    // offsets inside them (and hence the bases of the small/medium sub-runs it
    // produced) are only valid after the whole span is gathered again.  The
    // span's own base and length never change.
    for (auto &g : giant_spans)
      launch_gather(coder, d_perm + g.x, g.y, d_units, d_offsets, d_sorted_units, d_sorted_offsets + g.x,
                    S.lb_scan(), S.next_counter(), S.next_epoch(), s, d_sorted_offsets + g.x);
    dbg_so("after giant re-gather");
    launch_regather_runs(coder, list_sm, L.cap_sm, st, d_perm, d_units, d_offsets, d_sorted_units,
                         d_sorted_offsets, S.sms, s, s0, m0);
    dbg_so("after run re-gather");
  }

  HCHECK(cudaMemcpyAsync(out, st, sizeof *out, cudaMemcpyDeviceToHost, s));
  HCHECK(cudaStreamSynchronize(s));
  if (husky_status e = cuda_check("refine/fixup/gather")) return e;
  return HUSKY_OK;
}

}  // namespace husky

using namespace husky;

namespace husky {
// husky_encode's violation words: one per concurrent call that reads them
// back (slots 0..62, claimed per device under a bit mask), slot 63 is the
// shared sink of calls that do not (written, never read)
constexpr int kEncodeSlots = 64;
__device__ uint32_t g_encode_viol[kEncodeSlots];
static std::atomic<unsigned long long> g_encode_busy[64];

static int claim_encode_slot(int dev) {
  std::atomic<unsigned long long> &m = g_encode_busy[dev & 63];
  for (;;) {
    unsigned long long cur = m.load(std::memory_order_acquire);
    for (int i = 0; i < kEncodeSlots - 1; ++i)
      if (!(cur & (1ull << i)) && m.compare_exchange_weak(cur, cur | (1ull << i), std::memory_order_acq_rel))
        return i;
    std::this_thread::yield();
  }
}
static void release_encode_slot(int dev, int slot) {
  g_encode_busy[dev & 63].fetch_and(~(1ull << slot), std::memory_order_acq_rel);
}
}

extern "C" {

static const char *kStageNames[ST_COUNT] = {"encode", "hist_scan", "radix_pass", "runs_scan", "runs_classify",
                                            "fix_small", "fix_medium", "refine", "gather", "multi"};

void husky_profile_enable(int on) {
  Profiler &P = profiler();
  P.flush();
  std::lock_guard<std::mutex> g(P.mu);
  P.on = on == 2 ? 2 : (on != 0 ? 1 : 0);
}

void husky_profile_reset(void) {
  Profiler &P = profiler();
  P.flush();
  std::lock_guard<std::mutex> g(P.mu);
  for (int i = 0; i < ST_COUNT; ++i) { P.ms[i] = 0; P.launches[i] = 0; P.elems[i] = 0; }
  P.log.clear();
}

int husky_profile_launches(int *stages, uint64_t *elems, double *ms, int max_records) {
  Profiler &P = profiler();
  P.flush();
  std::lock_guard<std::mutex> g(P.mu);
  const int k = (int)std::min<size_t>(P.log.size(), (size_t)(max_records > 0 ? max_records : 0));
  for (int i = 0; i < k; ++i) {
    if (stages) stages[i] = P.log[i].stage;
    if (elems) elems[i] = P.log[i].elems;
    if (ms) ms[i] = P.log[i].ms;
  }
  return (int)P.log.size();
}

int husky_profile_read(double *ms, uint64_t *launches, uint64_t *elems, int max_stages) {
  Profiler &P = profiler();
  P.flush();
  std::lock_guard<std::mutex> g(P.mu);
  int k = max_stages < ST_COUNT ? max_stages : ST_COUNT;
  for (int i = 0; i < k; ++i) {
    if (ms) ms[i] = P.ms[i];
    if (launches) launches[i] = P.launches[i];
    if (elems) elems[i] = P.elems[i];
  }
  return ST_COUNT;
}

const char *husky_profile_stage_name(int stage) {
  return stage >= 0 && stage < ST_COUNT ? kStageNames[stage] : "";
}

uint64_t husky_launch_count(void) {
  Profiler &P = profiler();
  std::lock_guard<std::mutex> g(P.mu);
  return P.total_launches;
}

size_t husky_unit_bytes(int coder) {
  return coder_unit_bytes(coder);
}

const char *husky_last_error(void) { return g_last_error.c_str(); }

husky_status husky_encode(int coder, const void *d_units, const int64_t *d_offsets, uint64_t n,
                          uint64_t *d_codes, int32_t *h_perfect, void *stream) {
  if (!valid_coder(coder)) return fail(HUSKY_ERR_INVALID_ARG, "unknown coder %d", coder);
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    if (h_perfect) *h_perfect = 1;
    return HUSKY_OK;
  }
  if (!d_units || !d_offsets || !d_codes) return fail(HUSKY_ERR_INVALID_ARG, "null required pointer");
  // violation word: a private slot while this call reads it back (concurrent
  // calls on one device do not share it), the shared sink otherwise
  uint32_t *words = nullptr;
  HCHECK(cudaGetSymbolAddress((void **)&words, g_encode_viol));
  int dev = 0;
  HCHECK(cudaGetDevice(&dev));
  const int slot = h_perfect ? claim_encode_slot(dev) : kEncodeSlots - 1;
  uint32_t *viol = words + slot;
  husky_status rc = HUSKY_OK;
  uint32_t v = 0;
  cudaError_t e = h_perfect ? cudaMemsetAsync(viol, 0, 4, s) : cudaSuccess;
  if (e == cudaSuccess) {
    launch_encode(coder, d_units, d_offsets, n, d_codes, viol, device_sm_count(), s);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && h_perfect) e = cudaMemcpyAsync(&v, viol, 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && h_perfect) e = cudaStreamSynchronize(s);
  if (h_perfect) release_encode_slot(dev, slot);
  if (e != cudaSuccess) return fail(HUSKY_ERR_CUDA, "encode: %s", cudaGetErrorString(e));
  if (h_perfect) {
    if (v & kOffsetsBad) return fail(HUSKY_ERR_INVALID_ARG, "offsets are not non-decreasing");
    *h_perfect = !(v & kNotPerfect);
  }
  return rc;
}

husky_status husky_sort_workspace(int coder, uint64_t n, uint64_t total_units, size_t *bytes) {
  (void)total_units;
  if (!valid_coder(coder)) return fail(HUSKY_ERR_INVALID_ARG, "unknown coder %d", coder);
  if (!bytes) return fail(HUSKY_ERR_INVALID_ARG, "bytes is NULL");
  *bytes = make_layout(n).total;
  return HUSKY_OK;
}

husky_status husky_sort(int coder, const void *d_units, const int64_t *d_offsets, uint64_t n,
                        uint32_t *d_perm, void *d_sorted_units, int64_t *d_sorted_offsets, void *d_ws,
                        size_t ws_bytes, husky_outcome *h_out, void *stream) {
  return checked_result(sort_impl(coder, d_units, d_offsets, n, d_perm, d_sorted_units, d_sorted_offsets, d_ws,
                                   ws_bytes, h_out, (cudaStream_t)stream),
                         "husky_sort");
}

// host-buffer variant: [device units | device offsets | device perm | sorted units | sorted offsets | sort ws]
static size_t host_layout(int coder, uint64_t n, uint64_t total_units, size_t *o_units, size_t *o_off,
                          size_t *o_perm, size_t *o_su, size_t *o_so, size_t *o_ws) {
  size_t w = husky_unit_bytes(coder), off = 0;
  auto take = [&](size_t b) { size_t o = off; off = align_up(off + b, 256); return o; };
  *o_units = take(total_units * w + 16);
  *o_off = take((n + 1) * 8);
  *o_perm = take(n * 4 + 4);
  *o_su = take(total_units * w + 16);
  *o_so = take((n + 1) * 8);
  *o_ws = take(make_layout(n).total);
  return off;
}

// husky_sort_host_many: `depth` input slots [units | offsets | sort ws] and
// depth + 1 output slots [perm | sorted units | sorted offsets].  The extra
// output slot lets batch b+1 be sorted while batch b's outputs are still on
// their way to the host (with one slot of each, the next sort had to wait for
// the whole copy-out: C5 e2e ~785 ms per batch, of which the sort is ~91).
struct ManyLayout {
  size_t units, off, ws, in_slice;  // offsets within an input slot
  size_t perm, su, so, out_slice;   // offsets within an output slot
  size_t total(int depth) const { return (size_t)depth * in_slice + (size_t)(depth + 1) * out_slice; }
};
static ManyLayout many_layout(int coder, uint64_t n, uint64_t total_units) {
  const size_t w = husky_unit_bytes(coder);
  ManyLayout m{};
  size_t off = 0;
  auto take = [&](size_t b) { size_t o = off; off = align_up(off + b, 256); return o; };
  m.units = take(total_units * w + 16);
  m.off = take((n + 1) * 8);
  m.ws = take(make_layout(n).total);
  m.in_slice = off;
  off = 0;
  m.perm = take(n * 4 + 4);
  m.su = take(total_units * w + 16);
  m.so = take((n + 1) * 8);
  m.out_slice = off;
  return m;
}

husky_status husky_sort_host_workspace(int coder, uint64_t n, uint64_t total_units, size_t *bytes) {
  if (!valid_coder(coder)) return fail(HUSKY_ERR_INVALID_ARG, "unknown coder %d", coder);
  if (!bytes) return fail(HUSKY_ERR_INVALID_ARG, "bytes is NULL");
  size_t a, b, c, d, e, f;
  *bytes = host_layout(coder, n, total_units, &a, &b, &c, &d, &e, &f);
  return HUSKY_OK;
}

husky_status husky_sort_host(int coder, const void *h_units, const int64_t *h_offsets, uint64_t n,
                             uint32_t *h_perm, void *h_sorted_units, int64_t *h_sorted_offsets,
                             void *d_ws, size_t ws_bytes, husky_outcome *h_out, void *stream) {
  if (!valid_coder(coder)) return fail(HUSKY_ERR_INVALID_ARG, "unknown coder %d", coder);
  if (!h_offsets || (n && (!h_perm || !h_units)) || !d_ws)
    return fail(HUSKY_ERR_INVALID_ARG, "null required pointer");
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t total = n ? (uint64_t)(h_offsets[n] - h_offsets[0]) : 0;
  if (n && h_offsets[n] < h_offsets[0]) return fail(HUSKY_ERR_INVALID_ARG, "offsets are not non-decreasing");
  size_t o_units, o_off, o_perm, o_su, o_so, o_ws;
  size_t need = host_layout(coder, n, total, &o_units, &o_off, &o_perm, &o_su, &o_so, &o_ws);
  if (ws_bytes < need) return fail(HUSKY_ERR_WORKSPACE, "workspace %zu < required %zu", ws_bytes, need);
  uint8_t *ws = (uint8_t *)d_ws;
  size_t w = husky_unit_bytes(coder);
  // the device offsets are rebased to 0 so the device unit copy starts at unit 0
  int64_t base = n ? h_offsets[0] : 0;
  HCHECK(cudaMemcpyAsync(ws + o_units, (const uint8_t *)h_units + base * w, total * w, cudaMemcpyHostToDevice, s));
  HCHECK(cudaMemcpyAsync(ws + o_off, h_offsets, (n + 1) * 8, cudaMemcpyHostToDevice, s));
  const void *du = ws + o_units;
  if (base != 0) du = (const uint8_t *)du - base * (int64_t)w;  // offsets index the original buffer
  bool want_units = h_sorted_units != nullptr && h_sorted_offsets != nullptr;
  husky_status st = sort_impl(coder, du, (const int64_t *)(ws + o_off), n, (uint32_t *)(ws + o_perm),
                              want_units ? (void *)(ws + o_su) : nullptr,
                              want_units ? (int64_t *)(ws + o_so) : nullptr, ws + o_ws, ws_bytes - o_ws,
                              h_out, s);
  if (st != HUSKY_OK) return st;
  HCHECK(cudaMemcpyAsync(h_perm, ws + o_perm, n * 4, cudaMemcpyDeviceToHost, s));
  if (want_units) {
    HCHECK(cudaMemcpyAsync(h_sorted_units, ws + o_su, total * w, cudaMemcpyDeviceToHost, s));
    HCHECK(cudaMemcpyAsync(h_sorted_offsets, ws + o_so, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
  }
  HCHECK(cudaStreamSynchronize(s));
  return HUSKY_OK;
}

// husky_sort_host_many, one issuing thread and three streams: host->device
// copies (sh), kernels (sc) and device->host copies (sd); batch b uses input
// slot b % depth and output slot b % (depth + 1).  Batch b+1's input copy is
// enqueued before batch b is sorted (sort_impl synchronises sc once per sort)
// and batch b's output copy right after, so in steady state both copy
// directions and the SMs work on three different batches.  Events order the
// reuse of a slot: an input slot is overwritten only after the sort that read
// it, an output slot only after the copy-out that read it.
static husky_status host_many_pipelined(int coder, int k, const void *const *h_units,
                                        const int64_t *const *h_offsets, const uint64_t *n,
                                        uint32_t *const *h_perm, void *const *h_sorted_units,
                                        int64_t *const *h_sorted_offsets, int depth, uint8_t *ws,
                                        const ManyLayout &m, husky_outcome *h_out) {
  const size_t w = husky_unit_bytes(coder);
  const int odepth = depth + 1;
  cudaStream_t sh = nullptr, sc = nullptr, sd = nullptr;
  std::vector<cudaEvent_t> evH(depth, nullptr), evC(depth, nullptr), evO(odepth, nullptr), evD(odepth, nullptr);
  husky_status st = HUSKY_OK;
  auto cleanup = [&]() {
    if (sh) cudaStreamSynchronize(sh);
    if (sc) cudaStreamSynchronize(sc);
    if (sd) cudaStreamSynchronize(sd);
    for (auto *v : {&evH, &evC, &evO, &evD})
      for (cudaEvent_t e : *v)
        if (e) cudaEventDestroy(e);
    if (sh) cudaStreamDestroy(sh);
    if (sc) cudaStreamDestroy(sc);
    if (sd) cudaStreamDestroy(sd);
  };
#define HM_CHECK(expr)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      st = fail(HUSKY_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_));                   \
      cleanup();                                                                            \
      return st;                                                                            \
    }                                                                                       \
  } while (0)
  HM_CHECK(cudaStreamCreateWithFlags(&sh, cudaStreamNonBlocking));
  HM_CHECK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
  HM_CHECK(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
  for (int i = 0; i < depth; ++i) {
    HM_CHECK(cudaEventCreateWithFlags(&evH[i], cudaEventDisableTiming));
    HM_CHECK(cudaEventCreateWithFlags(&evC[i], cudaEventDisableTiming));
  }
  for (int i = 0; i < odepth; ++i) {
    HM_CHECK(cudaEventCreateWithFlags(&evO[i], cudaEventDisableTiming));
    HM_CHECK(cudaEventCreateWithFlags(&evD[i], cudaEventDisableTiming));
  }
  auto total_of = [&](int b) { return n[b] ? (uint64_t)(h_offsets[b][n[b]] - h_offsets[b][0]) : 0ull; };
  // ONE layout for every batch, sized by the largest batch (a slot's regions
  // never move between batches)
  auto in_base = [&](int b) { return ws + m.in_slice * (size_t)(b % depth); };
  auto out_base = [&](int b) { return ws + m.in_slice * (size_t)depth + m.out_slice * (size_t)(b % odepth); };
  std::vector<bool> used_in(depth, false), used_out(odepth, false);
  auto issue_in = [&](int b) -> cudaError_t {
    const int sl = b % depth;
    uint8_t *base = in_base(b);
    cudaError_t e = cudaSuccess;
    if (used_in[sl]) e = cudaStreamWaitEvent(sh, evC[sl], 0);  // the previous sort of this slot has read its inputs
    const int64_t b0 = n[b] ? h_offsets[b][0] : 0;
    if (e == cudaSuccess && total_of(b))
      e = cudaMemcpyAsync(base + m.units, (const uint8_t *)h_units[b] + b0 * w, total_of(b) * w,
                          cudaMemcpyHostToDevice, sh);
    if (e == cudaSuccess) e = cudaMemcpyAsync(base + m.off, h_offsets[b], (n[b] + 1) * 8, cudaMemcpyHostToDevice, sh);
    if (e == cudaSuccess) e = cudaEventRecord(evH[sl], sh);
    return e;
  };
  if (k > 0) HM_CHECK(issue_in(0));
  for (int b = 0; b < k; ++b) {
    const int sl = b % depth, so_ = b % odepth;
    uint8_t *ib = in_base(b), *ob = out_base(b);
    if (b + 1 < k && depth > 1) HM_CHECK(issue_in(b + 1));  // (one input slot: after this sort)
    if (n[b] && h_offsets[b][n[b]] < h_offsets[b][0]) {
      st = fail(HUSKY_ERR_INVALID_ARG, "batch %d: offsets are not non-decreasing", b);
      cleanup();
      return st;
    }
    HM_CHECK(cudaStreamWaitEvent(sc, evH[sl], 0));
    if (used_out[so_]) HM_CHECK(cudaStreamWaitEvent(sc, evD[so_], 0));  // this output slot copied out
    const int64_t b0 = n[b] ? h_offsets[b][0] : 0;
    const void *du = ib + m.units;
    if (b0 != 0) du = (const uint8_t *)du - b0 * (int64_t)w;  // offsets index the original buffer
    const bool want_units = h_sorted_units && h_sorted_offsets && h_sorted_units[b] && h_sorted_offsets[b];
    st = sort_impl(coder, du, (const int64_t *)(ib + m.off), n[b], (uint32_t *)(ob + m.perm),
                   want_units ? (void *)(ob + m.su) : nullptr, want_units ? (int64_t *)(ob + m.so) : nullptr,
                   ib + m.ws, m.in_slice - m.ws, h_out ? h_out + b : nullptr, sc);
    if (st != HUSKY_OK) {
      cleanup();
      return st;
    }
    HM_CHECK(cudaEventRecord(evC[sl], sc));
    HM_CHECK(cudaEventRecord(evO[so_], sc));
    HM_CHECK(cudaStreamWaitEvent(sd, evO[so_], 0));
    if (n[b]) HM_CHECK(cudaMemcpyAsync(h_perm[b], ob + m.perm, n[b] * 4, cudaMemcpyDeviceToHost, sd));
    if (want_units) {
      if (total_of(b))
        HM_CHECK(cudaMemcpyAsync(h_sorted_units[b], ob + m.su, total_of(b) * w, cudaMemcpyDeviceToHost, sd));
      HM_CHECK(cudaMemcpyAsync(h_sorted_offsets[b], ob + m.so, (n[b] + 1) * 8, cudaMemcpyDeviceToHost, sd));
    }
    HM_CHECK(cudaEventRecord(evD[so_], sd));
    used_in[sl] = true;
    used_out[so_] = true;
    if (b + 1 < k && depth == 1) HM_CHECK(issue_in(b + 1));
  }
#undef HM_CHECK
  cudaError_t e = cudaStreamSynchronize(sd);
  if (e == cudaSuccess) e = cudaStreamSynchronize(sh);
  cleanup();
  if (e != cudaSuccess) return fail(HUSKY_ERR_CUDA, "husky_sort_host_many: %s", cudaGetErrorString(e));
  return HUSKY_OK;
}

husky_status husky_sort_host_many_workspace(int coder, uint64_t n_max, uint64_t units_max, int depth,
                                            size_t *bytes) {
  if (!valid_coder(coder)) return fail(HUSKY_ERR_INVALID_ARG, "unknown coder %d", coder);
  if (!bytes || depth < 1 || depth > 16) return fail(HUSKY_ERR_INVALID_ARG, "bad arguments");
  *bytes = many_layout(coder, n_max, units_max).total(depth);
  return HUSKY_OK;
}

husky_status husky_sort_host_many(int coder, int k, const void *const *h_units, const int64_t *const *h_offsets,
                                  const uint64_t *n, uint32_t *const *h_perm, void *const *h_sorted_units,
                                  int64_t *const *h_sorted_offsets, int depth, void *d_ws, size_t ws_bytes,
                                  husky_outcome *h_out) {
  if (!valid_coder(coder)) return fail(HUSKY_ERR_INVALID_ARG, "unknown coder %d", coder);
  if (k < 0 || depth < 1 || depth > 16 || (k && (!h_units || !h_offsets || !n || !h_perm)) || !d_ws)
    return fail(HUSKY_ERR_INVALID_ARG, "bad arguments");
  if ((uintptr_t)d_ws % 256) return fail(HUSKY_ERR_INVALID_ARG, "workspace not 256-byte aligned");
  uint64_t n_max = 0, u_max = 0;
  for (int b = 0; b < k; ++b) {
    if (!h_offsets[b]) return fail(HUSKY_ERR_INVALID_ARG, "batch %d: null offsets", b);
    n_max = std::max<uint64_t>(n_max, n[b]);
    if (n[b]) u_max = std::max<uint64_t>(u_max, (uint64_t)(h_offsets[b][n[b]] - h_offsets[b][0]));
  }
  const ManyLayout m = many_layout(coder, n_max, u_max);
  if (ws_bytes < m.total(depth))
    return fail(HUSKY_ERR_WORKSPACE, "workspace %zu < required %zu", ws_bytes, m.total(depth));
  return host_many_pipelined(coder, k, h_units, h_offsets, n, h_perm, h_sorted_units, h_sorted_offsets, depth,
                             (uint8_t *)d_ws, m, h_out);
}

}  // extern "C"
