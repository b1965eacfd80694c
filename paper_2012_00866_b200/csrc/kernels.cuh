// kernels.cuh -- launch wrappers shared between the kernel files and the host
// orchestration (husky.cu).  Not part of the ABI.
#pragma once
#include "husky_internal.cuh"
#include "profile.h"

namespace husky {

int device_sm_count();  // husky.cu

// A1 encode
// 256 threads x 4 strings in flight per CTA iteration, persistent grid
#ifndef HUSKY_ENC_BPS
#define HUSKY_ENC_BPS 8
#endif
constexpr int kEncThreads = 256, kEncBlocksPerSM = HUSKY_ENC_BPS;  // grid (resident: HUSKY_ENC_MINB)
// packed (nullable, n <= 2^28): also writes the initial radix payload
// index | min(len, 15) << 28, so the gather knows short strings' lengths
// without a random offsets read.  slab (nullable, ASCII / UNICODE): the
// 16-byte string records the main gather reads (encode.cu); slab_all: a record
// for every string, else only for strings longer than PL.  viol: violation
// bits (OR-ed).
constexpr uint64_t kPackMaxN = 1ull << 28;
// slab records only above this many strings (offsets >= 2x the L2)
constexpr uint64_t kSlabMinN = 1ull << 25;
void launch_encode(int coder, const void *units, const int64_t *offsets, uint64_t n, uint64_t *codes,
                   uint32_t *viol, int num_sms, cudaStream_t s, uint32_t *packed = nullptr, uint4 *slab = nullptr,
                   bool slab_all = false, uint32_t *alpha = nullptr);
// 8 digit histograms (8-bit digits) of n keys into DevState::hist (accumulates)
void launch_hist_slots(const uint64_t *keys, uint64_t n, DevState *st, int num_sms, cudaStream_t s);
// histograms + k_hist_scan + the pass plan fused (the last CTA scans and plans)
// compress: ASCII codes with DevState::alpha from the encoder -- the keys are
// re-packed in place (alphabet compression, husky_internal.cuh) when that
// saves a pass, before the histograms
// skip: leave the lowest varying digit unsorted (0 never, 1 by the entropy
// rule, 2 always; ASCII codes only, R19); def_s / def_pl: the
// coder's run rule (DevState::seq_units / short_len when nothing is skipped)
void launch_hist_plan(const uint64_t *keys, uint64_t n, DevState *st, uint64_t *keysA, uint64_t *keysB,
                      int num_sms, cudaStream_t s, bool compress = false, int skip = 0, uint32_t def_s = 0,
                      uint32_t def_pl = 0, bool unicode = false);

// A2 onesweep radix
// 512 threads x 12 keys = 6144-key tiles, 92 KB smem (keys, payloads, u16
// positions, u16 per-warp counters), <= 64 registers -> 2 CTAs (32 warps) per
// SM.  Large tiles keep the number of tiles in flight low: each look-back round
// trip queues behind the SM's bulk DRAM loads (~1 us under load), so the walk
// length (tiles between a tile and the inclusive-prefix frontier) is what
// bounds the pass.  Measured on C2 per sort: 8 keys/thread
// 1115 us, 10: 1067, 12: 1057, 14: 1075, 16 (1 CTA/SM): 1199.
#ifndef HUSKY_RADIX_ITEMS
#define HUSKY_RADIX_ITEMS 12
#endif
#ifndef HUSKY_RADIX_THREADS
#define HUSKY_RADIX_THREADS 512
#endif
constexpr int kRadixThreads = HUSKY_RADIX_THREADS, kRadixItems = HUSKY_RADIX_ITEMS,
              kRadixTile = kRadixThreads * kRadixItems;
// Small inputs (n below kRadixSmallN) use 2048-key tiles (4 keys per thread):
// a 1e5-string sort has 17 large tiles for 148 SMs.  Measured per C2-like sort
// (small / large tiles): 1e5 140 / 165 us, 3e5 158 / 174, 1e6 248 / 235,
// 2e6 367 / 321 us -- the crossover lies between 3e5 and 1e6
constexpr int kRadixItemsSmall = 4;
#ifndef HUSKY_RADIX_SMALL_N
#define HUSKY_RADIX_SMALL_N 500000
#endif
constexpr uint64_t kRadixSmallN = HUSKY_RADIX_SMALL_N;
inline int radix_items(uint64_t n) { return n < kRadixSmallN ? kRadixItemsSmall : kRadixItems; }
inline uint64_t radix_tiles(uint64_t n) {
  const uint64_t t = (uint64_t)kRadixThreads * radix_items(n);
  return (n + t - 1) / t;
}
inline uint64_t radix_tiles_large(uint64_t n) { return (n + kRadixTile - 1) / kRadixTile; }
// look-back words: one per (tile, digit), tile-major
inline uint64_t radix_lb_words(uint64_t n) { return radix_tiles(n) * kBins + 2; }
// exclusive scans of DevState::hist -> digit_start, trivial_mask for the
// host-planned passes (the pass slots get theirs from launch_hist_plan)
void launch_hist_scan(uint64_t n, DevState *st, cudaStream_t s);
// One stable LSD pass on digit `digit` (bits 8*digit..8*digit+7).  vals_in == NULL
// synthesises payload = index.  lb: radix_tiles(n)*256 look-back words.
void launch_onesweep(const uint64_t *keys_in, const uint32_t *vals_in, uint64_t *keys_out,
                     uint32_t *vals_out, uint64_t n, int digit, DevState *st,
                     unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, cudaStream_t s);
void launch_iota(uint32_t *perm, uint64_t n, cudaStream_t s);
// Device-planned passes (no host sync): the last CTA of
// launch_hist_plan turns the trivial-digit mask into DevState::np / pass_digit /
// sorted_keys; slots 0..7 are launched unconditionally and resolve their digit
// and ping-pong buffers on device (the last planned pass writes vals_final);
// finalize copies the payload when np == 0.
void launch_onesweep_slot(int slot, uint64_t *keysA, uint64_t *keysB, const uint32_t *vals_init,
                          uint32_t *vals_final, uint32_t *vals_tmp, uint64_t n, DevState *st,
                          unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, cudaStream_t s);
void launch_radix_finalize(const DevState *st, const uint32_t *vals_init, uint32_t *vals_final, uint64_t n,
                           cudaStream_t s);

struct Sorter;


// A3 run detection (single-pass scan with decoupled look-back)
constexpr int kScanThreads = 512, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
// padded smem staging size of k_runs_scan (one pad u64 every 8)
constexpr int kScanKP = kScanTile + 2 + (kScanTile + 2) / 8 + 1;
inline uint64_t scan_tiles(uint64_t n) { return (n + kScanTile - 1) / kScanTile; }
// mode 0: keys are husky codes; a pair inside a run is checked with the exact
//         equal-code comparator (strings via perm -> offsets -> units).
// mode 1: keys are refinement keys; a pair is unresolved iff its tag is the cap.
void launch_runs_scan(int coder, int mode, const uint64_t *keys, uint64_t n, const uint32_t *perm,
                      const void *units, const int64_t *offsets, uint32_t base, uint32_t *run_start,
                      uint32_t *run_end, uint8_t *dirty, DevState *st, unsigned long long *lb,
                      uint32_t *tile_counter, uint32_t epoch, cudaStream_t s, unsigned long long refmask = ~0ull);
void launch_runs_classify(const uint32_t *run_start, const uint32_t *run_end, const uint8_t *dirty,
                          DevState *st, uint2 *list_sm, uint64_t cap_sm, uint2 *list_g,
                          bool count_stats, int num_sms, cudaStream_t s);

// A5 fix-up of dirty runs (lists filled by classify; counts read on device)
// entries [first, count) of each list (first > 0: the round after a refinement)
// staged: the main pass with sorted strings -- every medium run whose units
// fit kFixStageBytes is sorted in shared memory and written back in place
// (fixup.cu); k_fix_medium and the re-gather then skip those runs (staged_so =
// the sorted offsets), else they take every run (staged_so NULL).  Small runs
// always take k_fix_small.
constexpr int kFixStageBytes = 80 * 1024;
// sorted_units NULL (perm-only mode, sub-runs after a refinement): the runs'
// strings are gathered into the stage from units / offsets, only perm is
// written back and handled entries get length 0 (entries [first, n_medium))
void launch_fix_staged(int coder, const uint2 *list_sm, uint64_t cap_sm, const DevState *st, uint32_t *perm,
                       void *sorted_units, int64_t *sorted_offsets, int num_sms, cudaStream_t s,
                       const void *units = nullptr, const int64_t *offsets = nullptr, uint32_t first = 0);
// sorted_units / sorted_offsets (the main pass with sorted strings): runs of
// <= kTinyMax strings are also written back into the sorted strings (the
// re-gather then skips them); NULL in perm-only mode and after a refinement
void launch_fix_small(int coder, const uint2 *list_sm, const DevState *st, uint32_t *perm,
                      const void *units, const int64_t *offsets, int num_sms, cudaStream_t s, uint32_t first = 0,
                      void *sorted_units = nullptr, int64_t *sorted_offsets = nullptr);
void launch_fix_medium(int coder, const uint2 *list_sm, uint64_t cap_sm, const DevState *st,
                       uint32_t *perm, const void *units, const int64_t *offsets, int num_sms,
                       cudaStream_t s, uint32_t first = 0, const int64_t *staged_so = nullptr);

// A6 giant-run refinement
void launch_seg_prep(int coder, const uint32_t *perm_seg, uint64_t len, const void *units,
                     const int64_t *offsets, uint32_t from, DevState *st, cudaStream_t s);
void launch_seg_key2(int coder, const uint32_t *perm_seg, uint64_t len, const void *units,
                     const int64_t *offsets, uint32_t from, uint64_t *key2, DevState *st,
                     int num_sms, cudaStream_t s);

// A4 gather
// small tiles, many CTAs: the gather is bound by the latency of random reads
#ifndef HUSKY_GATHER_ITEMS
#define HUSKY_GATHER_ITEMS 4
#endif
constexpr int kGatherThreads = 256, kGatherItems = HUSKY_GATHER_ITEMS, kGatherTile = kGatherThreads * kGatherItems;
constexpr int kGatherStage = 24 * 1024;  // one window of output bytes (dynamic smem)
inline uint64_t gather_tiles(uint64_t n) { return (n + kGatherTile - 1) / kGatherTile; }
// base_ptr (nullable): device pointer to the first output offset of a span
// re-gather (positions start there); NULL = 0.
// packed: perm holds index | min(len,15) << 28; strings of length <= PL are
// rebuilt from the sorted codes (packed_codes, or DevState::sorted_keys when
// NULL) and perm is unpacked in place.  st (nullable): violation guard.
void launch_gather(int coder, uint32_t *perm, uint64_t n, const void *units, const int64_t *offsets,
                   void *sorted_units, int64_t *sorted_offsets, unsigned long long *lb,
                   uint32_t *tile_counter, uint32_t epoch, cudaStream_t s, const int64_t *base_ptr = nullptr,
                   bool packed = false, const uint64_t *packed_codes = nullptr, const DevState *st = nullptr,
                   const struct GatherRunsOut *runs_out = nullptr, const uint4 *slab = nullptr);
// A3 fused into the main gather (runs_out != NULL): run starts / ends / dirty
// flags as k_runs_scan writes them, DevState::n_runs; lb: gather_tiles(n) words
struct GatherRunsOut {
  uint32_t *run_start, *run_end;
  uint8_t *dirty;
  unsigned long long *lb;
  DevState *st;
};
// Multi-GPU exchange fused into the gather (NEXT-2): the partitioned order's
// strings go straight into the destination ranks' receive windows (NVLink peer
// memory, or the loopback driver's per-rank regions).  Position j of the
// partitioned order belongs to bucket b with start_n[b] <= j < start_n[b+1]
// (units: start_u); its length goes to lens[b] + 4 j, its global index to
// gidx[b] + 4 j and its units to units[b] + w * (virtual unit offset), every
// base pre-shifted by the bucket start and this rank's displacement in the
// destination (modular uint64 address arithmetic).
constexpr int kMaxPeers = 256;
struct PeerTable {
  uint32_t world, gbase;
  uint64_t start_n[kMaxPeers + 1], start_u[kMaxPeers + 1];
  uint64_t units[kMaxPeers], lens[kMaxPeers], gidx[kMaxPeers];
};
void launch_gather_peer(int coder, const uint32_t *perm, uint64_t n, const void *units, const int64_t *offsets,
                        unsigned long long *lb, uint32_t *tile_counter, uint32_t epoch, const PeerTable *d_table,
                        cudaStream_t s);
void launch_unpack_perm(uint32_t *perm, uint64_t n, cudaStream_t s);
void launch_regather_runs(int coder, const uint2 *list_sm, uint64_t cap_sm, const DevState *st,
                          const uint32_t *perm, const void *units, const int64_t *offsets,
                          void *sorted_units, int64_t *sorted_offsets, int num_sms, cudaStream_t s,
                          uint32_t first_small = 0, uint32_t first_medium = 0, bool skip_staged = false);

// Programmatic dependent launch (PDL): the kernel's CTAs may become resident
// while the previous kernel in the stream drains; the kernel must execute
// `griddepcontrol.wait` (pdl_wait) before touching that kernel's results.
// HUSKY_PDL=0 launches plainly (the wait is then a no-op).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char *v = getenv("HUSKY_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

}  // namespace husky
