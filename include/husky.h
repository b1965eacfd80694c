/*
 * husky.h -- C ABI of libhusky.so, a B200 (sm_100a) implementation of the
 * data-parallel hot path of Huskysort (Hillyard et al., arXiv 2012.00866):
 *
 *   encode every string into a 64-bit order-preserving "husky code"
 *       (Alg. 2-4; constants PAPER.md:486-494)
 *   -> sort the (code, index) pairs                       (Alg. 1 step 2)
 *   -> resolve every run of equal codes by full string comparison
 *                                                         (Alg. 1 step 3)
 *
 * Conventions (all functions):
 *   - Pointers prefixed d_ are DEVICE pointers (cudaMalloc / torch CUDA tensors),
 *     h_ are HOST pointers.  `stream` is a cudaStream_t passed as void*
 *     (NULL = legacy default stream).  No torch types cross this boundary.
 *   - Strings are given as a unit buffer plus int64 offsets[n+1] (non-decreasing);
 *     string i is units[offsets[i] .. offsets[i+1]).  offsets[0] need not be 0.
 *     Units are uint8 for HUSKY_CODER_ASCII / ENGLISH5 / ENGLISH6 and native
 *     little-endian uint16 (UTF-16 code units, Java String semantics, DESIGN.md
 *     reading R8) for HUSKY_CODER_UNICODE.
 *   - The caller owns every buffer.  Inputs are never written.  The library
 *     never allocates or frees caller memory; scratch memory comes only from
 *     the caller's workspace (size from the *_workspace query).  Plans and
 *     communicators are library-owned until destroyed.
 *   - Every call returns a husky_status; nothing is thrown or aborted across the
 *     ABI.  A human-readable message for the last failure on the calling thread
 *     is available from husky_last_error().
 *   - The sort order is the unique total order: code units compared as unsigned
 *     integers position by position; a proper prefix sorts first; equal strings
 *     are ordered by original index (north_star; reading R7).  This is
 *     exactly what Alg. 1's final "Arrays.sort(xs)" produces with the index as a
 *     tie-break.
 */
#ifndef HUSKY_H
#define HUSKY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HUSKY_OK = 0,
  HUSKY_ERR_INVALID_ARG = 1, /* null required pointer, unknown coder, n >= 2^32,
                                non-monotone offsets, workspace misaligned      */
  HUSKY_ERR_DOMAIN = 2,      /* reserved (no call returns it any more: input outside
                                a coder's domain is sorted by the general cleanup,
                                see husky_sort)                                 */
  HUSKY_ERR_CUDA = 3,        /* a CUDA runtime call failed                       */
  HUSKY_ERR_NCCL = 4,        /* an NCCL call failed (multi-GPU only)             */
  HUSKY_ERR_WORKSPACE = 5,   /* workspace smaller than the query returned        */
  HUSKY_ERR_CAPACITY = 6     /* caller output buffers too small (multi-GPU)      */
} husky_status;

typedef enum {
  HUSKY_CODER_ASCII = 0,   /* asciiToLong: stringToLong(s, 9, 7, 0x7F) */
  HUSKY_CODER_UNICODE = 1, /* unicodeToLong: stringToLong(s, 4, 16, 0xFFFF)>>>1 PAPER.md:463-465, 487-490 */
  HUSKY_CODER_ENGLISH5 = 2,/* "5-bit ASCII ... 12 (or fewer) characters":
                              stringToLong(s, 12, 5, 0x1F), uint8 units (reading R15).
                              Domain: every unit inside the 12-unit code window is a
                              lowercase letter, or every one is uppercase (case
                              folding is monotone only then); off-domain input is
                              sorted by the general cleanup                        */
  HUSKY_CODER_ENGLISH6 = 3 /* "case-dependent strings (6-bit ASCII) ... 10 characters"
                              (PAPER.md:219): stringToLong(s, 10, 6, 0x3F), uint8 units.
                              Domain: units inside the 10-unit window are letters A-Z /
                              a-z (reading R15); else the general cleanup          */
} husky_coder;

/* Mirrors SortOutcome (a reading of Alg. 1's `coding.perfect`, plus
 * run statistics of the step-3 fix-up). */
typedef struct {
  int32_t perfect;          /* Alg. 3 AND_i perfectForLength(len_i);
                               ASCII len<=9, UNICODE len<=3 (reading R4), ENGLISH5 12,
                               ENGLISH6 10 (R15).  Reported only:
                               the fix-up never relies on it.                           */
  int32_t domain_ok;        /* all code-window units in the coder's domain (UNICODE: 1)  */
  uint64_t n_runs;          /* runs of >= 2 equal codes after the key sort               */
  uint64_t n_in_runs;       /* strings inside those runs                                 */
  uint64_t max_run;         /* longest run                                               */
  uint64_t runs_by_class[4];/* [0] already ordered (check only)  [1] warp-sorted (<=32)
                               [2] CTA-sorted (<=4096)           [3] giant (refined)     */
  uint32_t refine_rounds;   /* giant-run refinement rounds (re-key + segment radix)      */
  uint32_t radix_passes;    /* key-sort partition passes: non-trivial 8-bit LSD passes;
                               refinement (A6) passes are added                          */
  uint64_t keys_partitioned;/* keys moved by the main key sort's passes, summed          */
  uint32_t exchange;        /* multi-GPU transport of the strings (husky_exchange)       */
  uint64_t bytes_to_peers;  /* multi-GPU: string bytes + 8 B (length, global index) per
                               string this rank sent to OTHER ranks (NVLink traffic)      */
  uint64_t bytes_from_peers;/* multi-GPU: the same, received from other ranks            */
} husky_outcome;

/* How a sample sort moved the strings between ranks (husky_outcome.exchange). */
typedef enum {
  HUSKY_EXCHANGE_NONE = 0,          /* single-GPU call                                    */
  HUSKY_EXCHANGE_NCCL = 1,          /* send buffers + grouped ncclSend/ncclRecv           */
  HUSKY_EXCHANGE_PEER = 2,          /* the gather stores straight into the destinations'
                                       NCCL symmetric windows over NVLink (NEXT-2)        */
  HUSKY_EXCHANGE_LOOPBACK_COPY = 3, /* loopback driver, device-to-device copies           */
  HUSKY_EXCHANGE_LOOPBACK_PEER = 4  /* loopback driver, the same peer-store gather into
                                       per-virtual-rank windows                           */
} husky_exchange;

/* 1 for ASCII / ENGLISH5 / ENGLISH6 (uint8 units), 2 for UNICODE, 0 for an unknown coder. */
size_t husky_unit_bytes(int coder);

/* A1 -- Alg. 2/3/4 over an array.
 * d_codes[i] = stringToLong(string i) exactly as Alg. 4 computes it, including
 * the per-unit mask (off-domain units are masked, never rejected: SPEC.md:198,
 * reading R5).  If h_perfect is non-NULL the call synchronizes `stream` and
 * stores Alg. 3's perfect flag there: every length <= 9 (ASCII), 3 (UNICODE),
 * 12 (ENGLISH5), 10 (ENGLISH6) (readings R4, R15).
 * Errors: INVALID_ARG (null pointer with n > 0, unknown coder, offsets not
 * non-decreasing -- detected on device, reported only when h_perfect != NULL),
 * CUDA.  n == 0 is a no-op. */
husky_status husky_encode(int coder, const void *d_units, const int64_t *d_offsets, uint64_t n,
                          uint64_t *d_codes, int32_t *h_perfect, void *stream);

/* Workspace bytes husky_sort needs for n strings with `total_units` units
 * (total_units is currently unused but reserved).  Alignment: 256 bytes. */
husky_status husky_sort_workspace(int coder, uint64_t n, uint64_t total_units, size_t *bytes);

/* The whole hot path on one GPU: encode (A1) -> onesweep LSD radix of
 * (code, index) (A2) -> equal-code run detection + order check (A3) ->
 * segmented fix-up of unordered runs (A5) with giant-run refinement (A6) ->
 * gather of the sorted strings (A4).
 *   d_perm[r]          (required, n entries) original index of the r-th string
 *   d_sorted_units     (nullable: perm-only mode) concatenation in sorted order,
 *                      total_units entries of the coder's unit type
 *   d_sorted_offsets   (nullable iff d_sorted_units is) n+1 entries, [0] = 0
 *   d_ws / ws_bytes    workspace of at least husky_sort_workspace() bytes,
 *                      256-byte aligned; contents need not be initialised
 *   h_out              (nullable) outcome statistics
 * Synchronizes `stream` before returning.  n in {0, 1} returns HUSKY_OK at once
 * (d_perm = {0} for n = 1; sorted outputs copied).
 * Input outside the coder's domain (a unit inside a code window that Alg. 4's
 * mask makes non-monotone -- ASCII: > 0x7F; ENGLISH5/6: see husky_coder) is
 * sorted exactly by the general cleanup (NEXT-4: the whole array refined as
 * one segment from unit 0, an MSD string radix over 7-unit windows;
 * h_out->domain_ok = 0 and refine_rounds > 0 report it).
 * Errors: INVALID_ARG, WORKSPACE, CUDA. */
husky_status husky_sort(int coder, const void *d_units, const int64_t *d_offsets, uint64_t n,
                        uint32_t *d_perm, void *d_sorted_units, int64_t *d_sorted_offsets,
                        void *d_ws, size_t ws_bytes, husky_outcome *h_out, void *stream);

/* ------------------------------------------------------------ numeric keys
 * The hot path for objects whose husky code is a PERFECT encoding (PAPER.md:
 * 213-217: "p = 0 ... we can skip step 3"): the code is an order-preserving
 * bijection of the key (SPEC.md:264-275 identity coder; reading R16), so
 * Alg. 1 reduces to encode -> sort (code, index) with no cleanup.
 *   key_type  HUSKY_KEY_U64: uint64 (unsigned order)
 *             HUSKY_KEY_I64: int64 (Java Long.compare order)
 *             HUSKY_KEY_F64: IEEE double in Java Double.compare order: -0.0 <
 *                            +0.0, every NaN equal and above +inf
 *   d_keys         n keys (8 bytes each, read only)
 *   d_perm         (required) stable argsort: original index of the r-th key
 *                  (equal keys by original index)
 *   d_sorted_keys  (nullable) d_keys[d_perm[r]], bit-exact
 * Synchronizes `stream`.  Errors: INVALID_ARG (unknown key_type, null pointer,
 * n >= 2^32 - 1), WORKSPACE, CUDA. */
typedef enum { HUSKY_KEY_U64 = 0, HUSKY_KEY_I64 = 1, HUSKY_KEY_F64 = 2 } husky_key_type;
husky_status husky_sort_keys_workspace(int key_type, uint64_t n, size_t *bytes);
husky_status husky_sort_keys(int key_type, const void *d_keys, uint64_t n, uint32_t *d_perm,
                             void *d_sorted_keys, void *d_ws, size_t ws_bytes, void *stream);

/* husky_sort on HOST buffers: copies units/offsets host->device, sorts, and
 * copies perm (and, if h_sorted_units != NULL, the sorted units and offsets)
 * device->host, all on `stream`.  Host buffers should be pinned for speed.
 * `d_ws` must hold husky_sort_host_workspace() bytes (it also stages the device
 * copies of the inputs and outputs). */
husky_status husky_sort_host_workspace(int coder, uint64_t n, uint64_t total_units, size_t *bytes);
husky_status husky_sort_host(int coder, const void *h_units, const int64_t *h_offsets, uint64_t n,
                             uint32_t *h_perm, void *h_sorted_units, int64_t *h_sorted_offsets,
                             void *d_ws, size_t ws_bytes, husky_outcome *h_out, void *stream);

/* Many independent sorts on HOST buffers, pipelined: `depth` input slots
 * (device inputs + sort workspace) and depth + 1 output slots (device outputs)
 * used round robin, and three streams -- host->device copies, kernels,
 * device->host copies -- so batch b+1's input copy, batch b's kernels and batch
 * b-1's output copy overlap (PCIe is full duplex; the copy engines are
 * independent of the SMs); events order the reuse of a slot.  Batch b:
 * h_units[b], h_offsets[b] (n[b] + 1 entries), outputs h_perm[b] and, if
 * non-NULL, h_sorted_units[b] / h_sorted_offsets[b] (pass NULL arrays for
 * perm-only).  Output copies complete in batch order, so batches may share
 * output buffers only if the caller reads them after the call.  Host buffers
 * must be pinned for the copies to overlap.  d_ws must hold
 * husky_sort_host_many_workspace(coder, n_max, units_max, depth) bytes, where
 * n_max / units_max bound every batch.  h_out (nullable) receives k outcomes.
 * Returns after every batch has finished; the first failing batch's status. */
husky_status husky_sort_host_many_workspace(int coder, uint64_t n_max, uint64_t units_max, int depth,
                                            size_t *bytes);
husky_status husky_sort_host_many(int coder, int k, const void *const *h_units, const int64_t *const *h_offsets,
                                  const uint64_t *n, uint32_t *const *h_perm, void *const *h_sorted_units,
                                  int64_t *const *h_sorted_offsets, int depth, void *d_ws, size_t ws_bytes,
                                  husky_outcome *h_out);

/* ------------------------------------------------------------------ multi-GPU
 * Sample sort over P ranks (one process per GPU).  Input is block-distributed
 * by global index: rank r holds strings [global_base_r, global_base_r + n_local)
 * (reading R12).  Splitters are sampled string prefixes compared in the sort
 * order (code first, units on a code tie), so equal strings never straddle
 * ranks and all-colliding codes still spread; after one all-to-all each rank
 * sorts its bucket with the single-GPU path.  Rank r's output is its shard of the global order; the global result is
 * the concatenation of the shards in rank order.  perm entries are GLOBAL indices.
 */

/* 128-byte NCCL unique id (rank 0 creates it; broadcast it with any transport). */
husky_status husky_comm_unique_id(uint8_t id[128]);
/* Creates the NCCL communicator on the current CUDA device. */
husky_status husky_comm_create(int rank, int world, const uint8_t id[128], void **comm);
/* The world size `comm` was created with (for husky_sort_multi_workspace). */
husky_status husky_comm_world(void *comm, int *world);
husky_status husky_comm_destroy(void *comm);

/* Phase 1: encode, sample splitters (all-gather), count, exchange counts.
 * Reports the sizes of this rank's output shard so the caller can allocate it.
 * d_ws must hold husky_sort_multi_workspace(n_local, local_units) bytes.
 * Synchronizes `stream`.  The plan keeps pointers to the inputs and d_ws. */
husky_status husky_sort_multi_workspace(int coder, uint64_t n_local, uint64_t local_units,
                                        int world, size_t *bytes);
husky_status husky_sort_multi_plan(void *comm, int coder, const void *d_units,
                                   const int64_t *d_offsets, uint64_t n_local, uint64_t global_base,
                                   void *d_ws, size_t ws_bytes, void **plan, uint64_t *h_n_out,
                                   uint64_t *h_units_out, void *stream);
/* Phase 2: exchange strings and sort the received bucket.  Transport: the
 * partitioning gather stores every string straight into its destination
 * rank's receive window -- an NCCL symmetric window (ncclMemAlloc +
 * ncclCommWindowRegister, owned by the communicator, grown collectively by
 * the plan call) written through NVLink peer addresses -- followed by a 4-byte
 * all-reduce barrier; with HUSKY_EXCHANGE=nccl in the environment (or if the
 * window cannot be registered on every rank) send buffers + grouped
 * ncclSend/ncclRecv.  h_out->exchange says which ran.  The receive window
 * is reused across calls: the plan of a call must not start on one rank while
 * another rank's exec of the previous call runs (exec synchronizes its stream
 * before returning, so sequential calls per rank satisfy this).  d_perm_out: h_n_out entries (global indices); d_sorted_units_out:
 * h_units_out units (nullable -> perm-only); d_sorted_offsets_out: h_n_out+1
 * (nullable iff d_sorted_units_out is), local offsets starting at 0.
 * d_recv_ws must hold husky_sort_multi_recv_workspace(plan) bytes. */
husky_status husky_sort_multi_recv_workspace(void *plan, size_t *bytes);
husky_status husky_sort_multi_exec(void *plan, uint32_t *d_perm_out, void *d_sorted_units_out,
                                   int64_t *d_sorted_offsets_out, void *d_recv_ws,
                                   size_t recv_ws_bytes, husky_outcome *h_out, void *stream);
husky_status husky_plan_destroy(void *plan);

/* Convenience: plan + exec with caller capacities.  If cap_n < h_n_out or
 * cap_units < h_units_out it returns HUSKY_ERR_CAPACITY with the required sizes
 * in *h_n_out / *h_units_out and does nothing else. */
husky_status husky_sort_multi(void *comm, int coder, const void *d_units, const int64_t *d_offsets,
                              uint64_t n_local, uint64_t global_base, uint32_t *d_perm_out,
                              void *d_sorted_units_out, int64_t *d_sorted_offsets_out,
                              uint64_t cap_n, uint64_t cap_units, uint64_t *h_n_out,
                              uint64_t *h_units_out, void *d_ws, size_t ws_bytes,
                              husky_outcome *h_out, void *stream);

/* Loopback driver of the sample sort on ONE GPU: sorts n strings as if they were
 * block-distributed over `world` virtual ranks, running the same phases
 * (encode, sampling, splitters, bucketing, stable partition, exchange, local
 * sort) with device-to-device copies as the transport.  Outputs are the
 * rank-order concatenation: global perm (n), sorted units, global sorted offsets
 * (n+1, nullable together with d_sorted_units).  h_shard_n (nullable) receives
 * `world` shard sizes.  Synchronizes `stream`.  Used to test the sharded path
 * where only one GPU is available. */
husky_status husky_sort_multi_loopback_workspace(int coder, int world, uint64_t n, uint64_t total_units,
                                                 size_t *bytes);
husky_status husky_sort_multi_loopback(int coder, int world, const void *d_units, const int64_t *d_offsets,
                                       uint64_t n, uint32_t *d_perm, void *d_sorted_units,
                                       int64_t *d_sorted_offsets, void *d_ws, size_t ws_bytes,
                                       uint64_t *h_shard_n, husky_outcome *h_out, void *stream);

/* The sample sort's splitter rule, on the host, exposed for testing (no GPU
 * needed; multi-GPU ranks apply the same rule on the GPU).  Input: the m
 * gathered sample strings (each rank's prefixes of at most 32 units, rank-major)
 * as units + offsets[m+1].  Output: h_idx[k-1] (k = 1..P-1) = index of the
 * sample at position floor(k*m/P) of the samples sorted in the sort order
 * (ties by index).  Splitter k is that sample's string; bucket(x) = number of
 * splitters <= x in the sort order (composite splitters, SURVEY.md 8(f)
 * NEXT-1): equal-code runs may straddle ranks, equal strings never do. */
husky_status husky_select_splitters(int coder, const void *h_units, const int64_t *h_offsets, uint64_t m,
                                    int world, uint64_t *h_idx);

/* --------------------------------------------------------------- profiling
 * Per-stage accounting (the T1/T2/T3 split of PAPER.md:238-245, per kernel
 * family).  Every kernel launch is counted; with profiling enabled each launch
 * is also bracketed by a CUDA event pair on its own stream (mode 1), or only
 * the encoder, histogram, radix-pass and main-gather groups are (mode 2: four
 * event pairs per sort, cheap enough inside a timed region).  Stage ids:
 * 0 encode, 1 hist_scan, 2 radix_pass, 3 runs_scan, 4 runs_classify,
 * 5 fix_small, 6 fix_medium, 7 refine, 8 gather, 9 multi.
 * husky_profile_read fills up to max_stages entries (ms = summed device time,
 * launches, elems = summed elements processed) and returns the stage count. */
void husky_profile_enable(int on);
void husky_profile_reset(void);
/* Profiling mode 1 (an event pair per launch) also logs every launch in order:
 * copies up to max_records (stage id, elements, device ms) and returns how
 * many are logged (at most 65536 since the last reset). */
int husky_profile_launches(int *stages, uint64_t *elems, double *ms, int max_records);
int husky_profile_read(double *ms, uint64_t *launches, uint64_t *elems, int max_stages);
const char *husky_profile_stage_name(int stage);
uint64_t husky_launch_count(void);

/* Thread-local message describing the last non-OK status ("" if none). */
const char *husky_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HUSKY_H */
