// host_common.h -- host-side helpers shared by husky.cu and multi.cu.
#pragma once
#include <cstdarg>
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include <utility>

#include "../../include/husky.h"
#include "kernels.cuh"

namespace husky {

// Workspace layout of husky_sort for n strings (byte offsets, 256-aligned).
struct Layout {
  uint64_t n = 0, tiles_r = 0, tiles_s = 0, cap_sm = 0, cap_g = 0;
  size_t state = 0, keysA = 0, keysB = 0, vals = 0, vals2 = 0, slab = 0, lb_radix = 0, lb_scan = 0, run_start = 0,
         run_end = 0, dirty = 0, list_sm = 0, list_g = 0, total = 0;
  uint64_t lb_radix_words = 0;
};
Layout make_layout(uint64_t n);

husky_status fail(husky_status st, const char *fmt, ...);
husky_status checked_result(husky_status st, const char *what);  // husky.cu

inline bool valid_coder(int c) { return c >= HUSKY_CODER_ASCII && c <= HUSKY_CODER_ENGLISH6; }
inline size_t coder_unit_bytes(int c) { return c == HUSKY_CODER_UNICODE ? 2 : (valid_coder(c) ? 1 : 0); }
// Kernels other than the encoder are instantiated for the unit type only: the
// byte coders (ASCII, ENGLISH5/6) share the ASCII instantiation.
inline int kernel_coder(int c) { return c == HUSKY_CODER_UNICODE ? HUSKY_CODER_UNICODE : HUSKY_CODER_ASCII; }
// Input outside the coder's domain inside a code window (readings R5, R15):
// the equal-run fix-up is exact only on the domain.
inline bool domain_violation(int c, uint32_t viol) {
  if (c == HUSKY_CODER_ASCII || c == HUSKY_CODER_ENGLISH6) return (viol & kDomainBad) != 0;
  if (c == HUSKY_CODER_ENGLISH5) return (viol & kNotLower) && (viol & kNotUpper);
  return false;
}
int device_sm_count();

// The single-GPU path (husky_sort) -- also the local phase of the sample sort.
// allow_graph: replay a cached CUDA graph of the launch sequence when the
// same call repeats (husky.cu); the sample sort's local sorts pass false
// (fresh receive buffers every call would only fill the cache).
husky_status sort_impl(int coder, const void *d_units, const int64_t *d_offsets, uint64_t n,
                       uint32_t *d_perm, void *d_sorted_units, int64_t *d_sorted_offsets, void *d_ws,
                       size_t ws_bytes, husky_outcome *h_out, cudaStream_t s, bool allow_graph = true);

// --------------------------------------------------------------- Sorter
// One husky_sort invocation: owns the epoch / tile-counter bookkeeping.
struct Sorter {
  int coder;
  const void *units;
  const int64_t *offsets;
  uint64_t n;
  uint32_t *perm;
  uint8_t *ws;
  Layout L;
  cudaStream_t s;
  int sms;
  DevState *st;
  uint32_t epoch = 0;
  uint32_t slot = 0;
  uint32_t radix_passes = 0, refine_rounds = 0;
  cudaError_t err = cudaSuccess;  // first failure of the bookkeeping resets (checked at the sync points)

  template <typename T> T *at(size_t o) const { return reinterpret_cast<T *>(ws + o); }
  uint64_t *keysA() const { return at<uint64_t>(L.keysA); }
  uint64_t *keysB() const { return at<uint64_t>(L.keysB); }
  unsigned long long *lb_radix() const { return at<unsigned long long>(L.lb_radix); }
  unsigned long long *lb_scan() const { return at<unsigned long long>(L.lb_scan); }
  // second scan-look-back array (the run-count scan fused into the gather)
  unsigned long long *lb_scan2() const { return at<unsigned long long>(L.lb_scan) + L.tiles_s; }

  cudaError_t reset_lookback() {
    cudaError_t e = cudaMemsetAsync(ws + L.lb_radix, 0, L.lb_radix_words * 8, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(ws + L.lb_scan, 0, L.tiles_s * 16, s);
    return e;
  }
  // next look-back epoch (1..255); wraps by clearing the flag arrays
  uint32_t next_epoch() {
    if (++epoch > 255) {
      cudaError_t e = reset_lookback();
      if (err == cudaSuccess) err = e;
      epoch = 1;
    }
    return epoch;
  }
  uint32_t *next_counter() {
    if (slot == 64) {
      cudaError_t e = cudaMemsetAsync(st->tile_counter, 0, sizeof(st->tile_counter), s);
      if (err == cudaSuccess) err = e;
      slot = 0;
    }
    return st->tile_counter + slot++;
  }

  // Stable LSD radix of (keys_in, vals_in) over m elements, skipping digits in
  // `trivial`.  vals_in == NULL synthesises payload = index.  The final payload
  // lands in `vals_final`, the final keys pointer is returned via *keys_sorted.
  // keys_in must be keysA() or keysB(); vals_tmp must not alias vals_final.
  husky_status radix(uint64_t *keys_in, const uint32_t *vals_in, uint64_t m, uint32_t trivial,
                     uint32_t *vals_final, uint32_t *vals_tmp, uint64_t **keys_sorted) {
    int digits[8], np = 0;
    for (int d = 0; d < 8; ++d)
      if (!(trivial & (1u << d))) digits[np++] = d;
    radix_passes += np;
    uint64_t *kin = keys_in, *kout = keys_in == keysA() ? keysB() : keysA();
    if (np == 0) {
      if (vals_in == nullptr) launch_iota(vals_final, m, s);
      else if (vals_in != vals_final)
        cudaMemcpyAsync(vals_final, vals_in, m * 4, cudaMemcpyDeviceToDevice, s);
      *keys_sorted = keys_in;
      return HUSKY_OK;
    }
    const uint32_t *vin = vals_in;
    for (int p = 0; p < np; ++p) {
      // choose the output so that the last pass writes vals_final (and never
      // writes the buffer it reads)
      bool last_is_final = ((np - 1 - p) % 2) == 0;
      uint32_t *vout = last_is_final ? vals_final : vals_tmp;
      if (vout == vin) vout = (vout == vals_final) ? vals_tmp : vals_final;
      launch_onesweep(kin, vin, kout, vout, m, digits[p], st, lb_radix(), next_counter(), next_epoch(), s);
      vin = vout;
      std::swap(kin, kout);
    }
    if (vin != vals_final) cudaMemcpyAsync(vals_final, vin, m * 4, cudaMemcpyDeviceToDevice, s);
    *keys_sorted = kin;
    return HUSKY_OK;
  }
};

}  // namespace husky
