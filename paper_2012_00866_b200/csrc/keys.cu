// keys.cu -- the hot path for numeric keys, whose husky code is a PERFECT
// encoding: "for some domains of X, we can definitely assert that p = 0 ... In
// such a case, we can skip step 3 of the algorithm".  The
// code is an order-preserving bijection of the key (SPEC.md:264-275's identity
// coder; reading R16), so Alg. 1 is encode -> sort (code, index), and
// the stable radix leaves equal keys in index order.
//   u64: code = x
//   i64: code = x ^ 2^63                      (Long.compare order)
//   f64: every NaN -> the canonical NaN (doubleToLongBits), then
//        code = bits ^ (sign ? ~0 : 2^63)     (Double.compare order: -0.0 < +0.0,
//                                              NaN above +inf)
// The LSD onesweep passes, their device-side plan and the histogram kernel are
// the string path's (radix.cu, encode.cu).
#include <algorithm>

#include "host_common.h"

namespace husky {

__global__ void k_key_encode(int type, const uint64_t *__restrict__ keys, uint64_t n, uint64_t *__restrict__ codes) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = __ldg(keys + i);
    if (type == HUSKY_KEY_I64) {
      x ^= 1ull << 63;
    } else if (type == HUSKY_KEY_F64) {
      if ((x & 0x7FF0000000000000ull) == 0x7FF0000000000000ull && (x & 0x000FFFFFFFFFFFFFull))
        x = 0x7FF8000000000000ull;  // canonical NaN
      x ^= (x >> 63) ? ~0ull : (1ull << 63);
    }
    codes[i] = x;
  }
}

__global__ void k_gather_keys(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ perm, uint64_t n,
                              uint64_t *__restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = __ldg(keys + __ldg(perm + i));
}

static unsigned grid_n(uint64_t n, int sms) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 8));
}

}  // namespace husky

using namespace husky;

extern "C" {

husky_status husky_sort_keys_workspace(int key_type, uint64_t n, size_t *bytes) {
  if (key_type < HUSKY_KEY_U64 || key_type > HUSKY_KEY_F64) return fail(HUSKY_ERR_INVALID_ARG, "unknown key type %d", key_type);
  if (!bytes) return fail(HUSKY_ERR_INVALID_ARG, "bytes is NULL");
  *bytes = make_layout(n).total;
  return HUSKY_OK;
}

husky_status husky_sort_keys(int key_type, const void *d_keys, uint64_t n, uint32_t *d_perm, void *d_sorted_keys,
                             void *d_ws, size_t ws_bytes, void *stream) {
  if (key_type < HUSKY_KEY_U64 || key_type > HUSKY_KEY_F64) return fail(HUSKY_ERR_INVALID_ARG, "unknown key type %d", key_type);
  if (n >= 0xFFFFFFFFull) return fail(HUSKY_ERR_INVALID_ARG, "n = %llu >= 2^32 - 1", (unsigned long long)n);
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) return HUSKY_OK;
  if (!d_keys || !d_perm || !d_ws) return fail(HUSKY_ERR_INVALID_ARG, "null required pointer");
  if ((uintptr_t)d_ws % 256) return fail(HUSKY_ERR_INVALID_ARG, "workspace not 256-byte aligned");
  Layout L = make_layout(n);
  if (ws_bytes < L.total) return fail(HUSKY_ERR_WORKSPACE, "workspace %zu < required %zu", ws_bytes, L.total);
  Sorter S;
  S.coder = HUSKY_CODER_ASCII;  // unused by the radix
  S.units = nullptr;
  S.offsets = nullptr;
  S.n = n;
  S.perm = d_perm;
  S.ws = (uint8_t *)d_ws;
  S.L = L;
  S.s = s;
  S.sms = device_sm_count();
  S.st = S.at<DevState>(L.state);
  DevState *st = S.st;
  cudaError_t e = cudaMemsetAsync(st, 0, sizeof(DevState), s);
  if (e == cudaSuccess) e = S.reset_lookback();
  if (e != cudaSuccess) return fail(HUSKY_ERR_CUDA, "husky_sort_keys: %s", cudaGetErrorString(e));
  uint64_t *keysA = S.keysA(), *keysB = S.keysB();
  {
    HUSKY_SCOPE(ST_ENCODE, s, n);
    k_key_encode<<<grid_n(n, S.sms), 256, 0, s>>>(key_type, (const uint64_t *)d_keys, n, keysA);
  }
  launch_hist_plan(keysA, n, st, keysA, keysB, S.sms, s);
  for (int slot = 0; slot < 8; ++slot)
    launch_onesweep_slot(slot, keysA, keysB, nullptr, d_perm, S.at<uint32_t>(L.vals), n, st, S.lb_radix(),
                         S.next_counter(), S.next_epoch(), s);
  launch_radix_finalize(st, nullptr, d_perm, n, s);
  if (d_sorted_keys) {
    HUSKY_SCOPE(ST_GATHER, s, n);
    k_gather_keys<<<grid_n(n, S.sms), 256, 0, s>>>((const uint64_t *)d_keys, d_perm, n, (uint64_t *)d_sorted_keys);
  }
  e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HUSKY_ERR_CUDA, "husky_sort_keys: %s", cudaGetErrorString(e));
  return HUSKY_OK;
}

}  // extern "C"
