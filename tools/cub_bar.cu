// cub_bar.cu -- the library bar for stage 2 (BENCH INFRASTRUCTURE, not product):
// cub::DeviceRadixSort::SortPairs<uint64_t, uint32_t> on the same husky codes
// the hand-written onesweep sorts (12 B per key and pass: key 8 + payload 4,
// like A2), so bench.py can report the library's time beside ours
// (SURVEY.md 8(d) "same-box library bar for stage 2").
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

extern "C" {

// temp bytes for n pairs
int cub_sortpairs_temp(uint64_t n, size_t *bytes) {
  *bytes = 0;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, *bytes, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                                  (const uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)n, 0, 64);
  return (int)e;
}

// sort (keys_in, vals_in) -> (keys_out, vals_out) on bits [begin_bit, end_bit)
int cub_sortpairs(const uint64_t *keys_in, uint64_t *keys_out, const uint32_t *vals_in, uint32_t *vals_out, uint64_t n,
                  int begin_bit, int end_bit, void *temp, size_t temp_bytes, void *stream) {
  cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, (int64_t)n,
                                                  begin_bit, end_bit, (cudaStream_t)stream);
  return (int)e;
}

}  // extern "C"
