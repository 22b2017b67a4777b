// gen.cu -- synthetic input generator (NOT part of the method's arithmetic).
//
// Device twin of synthgen.uniform_complex: splitmix64
// finalizer sm(x); stream key s = sm(seed ^ sm(array_id)); value
// sm(s + 2*i + part) >> 11 scaled to [-1, 1).  Tests check it bitwise
// against the numpy implementation.
#include <cstdint>

#include "../../include/idconv.h"
#include "pdl.cuh"

namespace {
__host__ __device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k_fill_uniform(double2* out, size_t n, uint64_t key, uint64_t start) {
  idc::pdl_entry();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint64_t b = key + 2ull * (start + i);
    const double re = (double)(sm64(b) >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    const double im = (double)(sm64(b + 1) >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    out[i] = make_double2(re, im);
  }
}
}  // namespace

extern "C" idc_status idc_fill_uniform(idc_c128* out, size_t n, uint64_t seed, uint64_t array_id, uint64_t start,
                                       idc_stream stream) {
  if (!out || n == 0) return IDC_ERR_INVALID;
  const uint64_t key = sm64(seed ^ sm64(array_id));
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_fill_uniform<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<double2*>(out), n, key, start);
  return cudaGetLastError() == cudaSuccess ? IDC_OK : IDC_ERR_CUDA;
}
