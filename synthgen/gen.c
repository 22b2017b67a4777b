/* synthgen/gen.c -- fast C twin of synthgen.uniform_complex (same counter
 * generator, bitwise identical; see synthgen/__init__.py).  Input generation
 * only: no arithmetic of the convolution method. */
#include <stdint.h>

static inline uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void sg_uniform_complex(double *out, int64_t n, uint64_t seed, uint64_t array_id, uint64_t start) {
  const uint64_t key = sm64(seed ^ sm64(array_id));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t b = key + 2ull * (start + (uint64_t)i);
    out[2 * i] = (double)(sm64(b) >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    out[2 * i + 1] = (double)(sm64(b + 1) >> 11) * 0x1.0p-53 * 2.0 - 1.0;
  }
}
