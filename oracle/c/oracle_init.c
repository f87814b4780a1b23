/* CPU ORACLE HELPER — TEST INFRASTRUCTURE ONLY (see oracle/model.py header).
 *
 * C restatement of oracle.model.init_values (the deterministic weight init
 * both the executor's init_kernel and the numpy oracle use): element i of a
 * tensor keyed `key` is
 *   z0 = splitmix64(key + (2i) * C), z1 = splitmix64(key + (2i+1) * C),
 *   s  = (z0>>40) + ((z0>>8)&0xFFFFFF) + (z1>>40) + ((z1>>8)&0xFFFFFF) - 2^25,
 *   v  = (float)((double)s * c)
 * (Irwin-Hall(4) normal approximation).  Same integer arithmetic and one
 * correctly rounded double multiply, so it is bit-identical to the numpy
 * path (checked by tests/test_oracle.py) — it only makes the large-width
 * parity tests' oracle init fast.  Built by oracle/Makefile into
 * oracle/_build/liboracle_init.so. */
#include <stdint.h>

static inline uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void oracle_init_values(uint64_t key, int64_t n, int64_t start, double c, float* out) {
  const uint64_t C = 0xD1B54A32D192ED03ull;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    const uint64_t i = (uint64_t)(start + j);
    const uint64_t z0 = splitmix(key + (2 * i) * C);
    const uint64_t z1 = splitmix(key + (2 * i + 1) * C);
    const int64_t s = (int64_t)(z0 >> 40) + (int64_t)((z0 >> 8) & 0xFFFFFF) + (int64_t)(z1 >> 40) +
                      (int64_t)((z1 >> 8) & 0xFFFFFF) - (1ll << 25);
    out[j] = (float)((double)s * c);
  }
}

/* Round-to-nearest-even to bfloat16 (returned widened to fp32), NaN kept:
 * oracle.model.bf16_round. */
void oracle_bf16_round(const float* x, float* y, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    union { float f; uint32_t u; } a, b;
    a.f = x[j];
    if (a.f != a.f) {
      y[j] = a.f;
      continue;
    }
    const uint64_t u = a.u;
    b.u = (uint32_t)(((u + 0x7FFFull + ((u >> 16) & 1ull)) >> 16) << 16);
    y[j] = b.f;
  }
}
