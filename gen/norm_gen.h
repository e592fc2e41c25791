/*
 * gen/norm_gen.h — seeded, counter-based synthetic input generator.
 *
 * This module is the ONLY code shared by the oracle side (tests, bench's
 * cpu_baseline) and the CUDA side (bench, GPU tests).  It holds none of the
 * method's arithmetic: it only manufactures input vectors.  The paper gives no
 * workload for `normalize` (Fig. 1), so the recipe is ours and
 * is stated in DESIGN.md §"Input recipe".
 *
 * value(seed, dist, i) is a pure function of (seed, dist, global index i), so a
 * shard generates its own slice with `offset` and the host regenerates any
 * element without transfers.  Every distribution is built from integer bit
 * manipulation only (no libm, no rounding), so host and device results are
 * bit-identical by construction (checked on the GPU in tests/test_gpu_parity.py).
 */
#ifndef NORM_GEN_H
#define NORM_GEN_H

#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define NG_FN __host__ __device__ static inline
#else
#define NG_FN static inline
#endif

enum {
  NG_DIST_UNIT = 0,   /* D0: max(1, z>>40) * 2^-24 in (0,1): positive, grid 2^-24   */
  NG_DIST_CONST = 1,  /* D1: 1.0f                                                    */
  NG_DIST_RAMP = 2,   /* D2: 1 + (i mod 8)                                           */
  NG_DIST_SIGNED = 3, /* D3: ((z>>40) - 2^23) * 2^-23 in [-1,1): cancellation        */
  NG_DIST_WIDE = 4,   /* D4: (1 + (z>>41) 2^-23) * 2^((z & 63) - 32): wide exponents */
  NG_DIST_COUNT = 5
};

/* SplitMix64 finaliser applied to a Weyl counter: stateless, counter-based. */
NG_FN uint64_t ng_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

NG_FN uint64_t ng_bits(uint64_t seed, uint64_t i) {
  uint64_t key = ng_mix64(seed + 0x2207002570000000ull);
  return ng_mix64(key + (i + 1) * 0x9E3779B97F4A7C15ull);
}

NG_FN float ng_from_bits(uint32_t u) {
  float f;
#ifdef __CUDA_ARCH__
  f = __uint_as_float(u);
#else
  memcpy(&f, &u, sizeof f);
#endif
  return f;
}

/* Exponent-field construction: 2^e * (1 + m/2^23) for normal e.  Exact. */
NG_FN float ng_make(uint32_t sign, int32_t e, uint32_t mant23) {
  return ng_from_bits((sign << 31) | ((uint32_t)(e + 127) << 23) | (mant23 & 0x7FFFFFu));
}

/* k * 2^-shift for 0 < k < 2^24, exact: normalise k into a 24-bit significand. */
NG_FN float ng_scaled_int(uint32_t sign, uint32_t k, int32_t shift) {
  int32_t top = 31;
  while (!((k >> top) & 1u)) --top; /* k != 0 */
  uint32_t mant = (top >= 23) ? (k >> (top - 23)) : (k << (23 - top));
  return ng_make(sign, top - shift, mant);
}

NG_FN float ng_value(uint64_t seed, int dist, uint64_t i) {
  uint64_t z = ng_bits(seed, i);
  switch (dist) {
    case NG_DIST_CONST:
      return 1.0f;
    case NG_DIST_RAMP:
      return (float)(1u + (uint32_t)(i & 7u));
    case NG_DIST_SIGNED: {
      int32_t k = (int32_t)(z >> 40) - (1 << 23); /* [-2^23, 2^23) */
      if (k == 0) return 0.0f;
      uint32_t sign = k < 0;
      uint32_t a = (uint32_t)(k < 0 ? -k : k);
      return ng_scaled_int(sign, a, 23);
    }
    case NG_DIST_WIDE:
      return ng_make(0u, (int32_t)(z & 63u) - 32, (uint32_t)(z >> 41));
    case NG_DIST_UNIT:
    default: {
      uint32_t k = (uint32_t)(z >> 40);
      if (k == 0) k = 1;
      return ng_scaled_int(0u, k, 24);
    }
  }
}

#endif /* NORM_GEN_H */
