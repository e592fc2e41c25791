// scripts/verify_division.cu — exhaustive check that libnorm's uniform-divisor
// division (device_common.cuh: make_divisor + div_rn) is bit-identical to
// __fdiv_rn for ALL 2^32 dividend bit patterns, for a set of divisors:
// specials (powers of two, all-ones / minimal mantissas, window edges,
// subnormals, FLT_MAX, inf, NaN, zeros) plus pseudo-random bit patterns.
// Usage: verify_division [n_random=1000] [seed=2207]; exit 0 iff no mismatch.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "device_common.cuh"

using namespace lnorm;

// Every dividend is checked through BOTH entry points: div8 (vector of 8
// consecutive bit patterns: the kernels' hot path, incl. its out-of-line
// fallback) and the scalar div_rn.
__global__ void check_kernel(float s, unsigned long long* mism, unsigned* first_a) {
  const Divisor d = make_divisor(s);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  unsigned long long local = 0;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < (1ull << 29); g += stride) {
    f8 a;
#pragma unroll
    for (int k = 0; k < 8; ++k) a.v[k] = __uint_as_float((unsigned)(g * 8 + k));
    const f8 q = div8(a, d);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float y = __fdiv_rn(a.v[k], s);
      const float x1 = q.v[k], x2 = div_rn(a.v[k], d), x3 = div_rn_fchk(a.v[k], d);
      const bool ok1 = __float_as_uint(x1) == __float_as_uint(y) || ((x1 != x1) && (y != y));
      const bool ok2 = __float_as_uint(x2) == __float_as_uint(y) || ((x2 != x2) && (y != y));
      const bool ok3 = __float_as_uint(x3) == __float_as_uint(y) || ((x3 != x3) && (y != y));
      if (!(ok1 && ok2 && ok3)) {
        if (local == 0) atomicCAS(first_a, 0xFFFFFFFFu, (unsigned)(g * 8 + k));
        ++local;
      }
    }
  }
  if (local) atomicAdd(mism, local);
}

static uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  const int nrand = argc > 1 ? atoi(argv[1]) : 1000;
  const uint64_t seed = argc > 2 ? strtoull(argv[2], 0, 10) : 2207;
  unsigned specials[] = {
      0x3f800000u, 0x40000000u, 0x40400000u, 0x40e00000u, 0x3fffffffu, 0x3f800001u, 0x3fffffffu,
      0x7f7fffffu, 0x00800000u, 0x00000001u, 0x007fffffu, 0x7f800000u, 0x7fc00000u, 0x00000000u,
      0x80000000u, 0xbf800000u, 0xc0400000u, 0x3b800000u /* 2^-8 */, 0x05800000u /* ~2^-116 */,
      0x7b800000u /* 2^120 */, 0x7b7fffffu, 0x03800000u /* 2^-120 */, 0x037fffffu,
      0x4f800000u /* 2^32 */, 0x4f800001u, 0x4effffffu, 0x49000001u, 0x3eaaaaabu /* 1/3 */};
  const int nspec = sizeof(specials) / sizeof(specials[0]);
  unsigned long long* mism;
  unsigned* first_a;
  cudaMalloc(&mism, 8);
  cudaMalloc(&first_a, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long total_bad = 0;
  int bad_divisors = 0;
  for (int k = 0; k < nspec + nrand; ++k) {
    unsigned sb = k < nspec ? specials[k] : (unsigned)mix(seed * 1000003ull + k);
    float s;
    memcpy(&s, &sb, 4);
    cudaMemset(mism, 0, 8);
    cudaMemset(first_a, 0xFF, 4);
    check_kernel<<<sms * 8, 256>>>(s, mism, first_a);
    unsigned long long m;
    unsigned fa;
    cudaMemcpy(&m, mism, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&fa, first_a, 4, cudaMemcpyDeviceToHost);
    if (cudaGetLastError() != cudaSuccess) { printf("cuda error\n"); return 2; }
    if (m) {
      ++bad_divisors;
      total_bad += m;
      printf("MISMATCH s=0x%08x (%g): %llu dividends, first a=0x%08x\n", sb, s, m, fa);
    }
  }
  printf("divisors checked: %d (%d special + %d random), dividends per divisor: 2^32, "
         "mismatching divisors: %d, mismatches: %llu\n",
         nspec + nrand, nspec, nrand, bad_divisors, total_bad);
  return total_bad ? 1 : 0;
}
