/* gen/gen_cuda.cu — device fill for the seeded input generator (gen/norm_gen.h).
 * Not part of the method: bench.py and the GPU tests use it to materialise the
 * synthetic input directly in HBM (n = 2^32 is 16 GiB; copying it from the host
 * would dominate the harness).  Bit-identical to gen_host.c by construction. */
#include <cuda_runtime.h>
#include "norm_gen.h"

__global__ void ng_fill_kernel(float* __restrict__ out, int64_t n, uint64_t seed, int dist,
                               int64_t offset) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = ng_value(seed, dist, (uint64_t)(offset + i));
}

extern "C" int ng_fill_cuda(float* out, int64_t n, uint64_t seed, int dist, int64_t offset,
                            void* stream) {
  if (n < 0 || (n > 0 && !out) || dist < 0 || dist >= NG_DIST_COUNT || offset < 0) return 1;
  if (n == 0) return 0;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  ng_fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(out, n, seed, dist, offset);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
