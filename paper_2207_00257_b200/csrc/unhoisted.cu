// unhoisted.cu — Fig. 1 BEFORE parallel LICM, on B200.
//
// The paper's motivating before/after: as printed, every
// thread of normalize<<<(n+31)/32, 32>>> evaluates `sum(in, n)` — O(N^2) work;
// the commented shared-memory variant evaluates it once per
// block — O(N^2/B); LICM hoists it out of the kernel — O(N) (reduce.cu + scale.cu).
// These kernels run the first two forms literally (the printed launch shape,
// the printed index expression) so the hoisted path can be timed against them.
// `sum` is a sequential fp64 loop in index order, identical in every thread, so
// every thread sees the same `val` (reading R3: fp32 accumulation would stagnate).
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "norm_internal.h"

namespace lnorm {

// sum(in, n) as one thread's sequential loop (reading R2/R3).  The
// loads are batched 8 at a time so several are in flight; the additions stay
// in index order.
__device__ __forceinline__ double fig1_sum(const float* __restrict__ in, int64_t n) {
  double val = 0.0;
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(in + i + k);
#pragma unroll
    for (int k = 0; k < 8; ++k) val += (double)v[k];
  }
  for (; i < n; ++i) val += (double)__ldg(in + i);
  return val;
}

__device__ __forceinline__ int64_t fig1_tid(int index) {
  // tid = blockIdx.x + blockDim.x * threadIdx.x (literal); dense reading R1
  return index == NORM_INDEX_LITERAL ? (int64_t)blockIdx.x + (int64_t)blockDim.x * threadIdx.x
                                     : (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
}

// Form 1 (as written): `float val = sum(in, n);` in every thread.
__global__ void __launch_bounds__(32)
    unhoisted_thread_kernel(float* __restrict__ out, const float* __restrict__ in, int64_t n,
                            int index, float* sum_out, double* sum_out_f64) {
  const double S = fig1_sum(in, n);
  const float val = (float)S;
  const int64_t tid = fig1_tid(index);
  if (tid < n) out[tid] = div_rn(in[tid], val);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (sum_out) *sum_out = val;
    if (sum_out_f64) *sum_out_f64 = S;
  }
}

// Form 2: `__shared__ val; if (threadIdx.x == 0) val = sum(in, n);
// __syncthreads();` — once per block.
__global__ void __launch_bounds__(32)
    unhoisted_block_kernel(float* __restrict__ out, const float* __restrict__ in, int64_t n,
                           int index, float* sum_out, double* sum_out_f64) {
  __shared__ double val_sh;
  if (threadIdx.x == 0) val_sh = fig1_sum(in, n);
  __syncthreads();
  const double S = val_sh;
  const float val = (float)S;
  const int64_t tid = fig1_tid(index);
  if (tid < n) out[tid] = div_rn(in[tid], val);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (sum_out) *sum_out = val;
    if (sum_out_f64) *sum_out_f64 = S;
  }
}

cudaError_t launch_unhoisted(float* out, const float* in, int64_t n, int index, int form,
                             float* sum_out, double* sum_out_f64, cudaStream_t st) {
  const int64_t G = (n + 31) / 32;  // normalize<<<(n+31)/32, 32>>>
  if (form == NORM_FORM_PER_THREAD)
    unhoisted_thread_kernel<<<(unsigned)G, 32, 0, st>>>(out, in, n, index, sum_out, sum_out_f64);
  else
    unhoisted_block_kernel<<<(unsigned)G, 32, 0, st>>>(out, in, n, index, sum_out, sum_out_f64);
  return cudaGetLastError();
}

}  // namespace lnorm
