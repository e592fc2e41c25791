// scripts/microbench_oneshot.cu — design-space probe (not product code), round 2:
// does the one-tile-per-CTA (non-persistent grid) scheme that made the scale
// faster (scripts/microbench_scale2.cu) also help
//  (a) the read-only reduce: each CTA sums one contiguous tile (256-bit loads,
//      fp32 8-element pre-sum -> fp64, block tree) into partial[blockIdx.x]; a
//      second one-CTA kernel adds the partials in index order.  Compared with
//      the TMA-ring reduce at the same n (libnorm: 7.49 TB/s at 2^32);
//  (b) the dense rows config (65536 x 4096): one CTA per row, the row in
//      registers (block sum, divide, store), vs rows_vec_kernel (persistent,
//      row queue: 6.88-6.92 TB/s).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_2207_00257_b200/csrc scripts/microbench_oneshot.cu -o scripts/mb_oneshot
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "device_common.cuh"

using namespace lnorm;

// lnorm::sum8: the product's fp32 8-element pairwise pre-sum
template <int T, int U>
__global__ void __launch_bounds__(T) tile_sum(const float* in, double* partial) {
  __shared__ double red[T / 32];
  const int64_t base = (int64_t)blockIdx.x * T * U * 8;
  f8 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = ld8_stream(in + base + ((int64_t)u * T + threadIdx.x) * 8);
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) acc += sum8(v[u]);
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = b;
}

// one CTA: fixed-order sum of the partials
__global__ void __launch_bounds__(1024) combine(const double* partial, int64_t np, double* S) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < np; i += 1024) acc += partial[i];
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) *S = b;
}

// dense rows, one CTA per row of C = T * U * 8 floats, the row in registers
template <int T, int U>
__global__ void __launch_bounds__(T) rows_oneshot(float* out, const float* in) {
  __shared__ double red[T / 32];
  const int64_t base = (int64_t)blockIdx.x * T * U * 8;
  f8 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = ld8_stream(in + base + ((int64_t)u * T + threadIdx.x) * 8);
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) acc += sum8(v[u]);
  const double S = block_sum(acc, red);
  const Divisor dv = make_divisor((float)S);
#pragma unroll
  for (int u = 0; u < U; ++u) st8_stream(out + base + ((int64_t)u * T + threadIdx.x) * 8, div8(v[u], dv));
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  f();
  float best = 1e30f;
  for (int i = 0; i < 8; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  const int e = argc > 1 ? atoi(argv[1]) : 32;
  const int64_t n = 1ll << e;
  float *in, *out;
  double *partial, *S;
  if (cudaMalloc(&in, n * 4) != cudaSuccess || cudaMalloc(&out, (1ll << 28) * 4) != cudaSuccess ||
      cudaMalloc(&partial, (n / 2048 + 1) * 8) != cudaSuccess || cudaMalloc(&S, 8) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(in, 0x3F, n * 4);
  printf("(a) read-only tile reduce, n = 2^%d fp32, best of 8 (GB/s = 4n / time, incl. the combine kernel)\n", e);
#define TS(NAME, T, U)                                                                              \
  {                                                                                                 \
    const int64_t nb = n / ((int64_t)T * U * 8);                                                    \
    float ms = timeit([&] {                                                                         \
      tile_sum<T, U><<<(unsigned)nb, T>>>(in, partial);                                              \
      combine<<<1, 1024>>>(partial, nb, S);                                                         \
    });                                                                                             \
    printf("%-40s %8.3f ms %8.1f GB/s %s\n", NAME, ms, 4.0 * n / ms / 1e6, cudaGetErrorString(cudaGetLastError())); \
  }
  TS("tile sum T256 U1", 256, 1);
  TS("tile sum T256 U2", 256, 2);
  TS("tile sum T256 U4", 256, 4);
  TS("tile sum T512 U2", 512, 2);
  TS("tile sum T128 U4", 128, 4);
  TS("tile sum T512 U4", 512, 4);
  TS("tile sum T1024 U2", 1024, 2);
  const int64_t R = 65536;
  printf("(b) dense rows 65536 x 4096 one CTA per row, best of 8 (GB/s = 8 R C / time)\n");
#define RO(NAME, T, U)                                                                                 \
  {                                                                                                    \
    float ms = timeit([&] { rows_oneshot<T, U><<<(unsigned)R, T>>>(out, in); });                       \
    printf("%-40s %8.3f ms %8.1f GB/s %s\n", NAME, ms, 8.0 * R * 4096 / ms / 1e6,                      \
           cudaGetErrorString(cudaGetLastError()));                                                    \
  }
  RO("rows one-shot T512 U1", 512, 1);
  RO("rows one-shot T256 U2", 256, 2);
  RO("rows one-shot T128 U4", 128, 4);
  return 0;
}
