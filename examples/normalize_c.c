/* examples/normalize_c.c — using libnorm from plain C (no Python, no torch).
 * Build: make examples   Run: ./examples/normalize_c [n]
 * Normalizes a vector with Fig. 1's literal index (norm_launch == the paper's
 * launch() after LICM), then the same vector with the dense index through
 * norm_launch_ex on a stream, and checks both against a host computation. */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "libnorm.h"

#define CHECK_NORM(x)                                                              \
  do {                                                                             \
    norm_status_t st_ = (x);                                                       \
    if (st_ != NORM_OK) {                                                          \
      fprintf(stderr, "%s: %s (%s)\n", #x, norm_status_string(st_), norm_last_error()); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 20) + 7;
  float* h_in = (float*)malloc((size_t)n * 4);
  float* h_out = (float*)malloc((size_t)n * 4);
  double S = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    h_in[i] = (float)((i * 2654435761u) % 1000 + 1) / 1000.0f;
    S += h_in[i];
  }
  float *d_in, *d_out;
  if (cudaMalloc((void**)&d_in, (size_t)n * 4) != cudaSuccess ||
      cudaMalloc((void**)&d_out, (size_t)n * 4) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 1;
  }
  cudaMemcpy(d_in, h_in, (size_t)n * 4, cudaMemcpyHostToDevice);
  cudaMemset(d_out, 0, (size_t)n * 4);

  /* 1. literal index, default stream: out[i] = in[i] / sum for i in C(n) only */
  CHECK_NORM(norm_launch(d_out, d_in, n));
  cudaMemcpy(h_out, d_out, (size_t)n * 4, cudaMemcpyDeviceToHost);
  int64_t count, prefix;
  CHECK_NORM(norm_coverage(n, NORM_INDEX_LITERAL, &count, &prefix));
  double worst = 0.0;
  int64_t written = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (h_out[i] != 0.0f) ++written;
    if (i < prefix) {
      double rel = fabs(h_out[i] - h_in[i] / S) / (h_in[i] / S);
      if (rel > worst) worst = rel;
    }
  }
  printf("literal: |C(n)| = %lld, written = %lld, max rel err = %.3g\n", (long long)count,
         (long long)written, worst);
  if (written != count || worst > 1e-5) return 2;

  /* 2. dense index on a stream, divisor returned on the device */
  cudaStream_t st;
  cudaStreamCreate(&st);
  float* d_s;
  cudaMalloc((void**)&d_s, 4);
  norm_opts_t o = NORM_OPTS_INIT;
  o.stream = st;
  o.index = NORM_INDEX_DENSE;
  o.sum_out = d_s;
  CHECK_NORM(norm_launch_ex(d_out, d_in, n, &o));
  float s;
  cudaMemcpyAsync(&s, d_s, 4, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaMemcpy(h_out, d_out, (size_t)n * 4, cudaMemcpyDeviceToHost);
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += h_out[i];
  printf("dense: s = %.9g (host fp64 sum %.9g), sum of outputs = %.9f\n", s, S, total);
  if (fabs(s - S) > 1e-6 * S || fabs(total - 1.0) > 1e-5) return 3;

  /* 3. errors come back as status codes */
  norm_status_t bad = norm_launch(d_out, d_out + 1, 100);
  printf("partial overlap -> %s\n", norm_status_string(bad));
  if (bad != NORM_ERR_OVERLAP) return 4;
  printf("ok\n");
  return 0;
}
