#define _POSIX_C_SOURCE 199309L
/* Host-side cost of one libnorm call from C (not product): n = 1024, small path. */
#include <cuda_runtime.h>
#include <stdio.h>
#include <time.h>
#include "libnorm.h"
static double now(void) { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec + 1e-9 * t.tv_nsec; }
int main(void) {
  const int n = 1024;
  float *in, *out;
  cudaMalloc((void**)&in, n * 4); cudaMalloc((void**)&out, n * 4);
  cudaMemset(in, 0, n * 4);
  cudaStream_t st; cudaStreamCreate(&st);
  norm_opts_t o = NORM_OPTS_INIT; o.stream = st;
  for (int i = 0; i < 1000; ++i) norm_launch_ex(out, in, n, &o);
  cudaStreamSynchronize(st);
  const int K = 20000;
  double t0 = now();
  for (int i = 0; i < K; ++i) norm_launch_ex(out, in, n, &o);
  double t1 = now();
  cudaStreamSynchronize(st);
  double t2 = now();
  printf("host enqueue %.2f us/call; enqueue+drain %.2f us/call\n", (t1 - t0) / K * 1e6, (t2 - t0) / K * 1e6);
  o.path = NORM_PATH_TWO_PASS;
  for (int i = 0; i < 100; ++i) norm_launch_ex(out, in, n, &o);
  cudaStreamSynchronize(st);
  t0 = now();
  for (int i = 0; i < K; ++i) norm_launch_ex(out, in, n, &o);
  t1 = now();
  cudaStreamSynchronize(st);
  t2 = now();
  printf("two-pass: host enqueue %.2f us/call; enqueue+drain %.2f us/call\n", (t1 - t0) / K * 1e6, (t2 - t0) / K * 1e6);
  return 0;
}
