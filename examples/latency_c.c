/* examples/latency_c.c — per-call latency of libnorm from plain C (no Python):
 * BASELINE configs 1-2 (n = 1024 with its 32 x 32 literal grid, n = 2^20 + 7)
 * are launch-bound, so what a C caller pays per call is the figure of merit.
 * For each path: the host time of one enqueue (norm_launch_ex returning; in
 * batches of 64 calls, so the launch queue never fills and the enqueue never
 * waits for the device), with libnorm's pointer checks and under
 * NORM_FLAG_TRUSTED_PTRS, and the back-to-back time per call (K calls enqueued,
 * then one stream synchronize: device- or host-bound, whichever is slower),
 * plus the same through a norm_graph_t replay.  Prints one JSON object per line.
 * Build: make examples   Run: ./examples/latency_c [n ...] */
#define _POSIX_C_SOURCE 199309L
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include "libnorm.h"

static double now(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + 1e-9 * t.tv_nsec;
}

static const char* kPath[] = {"auto", "two_pass", "fused", "small", "mid", "cluster"};

static int run(int64_t n, int path, unsigned flags, float* out, const float* in, cudaStream_t st,
               double* enq_us, double* b2b_us) {
  norm_opts_t o = NORM_OPTS_INIT;
  o.stream = st;
  o.path = path;
  o.flags = flags;
  for (int i = 0; i < 500; ++i)
    if (norm_launch_ex(out, in, n, &o) != NORM_OK) return 1;
  cudaStreamSynchronize(st);
  /* host cost: batches of 64 calls (far below the launch queue's depth, so the
   * enqueue never waits for the device), stream drained between batches */
  const int B = 64, NB = 200;
  double host = 0.0;
  for (int b = 0; b < NB; ++b) {
    double t0 = now();
    for (int i = 0; i < B; ++i) norm_launch_ex(out, in, n, &o);
    host += now() - t0;
    cudaStreamSynchronize(st);
  }
  *enq_us = host / (B * NB) * 1e6;
  /* back to back: K calls enqueued, then one drain (device- or host-bound) */
  const int K = 20000;
  double t0 = now();
  for (int i = 0; i < K; ++i) norm_launch_ex(out, in, n, &o);
  cudaStreamSynchronize(st);
  *b2b_us = (now() - t0) / K * 1e6;
  return cudaGetLastError() != cudaSuccess;
}

int main(int argc, char** argv) {
  int64_t sizes[8] = {1024, (1 << 20) + 7};
  int nsizes = 2;
  if (argc > 1) {
    nsizes = 0;
    for (int i = 1; i < argc && nsizes < 8; ++i) sizes[nsizes++] = atoll(argv[i]);
  }
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return 2;
  for (int s = 0; s < nsizes; ++s) {
    const int64_t n = sizes[s];
    float *in, *out;
    if (cudaMalloc((void**)&in, (size_t)n * 4) != cudaSuccess ||
        cudaMalloc((void**)&out, (size_t)n * 4) != cudaSuccess)
      return 2;
    float* h = (float*)malloc((size_t)n * 4);
    for (int64_t i = 0; i < n; ++i) h[i] = 1.0f + (float)(i % 8);
    cudaMemcpy(in, h, (size_t)n * 4, cudaMemcpyHostToDevice);
    free(h);
    for (int p = 0; p < 6; ++p) {
      double e0, b0, e1, b1;
      if (run(n, p, 0u, out, in, st, &e0, &b0) || run(n, p, NORM_FLAG_TRUSTED_PTRS, out, in, st, &e1, &b1)) {
        printf("{\"n\": %lld, \"path\": \"%s\", \"error\": \"%s\"}\n", (long long)n, kPath[p], norm_last_error());
        continue;
      }
      /* the same call as one CUDA graph replayed */
      norm_opts_t o = NORM_OPTS_INIT;
      o.path = p;
      norm_graph_t* g = NULL;
      double eg = -1, bg = -1;
      if (norm_graph_create(&g, out, in, n, &o) == NORM_OK) {
        const int K = 20000, B = 64, NB = 200;
        for (int i = 0; i < 500; ++i) norm_graph_launch(g, st);
        cudaStreamSynchronize(st);
        double host = 0.0;
        for (int b = 0; b < NB; ++b) {
          double t0 = now();
          for (int i = 0; i < B; ++i) norm_graph_launch(g, st);
          host += now() - t0;
          cudaStreamSynchronize(st);
        }
        eg = host / (B * NB) * 1e6;
        double t0 = now();
        for (int i = 0; i < K; ++i) norm_graph_launch(g, st);
        cudaStreamSynchronize(st);
        bg = (now() - t0) / K * 1e6;
        norm_graph_destroy(g);
      }
      int32_t chosen = p;
      int64_t count = 0, prefix = 0;
      norm_coverage(n, NORM_INDEX_LITERAL, &count, &prefix);
      norm_choose_path(n, prefix, p, &chosen);
      printf("{\"n\": %lld, \"path\": \"%s\", \"runs\": \"%s\", \"host_enqueue_us\": %.3f, "
             "\"back_to_back_us\": %.3f, \"trusted_host_enqueue_us\": %.3f, \"trusted_back_to_back_us\": %.3f, "
             "\"graph_host_enqueue_us\": %.3f, \"graph_back_to_back_us\": %.3f}\n",
             (long long)n, kPath[p], kPath[chosen], e0, b0, e1, b1, eg, bg);
      fflush(stdout);
    }
    cudaFree(in);
    cudaFree(out);
  }
  return 0;
}
