/* gen/gen_host.c — host fill for the seeded input generator (gen/norm_gen.h).
 * Not part of the method: it only manufactures inputs for tests and the bench.
 * Large fills are split over the host cores with pthreads (pure per-index
 * function, so the split does not change any value). */
#define _GNU_SOURCE
#include <pthread.h>
#include <unistd.h>

#include "norm_gen.h"

typedef struct { float* out; int64_t begin, end, offset; uint64_t seed; int dist; } job_t;

static void* fill_job(void* p) {
  job_t* j = (job_t*)p;
  for (int64_t i = j->begin; i < j->end; ++i)
    j->out[i] = ng_value(j->seed, j->dist, (uint64_t)(j->offset + i));
  return NULL;
}

int ng_fill_host(float* out, int64_t n, uint64_t seed, int dist, int64_t offset) {
  if (n < 0 || (n > 0 && !out) || dist < 0 || dist >= NG_DIST_COUNT || offset < 0) return 1;
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  if (nt < 1 || n < (1 << 20)) nt = 1;
  if (nt > 64) nt = 64;
  pthread_t th[64];
  job_t jobs[64];
  for (long t = 0; t < nt; ++t) {
    jobs[t] = (job_t){out, n * t / nt, n * (t + 1) / nt, offset, seed, dist};
    if (t > 0 && pthread_create(&th[t], NULL, fill_job, &jobs[t]) != 0) fill_job(&jobs[t]), th[t] = 0;
  }
  fill_job(&jobs[0]);
  for (long t = 1; t < nt; ++t) if (th[t]) pthread_join(th[t], NULL);
  return 0;
}

float ng_value_host(uint64_t seed, int dist, int64_t i) { return ng_value(seed, dist, (uint64_t)i); }
