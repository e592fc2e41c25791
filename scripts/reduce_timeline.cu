// scripts/reduce_timeline.cu — design probe (not product code): where does the
// reduce kernel's ~9.5 us fixed cost per launch go?  An instrumented copy of
// reduce_bulk_kernel's structure (same ring, chunking, combine) records
// %globaltimer per CTA at: entry, first chunk landed, last chunk consumed,
// partial written, (last CTA) S written.  Launched back to back like the bench;
// prints the medians over CTAs relative to the earliest CTA entry, for n = 2^29
// (the W = 8 shard) and 2^32.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_2207_00257_b200/csrc -I include scripts/reduce_timeline.cu -o scripts/mb_timeline
#include <cuda_runtime.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "stream_common.cuh"

using namespace lnorm;

__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(BK_THREADS, 1)
    reduce_timeline(const float* __restrict__ in, int64_t n, double* partials, unsigned* ticket,
                    double* S_out, unsigned long long* ts) {
  const unsigned long long t0 = now_ns();
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[BK_STAGES], empty[BK_STAGES];
  __shared__ double red[BK_THREADS / 32];
  __shared__ unsigned is_last;
  __shared__ unsigned long long t_first, t_last;
  auto r = bulk_ring_init<BK_STAGES, BK_CHUNK>(ring, full, empty);
  double acc = 0.0;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) bulk_produce<false>(r, in, n, 0);
  } else {
    const int ct = threadIdx.x - 32;
    constexpr int64_t CF = BulkRing<BK_STAGES, BK_CHUNK>::CF;
    int64_t head, nchunks;
    bulk_split<CF>(in, n, &head, &nchunks);
    bool first = true;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      mbar_wait(&r.full[r.stage], r.phase);
      if (first && ct == 0) t_first = now_ns();
      first = false;
      const float4* q = reinterpret_cast<const float4*>(r.buf + (size_t)r.stage * BK_CHUNK);
#pragma unroll
      for (int k = 0; k < BK_CHUNK / 32 / BK_CONSUMERS; ++k) {
        const int i = k * BK_CONSUMERS + ct;
        const float4 a = q[2 * i], b = q[2 * i + 1];
        f8 v = {{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}};
        acc += sum8(v);
      }
      stage_release(&r.empty[r.stage]);
      r.advance();
    }
    if (ct == 0) t_last = now_ns();
  }
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = b;
    __threadfence();
    const unsigned long long t_part = now_ns();
    ts[blockIdx.x * 5 + 0] = t0;
    ts[blockIdx.x * 5 + 1] = t_first;
    ts[blockIdx.x * 5 + 2] = t_last;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    ts[blockIdx.x * 5 + 3] = smid;
    is_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += BK_THREADS) v += __ldcg(partials + i);
  const double S = block_sum(v, red);
  if (threadIdx.x == 0) {
    *S_out = S;
    *ticket = 0u;
    ts[gridDim.x * 5] = now_ns();
  }
}

__global__ void empty_kernel() {}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t nmax = 1ll << 32;
  float* in;
  cudaMalloc(&in, nmax * 4);
  cudaMemset(in, 0x3c, nmax * 4);
  double *partials, *S;
  unsigned* ticket;
  unsigned long long* ts;
  cudaMalloc(&partials, 4096 * 8);
  cudaMalloc(&S, 64);
  cudaMalloc(&ticket, 64);
  cudaMemset(ticket, 0, 64);
  cudaMalloc(&ts, (sms * 5 + 8) * 8);
  cudaFuncSetAttribute(reduce_timeline, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BK_SMEM);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // back-to-back empty launches of the same geometry: the launch floor
  for (int i = 0; i < 10; ++i) empty_kernel<<<sms, BK_THREADS>>>();
  cudaEventRecord(a);
  for (int i = 0; i < 100; ++i) empty_kernel<<<sms, BK_THREADS>>>();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("empty kernel <<<%d, %d>>> back to back: %.2f us per launch\n", sms, BK_THREADS, ms * 10.f);
  for (int64_t n : {1ll << 29, 1ll << 32}) {
    const int K = n == (1ll << 29) ? 40 : 8;
    std::vector<unsigned long long> h((sms * 5 + 1));
    std::vector<double> first, last, part, ends, kern;
    for (int k = 0; k < K; ++k) {
      cudaEventRecord(a);
      reduce_timeline<<<sms, BK_THREADS, BK_SMEM>>>(in, n, partials, ticket, S, ts);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      cudaMemcpy(h.data(), ts, h.size() * 8, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ull, t0max = 0, lastmax = 0, partmax = 0;
      std::vector<double> f, l;
      for (int c = 0; c < sms; ++c) {
        t0 = std::min(t0, h[c * 5]);
        t0max = std::max(t0max, h[c * 5]);
      }
      for (int c = 0; c < sms; ++c) {
        f.push_back((double)(h[c * 5 + 1] - t0));
        l.push_back((double)(h[c * 5 + 2] - t0));
        lastmax = std::max(lastmax, h[c * 5 + 2]);
        partmax = 0;
      }
      if (k == K - 1) {  // per-SM finish offsets of the last run, to see whether the slow SMs repeat
        std::vector<std::pair<double, int>> fin;
        for (int c = 0; c < sms; ++c) fin.push_back({(double)(h[c * 5 + 2] - t0) / 1e3, (int)h[c * 5 + 3]});
        std::sort(fin.begin(), fin.end());
        printf("n=2^%d finish (us, smid) fastest 8:", n == (1ll << 29) ? 29 : 32);
        for (int i = 0; i < 8; ++i) printf(" %.1f/%d", fin[i].first, fin[i].second);
        printf("\n   percentiles 10/25/50/75/90: %.1f %.1f %.1f %.1f %.1f\n   slowest 12:", fin[sms / 10].first,
               fin[sms / 4].first, fin[sms / 2].first, fin[3 * sms / 4].first, fin[9 * sms / 10].first);
        for (int i = sms - 12; i < sms; ++i) printf(" %.1f/%d", fin[i].first, fin[i].second);
        printf("\n");
      }
      std::sort(f.begin(), f.end());
      std::sort(l.begin(), l.end());
      if (k == 0) continue;  // warm-up
      first.push_back(f[sms / 2]);
      last.push_back(l[0]);  // earliest CTA to finish streaming
      ends.push_back((double)(lastmax - t0));
      part.push_back((double)(h[sms * 5] - t0));
      kern.push_back(ms * 1e6);
      (void)t0max;
      (void)partmax;
    }
    auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
    const double bytes = 4.0 * n;
    printf("n=2^%d: event time %.1f us | from first CTA entry: median first chunk %.2f us, earliest CTA done "
           "streaming %.1f us, last CTA done streaming %.1f us, S written %.1f us | ideal at 7.5 TB/s %.1f us\n",
           n == (1ll << 29) ? 29 : 32, med(kern) / 1e3, med(first) / 1e3, med(last) / 1e3, med(ends) / 1e3,
           med(part) / 1e3, bytes / 7.5e12 * 1e6);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
