// scripts/microbench_reduce.cu — design-space probe for libnorm's reduce kernel
// (not product code): read-only streaming sum of n fp32 on B200 with several load
// schemes; prints GB/s for each.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -std=c++17 -I paper_2207_00257_b200/csrc scripts/microbench_reduce.cu -o mb
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "device_common.cuh"

using namespace lnorm;

__device__ __forceinline__ f8 ld8_l2pf(const float* p) {
  f8 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                 "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
               : "l"(p));
  return r;
}

template <int T, int U, int MINB, bool PF>
__global__ void __launch_bounds__(T, MINB) red_ldg(const float* in, int64_t nv, double* out) {
  __shared__ double red[T / 32];
  double acc = 0;
  constexpr int64_t CH = (int64_t)T * U;
  const int64_t nfull = nv / CH;
  for (int64_t c = blockIdx.x; c < nfull; c += gridDim.x) {
    const float* q = in + (c * CH + threadIdx.x) * 8;
    f8 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = PF ? ld8_l2pf(q + (int64_t)u * T * 8) : ld8_stream(q + (int64_t)u * T * 8);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += sum8(v[u]);
  }
  double b = block_sum(acc, red);
  if (threadIdx.x == 0) out[blockIdx.x] = b;
}

// TMA 1-D bulk copies into a ring of shared-memory stages (one elected producer
// thread), consumer warps sum from shared memory.
template <int T, int STAGES, int STAGE_BYTES>
__global__ void __launch_bounds__(T, 1) red_bulk(const float* in, int64_t nbytes_total, double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES];
  __shared__ double red[T / 32];
  const int64_t nchunks = nbytes_total / STAGE_BYTES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      unsigned a = (unsigned)__cvta_generic_to_shared(&full[s]);
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(a));
      unsigned b = (unsigned)__cvta_generic_to_shared(&empty[s]);
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(b), "r"(T / 32 - 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0;
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      unsigned ph = 0;
      int it = 0;
      for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        if (it >= STAGES) {
          unsigned b = (unsigned)__cvta_generic_to_shared(&empty[s]);
          asm volatile(
              "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(b),
              "r"(ph ^ 1));
        }
        unsigned fb = (unsigned)__cvta_generic_to_shared(&full[s]);
        unsigned dst = (unsigned)__cvta_generic_to_shared(smem + (size_t)s * STAGE_BYTES);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(fb), "r"(STAGE_BYTES));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
            "l"((const char*)in + c * STAGE_BYTES), "r"(STAGE_BYTES), "r"(fb)
            : "memory");
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {
    int s = 0;
    unsigned ph = 0;
    const int cw = warp - 1, ncw = T / 32 - 1;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      unsigned fb = (unsigned)__cvta_generic_to_shared(&full[s]);
      asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(fb),
                   "r"(ph));
      const float4* p = reinterpret_cast<const float4*>(smem + (size_t)s * STAGE_BYTES);
      for (int i = cw * 32 + lane; i < STAGE_BYTES / 16; i += ncw * 32) {
        float4 v = p[i];
        acc += (double)((v.x + v.y) + (v.z + v.w));
      }
      __syncwarp();
      if (lane == 0) {
        unsigned eb = (unsigned)__cvta_generic_to_shared(&empty[s]);
        asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(eb));
      }
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
  }
  double b = block_sum(acc, red);
  if (threadIdx.x == 0) out[blockIdx.x] = b;
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

int main() {
  const int64_t n = 1ll << 32;
  float* in;
  double* out;
  if (cudaMalloc(&in, n * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&out, 1 << 20);
  cudaMemset(in, 0, n * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = (double)n * 4;
  const int64_t nv = n / 8;
#define RUN(NAME, T, U, MINB, PF, CTAS)                                                   \
  {                                                                                     \
    float ms = timeit([&] { red_ldg<T, U, MINB, PF><<<sms * CTAS, T>>>(in, nv, out); });  \
    printf("%-40s %8.3f ms %8.1f GB/s\n", NAME, ms, bytes / ms / 1e6);                  \
  }
  RUN("ldg256 512x2 U4 (current)", 512, 4, 2, false, 2);
  RUN("ldg256 512x2 U4 L2::256B", 512, 4, 2, true, 2);
  RUN("ldg256 256x4 U4", 256, 4, 4, false, 4);
  RUN("ldg256 256x3 U8", 256, 8, 3, false, 3);
  RUN("ldg256 1024x1 U4", 1024, 4, 1, false, 1);
  RUN("ldg256 512x2 U2", 512, 2, 2, false, 2);
  RUN("ldg256 128x8 U4", 128, 4, 8, false, 8);
  RUN("ldg256 256x4 U4 L2::256B", 256, 4, 4, true, 4);
  RUN("ldg256 512x1 U8", 512, 8, 1, false, 1);
#define RUNB(NAME, T, ST, SB)                                                                   \
  {                                                                                             \
    cudaFuncSetAttribute(red_bulk<T, ST, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SB); \
    float ms = timeit([&] { red_bulk<T, ST, SB><<<sms, T, ST * SB>>>(in, n * 4, out); });        \
    cudaError_t e = cudaGetLastError();                                                         \
    printf("%-40s %8.3f ms %8.1f GB/s %s\n", NAME, ms, bytes / ms / 1e6, cudaGetErrorString(e)); \
  }
  RUNB("bulk 288thr 8x16KiB", 288, 8, 16384);
  RUNB("bulk 288thr 6x32KiB", 288, 6, 32768);
  RUNB("bulk 544thr 12x16KiB", 544, 12, 16384);
  RUNB("bulk 544thr 4x48KiB", 544, 4, 49152);
  // copy-rate reference: cudaMemcpy D2D of 8 GiB (read+write counted)
  float* o2;
  cudaMalloc(&o2, n * 2);
  float ms = timeit([&] { cudaMemcpyAsync(o2, in, n * 2, cudaMemcpyDeviceToDevice); });
  printf("%-40s %8.3f ms %8.1f GB/s (r+w)\n", "cudaMemcpy D2D 8 GiB", ms, 2.0 * n * 2 / ms / 1e6);
  return 0;
}
