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
template <int T, int STAGES, int STAGE_BYTES, int MINB = 1, bool CONTIG = false>
__global__ void __launch_bounds__(T, MINB) red_bulk(const float* in, int64_t nbytes_total, double* out) {
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
      const int64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
      const int64_t c0 = CONTIG ? blockIdx.x * per : blockIdx.x;
      const int64_t c1 = CONTIG ? (c0 + per < nchunks ? c0 + per : nchunks) : nchunks;
      const int64_t cs = CONTIG ? 1 : gridDim.x;
      for (int64_t c = c0; c < c1; c += cs, ++it) {
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
    const int64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
    const int64_t c0 = CONTIG ? blockIdx.x * per : blockIdx.x;
    const int64_t c1 = CONTIG ? (c0 + per < nchunks ? c0 + per : nchunks) : nchunks;
    const int64_t cs = CONTIG ? 1 : gridDim.x;
    for (int64_t c = c0; c < c1; c += cs) {
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

template <int T, int U, int MINB, int AHEAD>
__global__ void __launch_bounds__(T, MINB) red_ldg_pf(const float* in, int64_t nv, double* out) {
  __shared__ double red[T / 32];
  double acc = 0;
  constexpr int64_t CH = (int64_t)T * U;
  const int64_t nfull = nv / CH;
  for (int64_t c = blockIdx.x; c < nfull; c += gridDim.x) {
    if (threadIdx.x == 0) {
      const int64_t cp = c + (int64_t)AHEAD * gridDim.x;
      if (cp < nfull)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(in + cp * CH * 8), "r"((int)(CH * 32)) : "memory");
    }
    const float* q = in + (c * CH + threadIdx.x) * 8;
    f8 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld8_stream(q + (int64_t)u * T * 8);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += sum8(v[u]);
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

__global__ void fill_hash(float* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)(i * 2654435761u) ^ (uint32_t)(i >> 7);
    p[i] = 0.5f + (float)(h >> 8) * 5.9604645e-08f;
  }
}

int main(int argc, char** argv) {
  const int64_t n = 1ll << 32;
  const bool random = argc > 1;
  float* in;
  double* out;
  if (cudaMalloc(&in, n * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMalloc(&out, 1 << 20);
  cudaMemset(in, 0, n * 4);
  if (random) fill_hash<<<148 * 8, 256>>>(in, n);
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
#define RUNB2(NAME, T, ST, SB, MB, CG)                                                               \
  {                                                                                                \
    cudaFuncSetAttribute(red_bulk<T, ST, SB, MB, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST * SB); \
    float ms = timeit([&] { red_bulk<T, ST, SB, MB, CG><<<sms * MB, T, ST * SB>>>(in, n * 4, out); });       \
    cudaError_t e = cudaGetLastError();                                                            \
    printf("%-40s %8.3f ms %8.1f GB/s %s\n", NAME, ms, bytes / ms / 1e6, cudaGetErrorString(e));   \
  }
  RUNB2("bulk 288 6x16KiB", 288, 6, 16384, 1, false);
  RUNB2("bulk 288 7x16KiB", 288, 7, 16384, 1, false);
  RUNB2("bulk 288 8x16KiB", 288, 8, 16384, 1, false);
  RUNB2("bulk 288 9x16KiB", 288, 9, 16384, 1, false);
  RUNB2("bulk 288 10x16KiB", 288, 10, 16384, 1, false);
  RUNB2("bulk 288 16x8KiB", 288, 16, 8192, 1, false);
  RUNB2("bulk 288 20x8KiB", 288, 20, 8192, 1, false);
  RUNB2("bulk 288 4x32KiB", 288, 4, 32768, 1, false);
  RUNB2("bulk 160 8x16KiB", 160, 8, 16384, 1, false);
  RUNB2("bulk 544 8x16KiB", 544, 8, 16384, 1, false);
  RUNB2("bulk 288 8x16KiB contig", 288, 8, 16384, 1, true);
  RUNB2("bulk 288 6x16KiB contig", 288, 6, 16384, 1, true);
  RUNB2("bulk 288 12x16KiB contig", 288, 12, 16384, 1, true);
  RUNB2("bulk 2x160 4x16KiB", 160, 4, 16384, 2, false);
  RUNB2("bulk 2x160 4x16KiB contig", 160, 4, 16384, 2, true);
  // copy-rate reference: cudaMemcpy D2D of 8 GiB (read+write counted)
  float* o2;
  cudaMalloc(&o2, n * 2);
  float ms = timeit([&] { cudaMemcpyAsync(o2, in, n * 2, cudaMemcpyDeviceToDevice); });
  printf("%-40s %8.3f ms %8.1f GB/s (r+w)\n", "cudaMemcpy D2D 8 GiB", ms, 2.0 * n * 2 / ms / 1e6);
  return 0;
}
