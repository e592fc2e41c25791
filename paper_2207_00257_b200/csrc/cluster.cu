// cluster.cu — the whole call in ONE thread-block cluster (NORM_PATH_CLUSTER):
// for L2-sized inputs (BASELINE configs[1], n = 2^20 + 7) the cost is latency,
// not bandwidth -- two launches (two-pass), or one cooperative launch of 148
// CTAs with a grid barrier through global memory (mid), cost more than the
// bytes.  A cluster of 16 CTAs (the non-portable maximum; 16 SMs, 16 x 1024
// threads) is co-scheduled by the hardware without a cooperative launch, and
// its combine goes through distributed shared memory: every CTA sums its
// 256-bit vectors of `in` (the fixed per-thread order of accumulate_segment),
// reduces them in the block, and publishes the block partial in its own shared
// memory; one cluster barrier (release / acquire); every CTA reads the 16
// partials over DSMEM in rank order (identical S in every CTA, no global
// workspace, no counters); a second cluster barrier keeps every CTA's shared
// memory alive until all have read it; then the covered prefix is scaled.
// All loads of `in` precede the first barrier, so out may alias in.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include "stream_common.cuh"

namespace lnorm {

constexpr int CL_THREADS = 1024, CL_UNROLL = 4;

__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_nctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// fp64 load from CTA `rank`'s copy of the shared variable at local address `p`
__device__ __forceinline__ double ld_dsmem_f64(const double* p, unsigned rank) {
  const unsigned local = (unsigned)__cvta_generic_to_shared(p);
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
  return v;
}

template <bool VEC>
__global__ void __launch_bounds__(CL_THREADS, 1)
    cluster_kernel(float* out, const float* in, int64_t n, int64_t L, float* sum_out, double* sum_out_f64) {
  // programmatic dependent of the preceding kernel (pdl_chain): wait for it first
  pdl_wait();
  pdl_launch_dependents();
  __shared__ double red[CL_THREADS / 32];
  __shared__ double part;
  const unsigned rank = cluster_ctarank(), nrank = cluster_nctarank();
  double acc = 0.0;
  accumulate_segment<CL_THREADS, CL_UNROLL, LD_PLAIN>(in, n, (int)rank, (int)nrank, acc, 0);
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) part = b;
  cluster_sync_all();  // every partial published; every load of `in` done
  double S = 0.0;
  if (threadIdx.x < 32) {  // rank order, identical in every CTA
    double v = (threadIdx.x < nrank) ? ld_dsmem_f64(&part, threadIdx.x) : 0.0;
    // fixed-order combine: a sequential sum in rank order (lane 0)
    for (unsigned r = 0; r < nrank; ++r) {
      const double pr = __shfl_sync(0xffffffffu, v, (int)r);
      S = r == 0 ? pr : S + pr;
    }
  }
  cluster_sync_all();  // all DSMEM reads done before any CTA may exit
  if (threadIdx.x == 0) red[0] = S;
  __syncthreads();
  S = red[0];
  const float s = (float)S;
  if (rank == 0 && threadIdx.x == 0) {
    if (sum_out) *sum_out = s;
    if (sum_out_f64) *sum_out_f64 = S;
  }
  scale_segment<CL_THREADS, 2, VEC, true>(out, in, L, s, (int)rank, (int)nrank);
}

// Cluster size: 16 (non-portable) when the device can schedule it, else 8.
static int cluster_size_for(void* fn) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  cfg.blockDim = dim3(CL_THREADS);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int c : {16, 8}) {
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(c);
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) == cudaSuccess && nclusters >= 1) return c;
    cudaGetLastError();
  }
  return 0;
}

cudaError_t launch_cluster(float* out, const float* in, const Coverage& cov, float* sum_out,
                           double* sum_out_f64, const DeviceInfo& d, cudaStream_t st) {
  const bool vec = ((reinterpret_cast<uintptr_t>(out) - reinterpret_cast<uintptr_t>(in)) & 31u) == 0;
  void* fn = vec ? (void*)cluster_kernel<true> : (void*)cluster_kernel<false>;
  static int csize[64][2] = {};
  if (d.device >= 64) return cudaErrorInvalidDevice;
  if (!csize[d.device][vec]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    const int c = cluster_size_for(fn);
    if (!c) return cudaErrorInvalidConfiguration;
    csize[d.device][vec] = c;
  }
  const int c = csize[d.device][vec];
  int64_t n = cov.n, L = cov.L;
  void* args[] = {&out, (void*)&in, &n, &L, &sum_out, &sum_out_f64};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(c);
  cfg.blockDim = dim3(CL_THREADS);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = c;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_chain() && pdl_mode() != PDL_OFF) ? 2 : 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace lnorm
