// reduce.cu — the hoisted `sum` of Fig. 1 (hoisted by parallel
// LICM): S = sum in[0, n) as one HBM read stream.  A TMA-bulk
// ring kernel for n >= 2^22, an LDG.E.256 kernel below; per-CTA partials combined
// in index order by the last CTA (ticket), optionally published to peer GPUs.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include "stream_common.cuh"

namespace lnorm {

// --------------------------------------------------------------- reduce
// Pass 1 of the two-pass path: S = sum in[0, n).  Persistent grid (2 CTAs/SM),
// per-CTA partial, last-CTA ticket combines the partials in index order.
__global__ void __launch_bounds__(RED_THREADS, RED_CTAS_PER_SM)
    reduce_kernel(const float* __restrict__ in, int64_t n, double* __restrict__ partials,
                  unsigned* __restrict__ ticket, double* __restrict__ S_out, int early_trigger,
                  PeerPost post) {
  // The scale kernel (PDL dependent) may be scheduled once every CTA has
  // triggered; it blocks in griddepcontrol.wait until this grid has completed.
  if (early_trigger) pdl_launch_dependents();
  __shared__ double red[RED_THREADS / 32];
  __shared__ unsigned is_last;
  double acc = 0.0;
  accumulate_segment<RED_THREADS, RED_UNROLL, LD_STREAM>(in, n, blockIdx.x, gridDim.x, acc, 0);
  if (!early_trigger) pdl_launch_dependents();
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = b;
    __threadfence();
    is_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += RED_THREADS) v += __ldcg(partials + i);
  const double S = block_sum(v, red);
  if (threadIdx.x == 0) {
    *S_out = S;
    *ticket = 0u;  // leave the workspace reusable
  }
  if (threadIdx.x < 32) publish_partial_warp(post, S);
}

// Pass 1, TMA-bulk variant for n >= 2^22 (one CTA per SM), then the same
// last-CTA ticket combine as reduce_kernel.
__global__ void __launch_bounds__(BK_THREADS, 1)
    reduce_bulk_kernel(const float* __restrict__ in, int64_t n, double* __restrict__ partials,
                       unsigned* __restrict__ ticket, double* __restrict__ S_out, int early_trigger,
                       PeerPost post) {
  if (early_trigger) pdl_launch_dependents();
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[BK_STAGES], empty[BK_STAGES];
  __shared__ double red[BK_THREADS / 32];
  __shared__ unsigned is_last;
  auto r = bulk_ring_init<BK_STAGES, BK_CHUNK>(ring, full, empty);
  double acc = 0.0;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) bulk_produce<false>(r, in, n, 0);
  } else {
    bulk_consume(r, in, n, acc, threadIdx.x - 32);
  }
  if (!early_trigger) pdl_launch_dependents();
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = b;
    __threadfence();
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
  }
  if (threadIdx.x < 32) publish_partial_warp(post, S);
}

#ifdef NORM_TIMELINE  // probe builds only (scripts/pdl_timeline.py): per-CTA %globaltimer stamps
__device__ unsigned long long g_reduce_ts[4096 * 4];
#define RED_STAMP(k) \
  if (threadIdx.x == 0) g_reduce_ts[blockIdx.x * 4 + (k)] = globaltimer_ns();
extern "C" __attribute__((visibility("default"))) int norm_debug_reduce_timeline(unsigned long long* host,
                                                                                  int n) {
  return (int)cudaMemcpyFromSymbol(host, g_reduce_ts, (size_t)n * sizeof(unsigned long long));
}
#else
#define RED_STAMP(k)
#endif

// Pass 1, TMA-bulk with a dynamically scheduled, still deterministic tail
// (dyn_stream_sum, stream_common.cuh): per-CTA partials for the grid-strided
// chunks, task sums for the last `dyn` chunks; the last CTA adds the partials,
// then the task sums, in index order.
__global__ void __launch_bounds__(BK_THREADS, 1)
    reduce_dyn_kernel(const float* __restrict__ in, int64_t n, double* __restrict__ partials,
                      unsigned* __restrict__ ticket, double* __restrict__ S_out, int early_trigger,
                      PeerPost post, unsigned* __restrict__ task_ctr, double* __restrict__ task_sums,
                      int64_t dyn, int tc) {
  RED_STAMP(0);  // entry
  if (early_trigger) pdl_launch_dependents();
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[BK_STAGES], empty[BK_STAGES];
  __shared__ DynSmem dsm;
  __shared__ double red[BK_THREADS / 32];
  __shared__ unsigned is_last;
  if (threadIdx.x < 2) dsm.slot_cnt[threadIdx.x] = 0u;
  auto r = bulk_ring_init<BK_STAGES, BK_CHUNK>(ring, full, empty);
  const DynSeg seg[1] = {{in, n, 0, 0}};
  int64_t ntasks;
  const double acc = dyn_stream_sum<1>(r, seg, dyn, tc, task_ctr, task_sums, dsm, &ntasks);
  RED_STAMP(1);  // streaming done (the late PDL trigger)
  if (!early_trigger) pdl_launch_dependents();
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = b;
    __threadfence();
    is_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  RED_STAMP(2);  // partial published
  if (!is_last) return;
  __threadfence();
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += BK_THREADS) v += __ldcg(partials + i);
  for (int64_t t = threadIdx.x; t < ntasks; t += BK_THREADS) v += __ldcg(task_sums + t);
  const double S = block_sum(v, red);
  if (threadIdx.x == 0) {
    *S_out = S;
    *ticket = 0u;
    *task_ctr = 0u;
  }
  if (threadIdx.x < 32) publish_partial_warp(post, S);
  RED_STAMP(3);  // last CTA: S written
}

int reduce_grid(const DeviceInfo& d, int64_t n) {
  const int64_t chunks = (n / 8 + (int64_t)RED_THREADS * RED_UNROLL - 1) / ((int64_t)RED_THREADS * RED_UNROLL);
  int64_t g = (int64_t)d.sms * RED_CTAS_PER_SM;
  if (chunks < g) g = chunks < 1 ? 1 : chunks;
  if (g > kMaxGrid) g = kMaxGrid;
  return (int)g;
}

// Programmatic dependent launch of the scale after the reduce.  NORM_PDL=off |
// early (trigger at the reduce's start) | late (trigger after its streaming loop,
// the default): a tuning knob read once; every mode gives identical results.
int pdl_mode() {
  static int mode = [] {
    const char* e = getenv("NORM_PDL");
    if (e && !strcmp(e, "off")) return (int)PDL_OFF;
    if (e && !strcmp(e, "early")) return (int)PDL_EARLY;
    return (int)PDL_LATE;
  }();
  return mode;
}

// Latency-bound one-launch paths (small, mid) are launched as programmatic
// dependents of whatever precedes them on the stream and trigger their own
// dependents at entry, so back-to-back calls overlap one launch's latency with
// the previous call (NORM_PDL_CHAIN=0 turns it off for A/B runs).
bool pdl_chain() {
  static const bool on = [] {
    const char* e = getenv("NORM_PDL_CHAIN");
    return !(e && !strcmp(e, "0"));
  }();
  return on;
}

// Dynamic tail of the bulk reduce / fused phase 1: the last pct % of the chunks
// (NORM_DYN_PCT, default kDynPct; 0 = fully static reduce_bulk_kernel) but at
// least kDynMinTasksPerCTA tasks per CTA, so smaller inputs still get a fine
// enough tail (2^28: 3 % would be fewer tasks than CTAs), in tasks of tc chunks
// (NORM_DYN_TC, default kDynTC; kDynMinTC at those sizes), at most half the
// chunks and kMaxTasks tasks.
constexpr int kDynPct = 3, kDynTC = 8;  // profiles/r05/dyn_sweep2.txt
constexpr int kDynMinTasksPerCTA = 4;

int64_t dyn_chunks(int64_t n, int grid, int* tc_out) {
  static const int pct = [] {
    const char* e = getenv("NORM_DYN_PCT");
    return e ? atoi(e) : kDynPct;
  }();
  static const int tc_env = [] {
    const char* e = getenv("NORM_DYN_TC");
    const int v = e ? atoi(e) : kDynTC;
    return v < kDynMinTC ? kDynMinTC : v;
  }();
  const int64_t nchunks = n / (BK_CHUNK / 4);
  int tc = tc_env;
  int64_t dyn = nchunks * pct / 100;
  const int64_t floor_tasks = (int64_t)kDynMinTasksPerCTA * grid;
  if (dyn < floor_tasks * tc) {  // too few tasks: smallest tasks, and at least floor_tasks of them
    tc = kDynMinTC;
    if (dyn < floor_tasks * tc) dyn = floor_tasks * tc;
  }
  if (dyn > nchunks / 2) dyn = nchunks / 2;
  if (dyn > (int64_t)kMaxTasks * tc) dyn = (int64_t)kMaxTasks * tc;
  *tc_out = tc;
  return pct > 0 ? dyn : 0;
}

cudaError_t launch_reduce(const float* in, int64_t n, const Workspace& ws, double* S_out,
                          const DeviceInfo& d, cudaStream_t st, PeerPost post) {
#if defined(NORM_FAULT) && NORM_FAULT == 1  // fault (tests only): the sum drops the last element
  if (n > 1) n -= 1;
#endif
  if (n >= kBulkMinN) {
    static int configured[64] = {0};  // per device: opt in to 128 KiB of dynamic smem
    const size_t smem = BK_SMEM;
    if (d.device < 64 && !configured[d.device]) {
      cudaError_t e = cudaFuncSetAttribute(reduce_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      configured[d.device] = 1;
    }
    int tc = 0;
    const int64_t dyn = dyn_chunks(n, d.sms, &tc);
    if (dyn > 0) {
      static int configured_dyn[64] = {0};
      if (d.device < 64 && !configured_dyn[d.device]) {
        cudaError_t e = cudaFuncSetAttribute(reduce_dyn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured_dyn[d.device] = 1;
      }
      reduce_dyn_kernel<<<d.sms, BK_THREADS, smem, st>>>(in, n, ws.partials, ws.ticket, S_out,
                                                         pdl_mode() == PDL_EARLY, post, ws.task_ctr,
                                                         ws.task_sums, dyn, tc);
      return cudaGetLastError();
    }
    reduce_bulk_kernel<<<d.sms, BK_THREADS, smem, st>>>(in, n, ws.partials, ws.ticket, S_out,
                                                        pdl_mode() == PDL_EARLY, post);
    return cudaGetLastError();
  }
  reduce_kernel<<<reduce_grid(d, n), RED_THREADS, 0, st>>>(in, n, ws.partials, ws.ticket, S_out,
                                                            pdl_mode() == PDL_EARLY, post);
  return cudaGetLastError();
}

}  // namespace lnorm
