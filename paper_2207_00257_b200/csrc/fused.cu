// fused.cu — reduce + grid barrier + scale in one cooperative kernel when the
// input exceeds L2 but the covered prefix fits: the prefix is
// read last with an L2 evict_last hint and scaled out of L2.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include "stream_common.cuh"

namespace lnorm {

#ifdef NORM_TIMELINE  // probe builds only (scripts/fused_timeline.py): per-CTA %globaltimer stamps
__device__ unsigned long long g_fused_ts[4096 * 5];
__device__ __forceinline__ unsigned long long stamp_ns() {  // ordered with memory ops
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
  return t;
}
#define FUSED_STAMP(k)                                                         \
  if (threadIdx.x == 32) g_fused_ts[blockIdx.x * 5 + (k)] = stamp_ns();
#else
#define FUSED_STAMP(k)
#endif

// Grid barrier by arrival count (one per kernel): `arrivals` only grows — each
// CTA's thread 0 adds 1 with a release reduction (no round trip) and spins on an
// acquire load until the count reaches this barrier's target, the next multiple
// of the grid size above the value it read at kernel start (that value is at
// least the previous barriers' total and below it plus one grid: no CTA of this
// kernel can complete the barrier before this one arrives).  The last arrival's
// add itself releases everyone (acquire of the final value synchronises with
// every CTA's release through the RMW chain).  64-bit: no wrap in practice.
__device__ __forceinline__ void grid_barrier_count(unsigned long long* arrivals, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_add_release_u64(arrivals, 1ull);
    while (ld_acquire_u64(arrivals) < target) {
    }
#ifdef NORM_TIMELINE
    g_fused_ts[blockIdx.x * 5 + 2] = stamp_ns();
#endif
  }
  __syncthreads();
}

// ---------------------------------------------------------------- fused
// Single pass: one cooperative CTA per SM streams the uncovered
// tail [L, n) through the TMA-bulk ring, then the covered prefix [0, L) (read
// LAST, with an L2 evict_last hint, so as much of it as fits is still in L2);
// grid barrier; every CTA combines the per-CTA partials in the same fixed order
// (identical s everywhere); then every thread scales the prefix with 256-bit
// loads (8 in flight per thread; mostly L2 hits) — measured faster here than
// the TMA ring (profiles/r05/fused_p2.txt).  hints: 2 = also evict_first on
// the tail (best while the prefix is small, <= L2/3), 1 = evict_last on the
// prefix only (measured best beyond that, scripts/fused_vs_twopass.py).
// Multi-GPU (post.mail set): after the barrier CTA 0 publishes the rank partial
// into every rank's mailbox and every CTA waits on the local mailbox (rank-order
// combine), so the exchange costs no extra launch.  VEC = out and in co-aligned
// mod 32 B (else the prefix is scaled with scalar loads).
template <bool VEC>
__global__ void __launch_bounds__(BK_THREADS, 1)
    fused_kernel(float* out, const float* in, int64_t n, int64_t L, double* partials,
                 float* sum_out, double* sum_out_f64, int hints, PeerPost post,
                 const double* mailbox, unsigned* task_ctr, double* task_sums, int64_t dyn, int tc,
                 unsigned long long* arrivals) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[BK_STAGES], empty[BK_STAGES];
  __shared__ DynSmem dsm;
  __shared__ double red[BK_THREADS / 32];
  __shared__ double S_sh;
  FUSED_STAMP(0)
  unsigned long long target = 0;  // grid_barrier_count's target
  if (threadIdx.x == 0) target = (ld_acquire_u64(arrivals) / gridDim.x + 1) * gridDim.x;
  if (threadIdx.x < 2) dsm.slot_cnt[threadIdx.x] = 0u;
  auto r = bulk_ring_init<BK_STAGES, BK_CHUNK>(ring, full, empty);
  // phase 1: the tail, then the covered prefix (read last), with a dynamic,
  // deterministic end (dyn_stream_sum)
  const DynSeg seg[2] = {{in + L, n - L, policy_evict_first(), hints >= 2 ? 1 : 0},
                         {in, L, policy_evict_last(), hints >= 1 ? 1 : 0}};
  int64_t ntasks;
  const double acc = dyn_stream_sum<2>(r, seg, dyn, tc, task_ctr, task_sums, dsm, &ntasks);
  FUSED_STAMP(1)
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = b;
  grid_barrier_count(arrivals, target);  // all of `in` has been read: `out` (possibly == in) may be written
  if (blockIdx.x == 0 && threadIdx.x == 0) *task_ctr = 0u;  // every CTA is done claiming
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += BK_THREADS) v += __ldcg(partials + i);
  for (int64_t t = threadIdx.x; t < ntasks; t += BK_THREADS) v += __ldcg(task_sums + t);
  double S = block_sum(v, red);  // identical bits in every CTA
  if (post.mail) {
    if (threadIdx.x < 32) {  // warp 0: lane-parallel publish (CTA 0) and mailbox wait
      if (blockIdx.x == 0) publish_partial_warp(post, S);
      double Sf;
      combine_parts_warp(mailbox, post.world, &Sf, post.epoch);
      if (threadIdx.x == 0) S_sh = Sf;
    }
    __syncthreads();
    S = S_sh;
  }
  const float s = (float)S;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (sum_out) *sum_out = s;
    if (sum_out_f64) *sum_out_f64 = S;
  }
  FUSED_STAMP(3)
  scale_segment<BK_THREADS, FU_SCALE_UNROLL, VEC, true>(out, in, L, s, blockIdx.x, gridDim.x);
  FUSED_STAMP(4)
}

// ------------------------------------------------------------------ mid
// One launch for L2-sized inputs (configs 2: n = 2^20 + 7): the two-pass path
// pays two launches (~8 us of host enqueue per call on this box, more than
// the ~6 us of device time) and the TMA fused kernel's ring set-up and dynamic
// tail cost more than they save when the whole input is a few MiB.  One
// cooperative CTA per SM: every thread sums its 256-bit vectors of `in`
// (coherent loads: out may alias in) with the fixed per-thread order of
// accumulate_segment; block_sum -> partials[cta]; grid barrier (the arrival
// count shared with fused_kernel: both grids are the SM count, so the count
// stays a multiple of it between kernels); every CTA adds the partials in
// index order (identical S everywhere); then the covered prefix is scaled from
// L2.  Multi-GPU (post.mail): CTA 0 publishes the rank partial, every CTA waits
// on the local mailbox, as in fused_kernel.
constexpr int MID_THREADS = 512, MID_UNROLL = 2;
template <bool VEC>
__global__ void __launch_bounds__(MID_THREADS, 1)
    mid_kernel(float* out, const float* in, int64_t n, int64_t L, double* partials, float* sum_out,
               double* sum_out_f64, PeerPost post, const double* mailbox, unsigned long long* arrivals) {
  __shared__ double red[MID_THREADS / 32];
  __shared__ double S_sh;
  pdl_wait();  // programmatic dependent of the preceding kernel (pdl_chain): wait for it first
  pdl_launch_dependents();
  unsigned long long target = 0;
  if (threadIdx.x == 0) target = (ld_acquire_u64(arrivals) / gridDim.x + 1) * gridDim.x;
  double acc = 0.0;
  accumulate_segment<MID_THREADS, MID_UNROLL, LD_PLAIN>(in, n, blockIdx.x, gridDim.x, acc, 0);
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = b;
  grid_barrier_count(arrivals, target);  // all of `in` has been read: `out` (possibly == in) may be written
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += MID_THREADS) v += __ldcg(partials + i);
  double S = block_sum(v, red);  // identical bits in every CTA
  if (post.mail) {
    if (threadIdx.x < 32) {  // warp 0: lane-parallel publish (CTA 0) and mailbox wait
      if (blockIdx.x == 0) publish_partial_warp(post, S);
      double Sf;
      combine_parts_warp(mailbox, post.world, &Sf, post.epoch);
      if (threadIdx.x == 0) S_sh = Sf;
    }
    __syncthreads();
    S = S_sh;
  }
  const float s = (float)S;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (sum_out) *sum_out = s;
    if (sum_out_f64) *sum_out_f64 = S;
  }
  scale_segment<MID_THREADS, MID_UNROLL, VEC, true>(out, in, L, s, blockIdx.x, gridDim.x);
}

cudaError_t launch_mid(float* out, const float* in, const Coverage& cov, const Workspace& ws,
                       float* sum_out, double* sum_out_f64, const DeviceInfo& d, cudaStream_t st,
                       PeerPost post, const double* mailbox) {
  const bool vec = ((reinterpret_cast<uintptr_t>(out) - reinterpret_cast<uintptr_t>(in)) & 31u) == 0;
  void* fn = vec ? (void*)mid_kernel<true> : (void*)mid_kernel<false>;
  int grid = d.sms;  // one CTA per SM (the arrival count's invariant, see mid_kernel)
  int64_t n = cov.n, L = cov.L;
  double* partials = ws.partials;
  unsigned long long* arrivals = ws.arrivals;
  void* args[] = {&out, (void*)&in, &n, &L, &partials, &sum_out, &sum_out_f64, &post, (void*)&mailbox,
                  &arrivals};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(MID_THREADS);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_chain() ? 2 : 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

#ifdef NORM_TIMELINE
extern "C" __attribute__((visibility("default"))) int norm_debug_fused_timeline(unsigned long long* host,
                                                                                 int n) {
  return (int)cudaMemcpyFromSymbol(host, g_fused_ts, (size_t)n * sizeof(unsigned long long));
}
#endif

// L2 hint policy (kernel comment): 2 while the covered prefix is <= L2/3, else 1.
// NORM_FUSED_HINTS=0|1|2 overrides (A/B experiments), read once.
static int fused_hints(const Coverage& cov, const DeviceInfo& d) {
  static const int forced = [] {
    const char* e = getenv("NORM_FUSED_HINTS");
    return e ? atoi(e) : -1;
  }();
  if (forced >= 0) return forced;
  return (size_t)cov.L * 4 <= d.l2_bytes / 3 ? 2 : 1;
}

cudaError_t launch_fused(float* out, const float* in, const Coverage& cov, const Workspace& ws,
                         float* sum_out, double* sum_out_f64, const DeviceInfo& d,
                         cudaStream_t st, PeerPost post, const double* mailbox) {
  const bool vec = ((reinterpret_cast<uintptr_t>(out) - reinterpret_cast<uintptr_t>(in)) & 31u) == 0;
  void* fn = vec ? (void*)fused_kernel<true> : (void*)fused_kernel<false>;
  static int configured[64][2] = {};
  if (d.device < 64 && !configured[d.device][vec]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BK_SMEM);
    if (e != cudaSuccess) return e;
    configured[d.device][vec] = 1;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, BK_THREADS, BK_SMEM);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  int grid = d.sms;  // one CTA per SM
  int64_t n = cov.n, L = cov.L;
  double* partials = ws.partials;
  int hints = fused_hints(cov, d);
  unsigned* task_ctr = ws.task_ctr;
  double* task_sums = ws.task_sums;
  int tc = 0;
  int64_t dyn = dyn_chunks(n, grid, &tc);
  if (tc < kDynMinTC) tc = kDynMinTC;
  unsigned long long* arrivals = ws.arrivals;
  void* args[] = {&out, (void*)&in, &n, &L, &partials, &sum_out, &sum_out_f64, &hints,
                  &post, (void*)&mailbox, &task_ctr, &task_sums, &dyn, &tc, &arrivals};
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(BK_THREADS), args, BK_SMEM, st);
}

}  // namespace lnorm
