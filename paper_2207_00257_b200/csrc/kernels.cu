// kernels.cu — libnorm's sm_100a kernels for Fig. 1 `normalize` after parallel LICM
// (the hoisted `sum` of PAPER.md:117/226-230 becomes a global
// reduction, the kernel body `out[tid] = in[tid] / val` the scale).
//
// The path is HBM-bound (0.25-1 flop/B), so there is no tensor-core work: the
// kernels are persistent grids of 256-bit vector loads (LDG.E.256) with several
// loads in flight per thread, fp32-pairwise-then-fp64 accumulation, fixed-order
// combines (bitwise deterministic), and PDL between the reduce and the scale.
// DESIGN.md §4 gives each kernel's roofline and algorithmic bytes.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include "device_common.cuh"
#include "norm_internal.h"

namespace lnorm {

// ------------------------------------------------------------------ tuning
constexpr int RED_THREADS = 512, RED_UNROLL = 4, RED_CTAS_PER_SM = 2;
constexpr int SC_THREADS = 256, SC_UNROLL = 4, SC_CTAS_PER_SM = 4;
constexpr int SMALL_THREADS = 1024;
constexpr int ROW_THREADS = 256, ROW_MAXV = 4, ROW_CTAS_PER_SM = 4;
constexpr int FU_SCALE_UNROLL = 8;  // fused phase 2 reads from L2: 256 B in flight per thread

enum LoadKind { LD_STREAM = 0, LD_HINT = 1, LD_PLAIN = 2 };

template <int K>
__device__ __forceinline__ f8 load8(const float* p, uint64_t pol) {
  if constexpr (K == LD_STREAM) return ld8_stream(p);
  else if constexpr (K == LD_HINT) return ld8_policy(p, pol);
  else return ld8(p);
}

// acc += sum of p[0, len), split over CTAs [cta, ncta) of the grid.  32-byte
// aligned body as 8-float vectors in chunks of THREADS*UNROLL vectors (UNROLL
// independent 256-bit loads in flight per thread); the < 8-element unaligned
// head and < 8-element tail go to CTA 0.  The partition is a pure function of
// (len, address mod 32, ncta), hence deterministic.
template <int THREADS, int UNROLL, int K>
__device__ __forceinline__ void accumulate_segment(const float* __restrict__ p, int64_t len,
                                                   int cta, int ncta, double& acc, uint64_t pol) {
  if (len <= 0) return;
  const unsigned mis = (unsigned)(reinterpret_cast<uintptr_t>(p) & 31u);
  int64_t head = (int64_t)(((32u - mis) & 31u) >> 2);
  if (head > len) head = len;
  const float* body = p + head;
  const int64_t nv = (len - head) >> 3;
  constexpr int64_t CH = (int64_t)THREADS * UNROLL;
  const int64_t nfull = nv / CH;
  for (int64_t c = cta; c < nfull; c += ncta) {
    const float* q = body + (c * CH + threadIdx.x) * 8;
    f8 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = load8<K>(q + (int64_t)u * THREADS * 8, pol);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += sum8(v[u]);
  }
  for (int64_t vi = nfull * CH + (int64_t)cta * THREADS + threadIdx.x; vi < nv;
       vi += (int64_t)ncta * THREADS)
    acc += sum8(load8<K>(body + vi * 8, pol));
  if (cta == 0) {
    if ((int64_t)threadIdx.x < head) acc += (double)p[threadIdx.x];
    const int64_t t = head + nv * 8 + threadIdx.x;
    if (threadIdx.x < 8 && t < len) acc += (double)p[t];
  }
}

// out[i] = in[i] / s for i in [0, len), split over CTAs; vectorised when out and
// in are co-aligned mod 32 B (VEC), scalar otherwise.
template <int THREADS, int UNROLL, bool VEC, bool ALIAS>
__device__ __forceinline__ void scale_segment(float* out, const float* in, int64_t len, float s,
                                              int cta, int ncta) {
  if (len <= 0) return;
  const Divisor dv = make_divisor(s);
  if constexpr (VEC) {
    const unsigned mis = (unsigned)(reinterpret_cast<uintptr_t>(out) & 31u);
    int64_t head = (int64_t)(((32u - mis) & 31u) >> 2);
    if (head > len) head = len;
    const int64_t nv = (len - head) >> 3;
    const float* ib = in + head;
    float* ob = out + head;
    constexpr int64_t CH = (int64_t)THREADS * UNROLL;
    const int64_t nfull = nv / CH;
    for (int64_t c = cta; c < nfull; c += ncta) {
      const int64_t off = (c * CH + threadIdx.x) * 8;
      f8 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        v[u] = ALIAS ? ld8(ib + off + (int64_t)u * THREADS * 8)
                     : ld8_stream(ib + off + (int64_t)u * THREADS * 8);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) st8_stream(ob + off + (int64_t)u * THREADS * 8, div8(v[u], dv));
    }
    for (int64_t vi = nfull * CH + (int64_t)cta * THREADS + threadIdx.x; vi < nv;
         vi += (int64_t)ncta * THREADS) {
      f8 v = ALIAS ? ld8(ib + vi * 8) : ld8_stream(ib + vi * 8);
      st8_stream(ob + vi * 8, div8(v, dv));
    }
    if (cta == 0) {
      if ((int64_t)threadIdx.x < head) out[threadIdx.x] = div_rn(in[threadIdx.x], dv);
      const int64_t t = head + nv * 8 + threadIdx.x;
      if (threadIdx.x < 8 && t < len) out[t] = div_rn(in[t], dv);
    }
  } else {
    const int64_t stride = (int64_t)ncta * THREADS;
    for (int64_t i = (int64_t)cta * THREADS + threadIdx.x; i < len; i += stride)
      out[i] = div_rn(in[i], dv);
  }
}

// Fused exchange: the rank's partial goes straight from the reduce's last CTA into
// slot [epoch & 1][rank] of every rank's mailbox (peer stores through NVLink),
// then one system-scope fence and the epoch flags (release).  Parity double
// buffering makes a fast rank's next epoch unable to overwrite a slot that a slow
// rank has not read yet (the next epoch's reduce needs this epoch's scale done).
__device__ __forceinline__ void publish_partial(const PeerPost& post, double S) {
  if (!post.mail) return;
  const size_t slot = ((size_t)(post.epoch & 1) * post.world + post.rank) * 2;
  for (int r = 0; r < post.world; ++r) st_relaxed_sys_f64(post.mail[r] + slot, S);
  __threadfence_system();
  for (int r = 0; r < post.world; ++r)
    st_release_sys_u64(reinterpret_cast<unsigned long long*>(post.mail[r] + slot + 1), post.epoch);
}

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
    publish_partial(post, S);
  }
}

// ---- TMA-bulk streaming sum (cp.async.bulk + mbarrier ring) ----------------
// One CTA per SM; warp 0 (one elected lane) streams 32 KiB chunks of a segment's
// 16-byte-aligned body into a 4-stage shared-memory ring (128 KiB in flight per
// SM: the measured sweet spot of scripts/microbench_reduce.cu, 7.56 TB/s vs
// 7.29 TB/s for the best LDG.E.256 geometry; deeper rings lose); 8 consumer
// warps sum each landed chunk from shared memory in a fixed per-thread order and
// release the stage.  Chunks are dealt grid-strided; the < 32 KiB remainder and
// the < 16 B head of each segment go through plain loads.  The ring state
// carries across segments, so a kernel can stream several segments in a row.
constexpr int BK_CONSUMERS = 256, BK_THREADS = BK_CONSUMERS + 32;
constexpr int BK_STAGES = 4, BK_CHUNK = 32768;  // reduce: 4 x 32 KiB in flight per SM
constexpr int SB_STAGES = 2, SB_CHUNK = 49152;  // scale: 2 x 48 KiB (loads share HBM with stores)
constexpr size_t BK_SMEM = (size_t)BK_STAGES * BK_CHUNK;
// The scale ring uses 96 KiB but reserves 116 KiB (> half of the SM's 228 KiB):
// exactly one scale CTA fits per SM, so its persistent grid spreads one CTA per
// SM even when PDL launches it while reduce CTAs are still resident (without
// the reservation two scale CTAs can land on one SM: measured 0.5 ms slower on
// dense 2^32).
constexpr size_t SB_SMEM = 116 * 1024;
static_assert((size_t)SB_STAGES * SB_CHUNK <= SB_SMEM, "ring fits the reservation");
constexpr int64_t kBulkMinN = 1 << 22;  // below this the LDG kernels are as fast

template <int STAGES, int CHUNK>
struct BulkRing {
  static constexpr int64_t CF = CHUNK / 4;  // floats per stage
  unsigned char* buf;
  uint64_t* full;
  uint64_t* empty;
  int stage;
  unsigned phase;
  int issued;
  __device__ __forceinline__ void advance() {
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
};

// head = floats before the first 32-byte boundary of p; then whole chunks.
template <int64_t CF>
__device__ __forceinline__ void bulk_split(const float* p, int64_t len, int64_t* head, int64_t* nchunks) {
  const unsigned mis = (unsigned)(reinterpret_cast<uintptr_t>(p) & 31u);
  int64_t h = (int64_t)(((32u - mis) & 31u) >> 2);
  if (h > len) h = len;
  *head = h;
  *nchunks = (len - h) / CF;
}

// Producer side (call from one lane): issue this CTA's chunks of [p, p + len).
template <bool HINT, int STAGES, int CHUNK>
__device__ __forceinline__ void bulk_produce(BulkRing<STAGES, CHUNK>& r, const float* p, int64_t len,
                                             uint64_t pol) {
  if (len <= 0) return;
  constexpr int64_t CF = BulkRing<STAGES, CHUNK>::CF;
  int64_t head, nchunks;
  bulk_split<CF>(p, len, &head, &nchunks);
  const float* body = p + head;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    if (r.issued >= STAGES) stage_acquire(&r.empty[r.stage], r.phase ^ 1);
    mbar_arrive_expect_tx(&r.full[r.stage], CHUNK);
    void* dst = r.buf + (size_t)r.stage * CHUNK;
    if (HINT) bulk_g2s_hint(dst, body + c * CF, CHUNK, &r.full[r.stage], pol);
    else bulk_g2s(dst, body + c * CF, CHUNK, &r.full[r.stage]);
    ++r.issued;
    r.advance();
  }
}

// Consumer side (warps 1..8, ct = consumer thread index): acc += this CTA's share.
template <int STAGES, int CHUNK>
__device__ __forceinline__ void bulk_consume(BulkRing<STAGES, CHUNK>& r, const float* p, int64_t len,
                                             double& acc, int ct) {
  if (len <= 0) return;
  constexpr int64_t CF = BulkRing<STAGES, CHUNK>::CF;
  static_assert(CHUNK % (32 * BK_CONSUMERS) == 0, "whole 8-float groups per consumer");
  int64_t head, nchunks;
  bulk_split<CF>(p, len, &head, &nchunks);
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    mbar_wait(&r.full[r.stage], r.phase);
    const float4* q = reinterpret_cast<const float4*>(r.buf + (size_t)r.stage * CHUNK);
#pragma unroll
    for (int k = 0; k < CHUNK / 32 / BK_CONSUMERS; ++k) {
      const int i = k * BK_CONSUMERS + ct;  // 8-float group i of the chunk
      const float4 a = q[2 * i], b = q[2 * i + 1];
      f8 v = {{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}};
      acc += sum8(v);
    }
    stage_release(&r.empty[r.stage]);
    r.advance();
  }
  const int64_t rbeg = head + nchunks * CF;  // remainder, then the head: plain loads
  for (int64_t i = rbeg + (int64_t)blockIdx.x * BK_CONSUMERS + ct; i < len;
       i += (int64_t)gridDim.x * BK_CONSUMERS)
    acc += (double)p[i];
  if (blockIdx.x == 0 && ct < head) acc += (double)p[ct];
}

template <int STAGES, int CHUNK>
__device__ __forceinline__ BulkRing<STAGES, CHUNK> bulk_ring_init(unsigned char* buf, uint64_t* full,
                                                                  uint64_t* empty) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], BK_CONSUMERS / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();
  return BulkRing<STAGES, CHUNK>{buf, full, empty, 0, 0u, 0};
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
    publish_partial(post, S);
  }
}

__device__ __forceinline__ float combine_parts(const double* S_parts, int nparts, double* S_full,
                                              unsigned long long epoch = 0) {
  double S;
  if (epoch == 0) {
    S = __ldcg(S_parts);
    for (int r = 1; r < nparts; ++r) S += __ldcg(S_parts + r);  // fixed (rank / chunk) order
  } else {
    // mailbox: wait for every rank's slot of this epoch (peer stores over NVLink)
    const double* box = S_parts + (size_t)(epoch & 1) * nparts * 2;
    const unsigned long long t0 = globaltimer_ns();
    bool ok = true;
    for (int r = 0; r < nparts && ok; ++r) {
      const unsigned long long* flag = reinterpret_cast<const unsigned long long*>(box + 2 * r + 1);
      while (ld_acquire_sys_u64(flag) != epoch) {
        if (globaltimer_ns() - t0 > 30000000000ull) { ok = false; break; }  // peer lost: no hang
        __nanosleep(64);
      }
    }
    if (!ok) {
      S = __longlong_as_double(0x7ff8000000000000ll);
    } else {
      S = ld_relaxed_sys_f64(box);
      for (int r = 1; r < nparts; ++r) S += ld_relaxed_sys_f64(box + 2 * r);  // rank order
    }
  }
  *S_full = S;
  return (float)S;  // RN to binary32
}

// ---------------------------------------------------------------- scale
template <bool VEC, bool ALIAS>
__global__ void __launch_bounds__(SC_THREADS)
    scale_kernel(float* out, const float* in, int64_t len, const double* __restrict__ S_parts,
                 int nparts, float* sum_out, double* sum_out_f64, unsigned long long epoch) {
  __shared__ float s_sh;
  pdl_wait();  // S_parts are complete and visible; `in` is no longer being read
  if (threadIdx.x == 0) {
    double S;
    const float s = combine_parts(S_parts, nparts, &S, epoch);
    s_sh = s;
    if (blockIdx.x == 0) {
      if (sum_out) *sum_out = s;
      if (sum_out_f64) *sum_out_f64 = S;
    }
  }
  __syncthreads();
  scale_segment<SC_THREADS, SC_UNROLL, VEC, ALIAS>(out, in, len, s_sh, blockIdx.x, gridDim.x);
}

// Scale, TMA-bulk variant for len >= 2^22 with out/in co-aligned mod 32 B: one
// CTA per SM, 2 x 48 KiB chunks of `in` in flight per SM via cp.async.bulk
// (the measured optimum for a read+write stream: 6.76 TB/s vs 6.12 TB/s for
// LDG/STG and 6.57 TB/s for cudaMemcpy D2D, scripts/microbench_scale.cu);
// consumers divide out of shared memory and store with STG.E.256 (.cs).  The
// producer starts streaming BEFORE griddepcontrol.wait — `in` is not written by
// the preceding reduce — so under PDL the first chunks overlap the reduce's
// tail; no store happens before the wait (out may alias in).
__global__ void __launch_bounds__(BK_THREADS, 1)
    scale_bulk_kernel(float* out, const float* in, int64_t len, const double* __restrict__ S_parts,
                      int nparts, float* sum_out, double* sum_out_f64, unsigned long long epoch) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[SB_STAGES], empty[SB_STAGES];
  __shared__ float s_sh;
  auto r = bulk_ring_init<SB_STAGES, SB_CHUNK>(ring, full, empty);
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) bulk_produce<false>(r, in, len, 0);
    return;
  }
  const int ct = threadIdx.x - 32;
  pdl_wait();
  if (ct == 0) {
    double S;
    const float s = combine_parts(S_parts, nparts, &S, epoch);
    s_sh = s;
    if (blockIdx.x == 0) {
      if (sum_out) *sum_out = s;
      if (sum_out_f64) *sum_out_f64 = S;
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(BK_CONSUMERS) : "memory");  // consumers only
  const float s = s_sh;
  const Divisor dv = make_divisor(s);
  constexpr int64_t CF = SB_CHUNK / 4;
  int64_t head, nchunks;
  bulk_split<CF>(in, len, &head, &nchunks);
  float* ob = out + head;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    mbar_wait(&r.full[r.stage], r.phase);
    const float4* q = reinterpret_cast<const float4*>(r.buf + (size_t)r.stage * SB_CHUNK);
    float* oc = ob + c * CF;
#pragma unroll
    for (int k = 0; k < SB_CHUNK / 32 / BK_CONSUMERS; ++k) {
      const int i = k * BK_CONSUMERS + ct;
      const float4 a = q[2 * i], b = q[2 * i + 1];
#if defined(NORM_AB_SCALE_DIV8)  // A/B experiments only
      st8_stream(oc + (int64_t)i * 8, div8(f8{{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}}, dv));
#else
      st8_stream(oc + (int64_t)i * 8, div8_fchk(f8{{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}}, dv));
#endif
    }
    stage_release(&r.empty[r.stage]);
    r.advance();
  }
  const int64_t rbeg = head + nchunks * CF;  // remainder, then the head
  for (int64_t i = rbeg + (int64_t)blockIdx.x * BK_CONSUMERS + ct; i < len;
       i += (int64_t)gridDim.x * BK_CONSUMERS)
    out[i] = div_rn(in[i], dv);
  if (blockIdx.x == 0 && ct < head) out[ct] = div_rn(in[ct], dv);
}

__global__ void __launch_bounds__(256)
    scale_residue_kernel(float* out, const float* in, int64_t len, int64_t gbegin, int64_t G,
                         const double* __restrict__ S_parts, int nparts, float* sum_out,
                         double* sum_out_f64, unsigned long long epoch) {
  __shared__ float s_sh;
  pdl_wait();
  if (threadIdx.x == 0) {
    double S;
    const float s = combine_parts(S_parts, nparts, &S, epoch);
    s_sh = s;
    if (blockIdx.x == 0) {
      if (sum_out) *sum_out = s;
      if (sum_out_f64) *sum_out_f64 = S;
    }
  }
  __syncthreads();
  const float s = s_sh;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < len;
       j += (int64_t)gridDim.x * blockDim.x)
    if ((gbegin + j) % 32 < G) out[j] = div_rn(in[j], s);  // tid = b + 32 t, b < G
}

// ---------------------------------------------------------------- small
// One CTA does the whole call: no workspace, one launch (latency-bound sizes).
__global__ void __launch_bounds__(SMALL_THREADS)
    small_kernel(float* out, const float* in, int64_t n, int kind, int64_t L, int64_t G,
                 float* sum_out, double* sum_out_f64) {
  __shared__ double red[SMALL_THREADS / 32];
  double acc = 0.0;
  accumulate_segment<SMALL_THREADS, 1, LD_PLAIN>(in, n, 0, 1, acc, 0);
  const double S = block_sum(acc, red);  // barrier: every load precedes every store
  const float s = (float)S;
  if (threadIdx.x == 0) {
    if (sum_out) *sum_out = s;
    if (sum_out_f64) *sum_out_f64 = S;
  }
  if (kind == COV_PREFIX) {
    for (int64_t i = threadIdx.x; i < L; i += SMALL_THREADS) out[i] = div_rn(in[i], s);
  } else if (kind == COV_RESIDUE) {
    for (int64_t i = threadIdx.x; i < n; i += SMALL_THREADS)
      if (i % 32 < G) out[i] = div_rn(in[i], s);
  }
}

// ---------------------------------------------------------------- fused
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire_u32(bar + 1);
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire_u32(bar + 1) == gen) __nanosleep(40);
    }
    __threadfence();
  }
  __syncthreads();
}

// Single pass over HBM when the covered prefix fits in L2: one cooperative CTA
// per SM streams the uncovered tail [L, n) through the TMA-bulk ring with an L2
// evict_first hint, then the covered prefix [0, L) with evict_last (read LAST,
// so it is the most recent data in L2); grid barrier; every CTA combines the
// per-CTA partials in the same fixed order (identical s everywhere); then all
// threads scale the prefix out of L2.  Co-residency by cooperative launch.
template <bool VEC>
__global__ void __launch_bounds__(BK_THREADS, 1)
    fused_kernel(float* out, const float* in, int64_t n, int64_t L, double* partials,
                 unsigned* bar, float* sum_out, double* sum_out_f64) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[BK_STAGES], empty[BK_STAGES];
  __shared__ double red[BK_THREADS / 32];
  auto r = bulk_ring_init<BK_STAGES, BK_CHUNK>(ring, full, empty);
  double acc = 0.0;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      bulk_produce<true>(r, in + L, n - L, policy_evict_first());
      bulk_produce<true>(r, in, L, policy_evict_last());
    }
  } else {
    bulk_consume(r, in + L, n - L, acc, threadIdx.x - 32);
    bulk_consume(r, in, L, acc, threadIdx.x - 32);
  }
  const double b = block_sum(acc, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = b;
  grid_barrier(bar);  // all of `in` has been read: `out` (possibly == in) may be written
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += BK_THREADS) v += __ldcg(partials + i);
  const double S = block_sum(v, red);  // identical bits in every CTA
  const float s = (float)S;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (sum_out) *sum_out = s;
    if (sum_out_f64) *sum_out_f64 = S;
  }
  scale_segment<BK_THREADS, FU_SCALE_UNROLL, VEC, true>(out, in, L, s, blockIdx.x, gridDim.x);
}

// ----------------------------------------------------------------- rows
__device__ __forceinline__ bool row_covered(int64_t i, int64_t L, int64_t G) {
  return L >= 0 ? i < L : (i % 32) < G;
}

// Batched rows, register-resident (row <= ROW_THREADS*8*MAXV floats, 32 B aligned,
// cols % 8 == 0): persistent CTAs walk rows r, r + grid, ...; the NEXT row's
// 256-bit loads are issued before the current row's block reduction, so HBM
// always has a row in flight per CTA (software pipelining across rows).  One
// HBM read and one write (of the covered part) per element.
template <bool ALIAS, int MAXV>
__device__ __forceinline__ void row_load(const float* src, int nvr, f8* v) {
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const int idx = k * ROW_THREADS + threadIdx.x;
    if (idx < nvr) v[k] = ALIAS ? ld8(src + (int64_t)idx * 8) : ld8_stream(src + (int64_t)idx * 8);
  }
}

template <int MAXV>
__device__ __forceinline__ void row_finish(float* dst, int nvr, const f8* v, int64_t r, int64_t L,
                                           int64_t G, double* red, float* sum_out,
                                           double* sum_out_f64) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < MAXV; ++k)
    if (k * ROW_THREADS + (int)threadIdx.x < nvr) acc += sum8(v[k]);
  const double S = block_sum_1b(acc, red);  // caller alternates `red` between rows
  const float s = (float)S;
  const Divisor dv = make_divisor(s);
  if (threadIdx.x == 0) {
    if (sum_out) sum_out[r] = s;
    if (sum_out_f64) sum_out_f64[r] = S;
  }
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const int idx = k * ROW_THREADS + threadIdx.x;
    if (idx >= nvr) continue;
    const int64_t e0 = (int64_t)idx * 8;
    if (L >= 0 && e0 + 8 <= L) {
      st8_stream(dst + e0, div8(v[k], dv));
    } else if (L < 0 || e0 < L) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (row_covered(e0 + j, L, G)) dst[e0 + j] = div_rn(v[k].v[j], dv);
    }
  }
}

__host__ __device__ constexpr int row_ctas_per_sm(int maxv) { return maxv >= 4 ? 2 : ROW_CTAS_PER_SM; }

template <bool ALIAS, int MAXV>
__global__ void __launch_bounds__(ROW_THREADS, row_ctas_per_sm(MAXV))
    rows_vec_kernel(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                    int64_t ld_in, int64_t L, int64_t G, float* sum_out, double* sum_out_f64) {
  __shared__ double red[2][ROW_THREADS / 32];  // alternated by row: one barrier per row
  const int nvr = (int)(cols >> 3);
  const int64_t step = gridDim.x;
  f8 a[MAXV], b[MAXV];
  int64_t r = blockIdx.x;
  if (r < rows) row_load<ALIAS, MAXV>(in + r * ld_in, nvr, a);
  while (r < rows) {
    int64_t rn = r + step;
    if (rn < rows) row_load<ALIAS, MAXV>(in + rn * ld_in, nvr, b);
    row_finish<MAXV>(out + r * ld_out, nvr, a, r, L, G, red[0], sum_out, sum_out_f64);
    r = rn;
    if (r >= rows) break;
    rn = r + step;
    if (rn < rows) row_load<ALIAS, MAXV>(in + rn * ld_in, nvr, a);
    row_finish<MAXV>(out + r * ld_out, nvr, b, r, L, G, red[1], sum_out, sum_out_f64);
    r = rn;
  }
}

// Batched rows, TMA-staged, one WARP per row (rows of <= 48 KiB, 16-byte aligned
// with cols % 4 == 0).  One CTA per SM: lane 0 of warp 0 streams whole rows
// into a ring of S = 2W shared-memory stages with cp.async.bulk; consumer warp w
// owns stages w and w + W and processes this CTA's rows k = w, w + W, ...: sum
// the row out of shared memory, warp-shuffle reduce (no block barrier on the
// per-row critical path), then scale the covered elements out of shared memory
// into `out`.  Up to S rows are in flight per SM, so HBM stays busy while each
// warp finishes its row.
constexpr int RB_MAX_STAGES = 16;
constexpr size_t RB_SMEM_BUDGET = 200 * 1024;

__global__ void __launch_bounds__(32 * (1 + RB_MAX_STAGES / 2), 1)
    rows_bulk_kernel(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                     int64_t ld_in, int64_t L, int64_t G, int S, float* sum_out,
                     double* sum_out_f64) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[RB_MAX_STAGES], empty[RB_MAX_STAGES];
  const int W = S / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned row_bytes = (unsigned)(cols * 4);
  const size_t stage_bytes = ((size_t)row_bytes + 127) & ~(size_t)127;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t step = gridDim.x;
  if (warp == 0) {
    if (lane == 0) {
      int64_t k = 0;
      for (int64_t r = blockIdx.x; r < rows; r += step, ++k) {
        const int st = (int)(k % S);
        if (k >= S) stage_acquire(&empty[st], (unsigned)(((k / S) - 1) & 1));
        mbar_arrive_expect_tx(&full[st], row_bytes);
        bulk_g2s(ring + st * stage_bytes, in + r * ld_in, row_bytes, &full[st]);
      }
    }
    return;
  }
  const int w = warp - 1;
  const int nq = (int)(cols >> 2);  // float4s per row
  const bool vst = ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) && (ld_out % 4 == 0);
  for (int64_t k = w; blockIdx.x + k * step < rows; k += W) {
    const int64_t r = blockIdx.x + k * step;
    const int st = (int)(k % S);
    mbar_wait(&full[st], (unsigned)((k / S) & 1));
    const float4* q = reinterpret_cast<const float4*>(ring + st * stage_bytes);
    double acc = 0.0;
    for (int j = lane; j < nq; j += 32) {
      const float4 a = q[j];
      acc += (double)((a.x + a.y) + (a.z + a.w));
    }
    const double Srow = warp_sum(acc);
    const float s = (float)Srow;
    const Divisor dv = make_divisor(s);
    if (lane == 0) {
      if (sum_out) sum_out[r] = s;
      if (sum_out_f64) sum_out_f64[r] = Srow;
    }
    float* dst = out + r * ld_out;
    const float* src = reinterpret_cast<const float*>(q);
    if (L >= 0) {
      const int full4 = (int)(L >> 2);
      for (int j = lane; j < full4; j += 32) {
        const float4 a = q[j];
        const float4 y = make_float4(div_rn_fchk(a.x, dv), div_rn_fchk(a.y, dv), div_rn_fchk(a.z, dv),
                                     div_rn_fchk(a.w, dv));
        if (vst) __stcs(reinterpret_cast<float4*>(dst) + j, y);
        else { dst[4 * j] = y.x; dst[4 * j + 1] = y.y; dst[4 * j + 2] = y.z; dst[4 * j + 3] = y.w; }
      }
      const int64_t t = (int64_t)full4 * 4 + lane;
      if (lane < 4 && t < L) dst[t] = div_rn_fchk(src[t], dv);
    } else {
      for (int64_t i = lane; i < cols; i += 32)
        if ((i % 32) < G) dst[i] = div_rn_fchk(src[i], dv);
    }
    stage_release(&empty[st]);
  }
}

// Any shape / alignment: one CTA per row, a scalar sum sweep then a scale sweep.
__global__ void __launch_bounds__(ROW_THREADS)
    rows_generic_kernel(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                        int64_t ld_in, int64_t L, int64_t G, float* sum_out, double* sum_out_f64) {
  __shared__ double red[ROW_THREADS / 32];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const float* src = in + r * ld_in;
    float* dst = out + r * ld_out;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < cols; i += ROW_THREADS) acc += (double)src[i];
    const double S = block_sum(acc, red);  // barrier: the row's loads precede its stores
    const float s = (float)S;
    if (threadIdx.x == 0) {
      if (sum_out) sum_out[r] = s;
      if (sum_out_f64) sum_out_f64[r] = S;
    }
    for (int64_t i = threadIdx.x; i < cols; i += ROW_THREADS)
      if (row_covered(i, L, G)) dst[i] = div_rn(src[i], s);
  }
}

// ============================================================ launchers

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
    reduce_bulk_kernel<<<d.sms, BK_THREADS, smem, st>>>(in, n, ws.partials, ws.ticket, S_out,
                                                        pdl_mode() == PDL_EARLY, post);
    return cudaGetLastError();
  }
  reduce_kernel<<<reduce_grid(d, n), RED_THREADS, 0, st>>>(in, n, ws.partials, ws.ticket, S_out,
                                                            pdl_mode() == PDL_EARLY, post);
  return cudaGetLastError();
}

template <typename Kern, typename... Args>
static cudaError_t launch_maybe_pdl_smem(Kern k, int grid, int block, size_t smem, bool pdl,
                                         cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && pdl_mode() != PDL_OFF) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

template <typename Kern, typename... Args>
static cudaError_t launch_maybe_pdl(Kern k, int grid, int block, bool pdl, cudaStream_t st,
                                    Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && pdl_mode() != PDL_OFF) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

cudaError_t launch_scale(float* out, const float* in, int64_t len, const double* S_parts,
                         int nparts, float* sum_out, double* sum_out_f64, const DeviceInfo& d,
                         bool pdl, cudaStream_t st, unsigned long long epoch) {
  const int64_t per_chunk = (int64_t)SC_THREADS * SC_UNROLL * 8;
  int64_t g = (len + per_chunk - 1) / per_chunk;
  const int64_t gmax = (int64_t)d.sms * SC_CTAS_PER_SM;
  if (g > gmax) g = gmax;
  if (g < 1) g = 1;
  const bool vec = ((reinterpret_cast<uintptr_t>(out) - reinterpret_cast<uintptr_t>(in)) & 31u) == 0;
  const bool alias = out == in;
  if (vec && len >= kBulkMinN) {
    static int configured[64] = {0};
    if (d.device < 64 && !configured[d.device]) {
      cudaError_t e = cudaFuncSetAttribute(scale_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)SB_SMEM);
      if (e != cudaSuccess) return e;
      configured[d.device] = 1;
    }
    return launch_maybe_pdl_smem(scale_bulk_kernel, d.sms, BK_THREADS, SB_SMEM, pdl, st, out, in,
                                 len, S_parts, nparts, sum_out, sum_out_f64, epoch);
  }
  if (vec && alias)
    return launch_maybe_pdl(scale_kernel<true, true>, (int)g, SC_THREADS, pdl, st, out, in, len,
                            S_parts, nparts, sum_out, sum_out_f64, epoch);
  if (vec)
    return launch_maybe_pdl(scale_kernel<true, false>, (int)g, SC_THREADS, pdl, st, out, in, len,
                            S_parts, nparts, sum_out, sum_out_f64, epoch);
  return launch_maybe_pdl(scale_kernel<false, false>, (int)g, SC_THREADS, pdl, st, out, in, len,
                          S_parts, nparts, sum_out, sum_out_f64, epoch);
}

cudaError_t launch_scale_residue(float* out, const float* in, int64_t len, int64_t gbegin,
                                 int64_t G, const double* S_parts, int nparts, float* sum_out,
                                 double* sum_out_f64, bool pdl, cudaStream_t st,
                                 unsigned long long epoch) {
  int64_t g = (len + 255) / 256;
  if (g < 1) g = 1;
  if (g > 1024) g = 1024;
  return launch_maybe_pdl(scale_residue_kernel, (int)g, 256, pdl, st, out, in, len, gbegin, G,
                          S_parts, nparts, sum_out, sum_out_f64, epoch);
}

cudaError_t launch_small(float* out, const float* in, const Coverage& cov, float* sum_out,
                         double* sum_out_f64, cudaStream_t st) {
  small_kernel<<<1, SMALL_THREADS, 0, st>>>(out, in, cov.n, cov.kind, cov.L, cov.G, sum_out,
                                            sum_out_f64);
  return cudaGetLastError();
}

cudaError_t launch_fused(float* out, const float* in, const Coverage& cov, const Workspace& ws,
                         float* sum_out, double* sum_out_f64, const DeviceInfo& d,
                         cudaStream_t st) {
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
  unsigned* bar = ws.bar;
  void* args[] = {&out, (void*)&in, &n, &L, &partials, &bar, &sum_out, &sum_out_f64};
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(BK_THREADS), args, BK_SMEM, st);
}

cudaError_t launch_rows(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                        int64_t ld_in, const Coverage& rc, float* sum_out, double* sum_out_f64,
                        const DeviceInfo& d, cudaStream_t st) {
  const int maxv = cols <= ROW_THREADS * 8 ? 1 : (cols <= ROW_THREADS * 16 ? 2 : 4);
  int64_t g = (int64_t)d.sms * row_ctas_per_sm(maxv);  // persistent: one wave
  if (rows < g) g = rows;
  const int64_t L = rc.kind == COV_PREFIX ? rc.L : -1;
  const bool aligned = ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(in)) & 31u) == 0 &&
                       (ld_out % 8) == 0 && (ld_in % 8) == 0 && (cols % 8) == 0;
  const bool vec = aligned && cols <= (int64_t)ROW_THREADS * 8 * ROW_MAXV;
  const bool alias = out == in;
  // The warp-per-row TMA kernel wins when few elements are written (literal rows:
  // 6.1 vs 5.4 TB/s at 65536x4096); with every element written the per-warp
  // division/store work needs more warps than it has, and the register-resident
  // CTA-per-row kernel wins (5.9 vs 4.5 TB/s, dense) -- DESIGN.md §4.
  const int64_t covered = rc.kind == COV_PREFIX ? rc.L : rc.count;
  const bool bulk_ok = ((reinterpret_cast<uintptr_t>(in) & 15u) == 0) && (ld_in % 4) == 0 &&
                       (cols % 4) == 0 && cols * 4 <= 48 * 1024 && cols >= 256 &&
                       covered * 2 <= cols;
  if (bulk_ok && !getenv("NORM_ROWS_NO_BULK")) {
    const size_t stage_bytes = ((size_t)cols * 4 + 127) & ~(size_t)127;
    int S = (int)(RB_SMEM_BUDGET / stage_bytes);
    if (S > RB_MAX_STAGES) S = RB_MAX_STAGES;
    S &= ~1;
    if (S >= 2) {
      static int configured[64] = {0};
      if (d.device < 64 && !configured[d.device]) {
        cudaError_t e = cudaFuncSetAttribute(rows_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)RB_SMEM_BUDGET);
        if (e != cudaSuccess) return e;
        configured[d.device] = 1;
      }
      int64_t gb = d.sms;
      if (rows < gb) gb = rows;
      rows_bulk_kernel<<<(int)gb, 32 * (1 + S / 2), (size_t)S * stage_bytes, st>>>(
          out, in, rows, cols, ld_out, ld_in, L, rc.G, S, sum_out, sum_out_f64);
      return cudaGetLastError();
    }
  }
#define NORM_ROWS(A, M)                                                                           \
  rows_vec_kernel<A, M><<<(int)g, ROW_THREADS, 0, st>>>(out, in, rows, cols, ld_out, ld_in, L, rc.G, \
                                                       sum_out, sum_out_f64)
  if (!vec)
    rows_generic_kernel<<<(int)g, ROW_THREADS, 0, st>>>(out, in, rows, cols, ld_out, ld_in, L, rc.G,
                                                        sum_out, sum_out_f64);
  else if (alias && maxv == 1) NORM_ROWS(true, 1);
  else if (alias && maxv == 2) NORM_ROWS(true, 2);
  else if (alias) NORM_ROWS(true, 4);
  else if (maxv == 1) NORM_ROWS(false, 1);
  else if (maxv == 2) NORM_ROWS(false, 2);
  else NORM_ROWS(false, 4);
#undef NORM_ROWS
  return cudaGetLastError();
}

}  // namespace lnorm
