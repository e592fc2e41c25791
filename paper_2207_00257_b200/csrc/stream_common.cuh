// stream_common.cuh — pieces shared by libnorm's streaming kernels (reduce.cu,
// scale.cu, fused.cu, rows.cu): tuning constants, the LDG.E.256 segment loops,
// the TMA-bulk (cp.async.bulk + mbarrier) ring, and the PDL launch helpers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

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
#ifndef NORM_SB_STAGES  // probe builds may override (scripts/ab_libs.py)
#define NORM_SB_STAGES 2
#define NORM_SB_CHUNK 49152
#endif
constexpr int SB_STAGES = NORM_SB_STAGES, SB_CHUNK = NORM_SB_CHUNK;  // scale: 2 x 48 KiB (loads share HBM with stores)
constexpr size_t BK_SMEM = (size_t)BK_STAGES * BK_CHUNK;
// The scale ring uses 96 KiB but reserves 116 KiB (> half of the SM's 228 KiB):
// exactly one scale CTA fits per SM, so its persistent grid spreads one CTA per
// SM even when PDL launches it while reduce CTAs are still resident (without
// the reservation two scale CTAs can land on one SM: measured 0.5 ms slower on
// dense 2^32).
constexpr size_t SB_SMEM = (size_t)SB_STAGES * SB_CHUNK > 116 * 1024 ? (size_t)SB_STAGES * SB_CHUNK : 116 * 1024;
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

// Producer cursor over this CTA's chunks of a segment [p, p + len): chunk c of
// the 32-byte-aligned body, c = blockIdx.x, blockIdx.x + gridDim.x, ...  Lets a
// kernel issue part of a segment (e.g. prefetch the first stages of a later
// phase) and resume it later; bulk_produce issues it all.
struct BulkCursor {
  const float* body;
  int64_t c, nchunks;
};

template <int64_t CF>
__device__ __forceinline__ BulkCursor bulk_cursor(const float* p, int64_t len) {
  if (len <= 0) return BulkCursor{p, 0, 0};
  int64_t head, nchunks;
  bulk_split<CF>(p, len, &head, &nchunks);
  return BulkCursor{p + head, (int64_t)blockIdx.x, nchunks};
}

// Issue up to max_issue of the cursor's remaining chunks (call from one lane).
template <bool HINT, int STAGES, int CHUNK>
__device__ __forceinline__ void bulk_issue(BulkRing<STAGES, CHUNK>& r, BulkCursor& cur, int64_t max_issue,
                                           uint64_t pol) {
  constexpr int64_t CF = BulkRing<STAGES, CHUNK>::CF;
  for (int64_t k = 0; k < max_issue && cur.c < cur.nchunks; ++k, cur.c += gridDim.x) {
    if (r.issued >= STAGES) stage_acquire(&r.empty[r.stage], r.phase ^ 1);
    mbar_arrive_expect_tx(&r.full[r.stage], CHUNK);
    void* dst = r.buf + (size_t)r.stage * CHUNK;
    if (HINT) bulk_g2s_hint(dst, cur.body + cur.c * CF, CHUNK, &r.full[r.stage], pol);
    else bulk_g2s(dst, cur.body + cur.c * CF, CHUNK, &r.full[r.stage]);
    ++r.issued;
    r.advance();
  }
}

// Producer side (call from one lane): issue this CTA's chunks of [p, p + len).
template <bool HINT, int STAGES, int CHUNK>
__device__ __forceinline__ void bulk_produce(BulkRing<STAGES, CHUNK>& r, const float* p, int64_t len,
                                             uint64_t pol) {
  BulkCursor cur = bulk_cursor<BulkRing<STAGES, CHUNK>::CF>(p, len);
  bulk_issue<HINT>(r, cur, INT64_MAX, pol);
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

// Consumer side of a scale stream (warps 1..8): out[i] = in[i] / s for this CTA's
// chunks of [in, in + len), read from the ring, stored with STG.E.256 (.cs);
// out must be co-aligned with in mod 32 B.  The remainder and the head go through
// plain loads, each element read and written by the same thread (so out may
// alias in: every chunk is loaded into shared memory before this CTA, its only
// writer, stores over it).
template <int STAGES, int CHUNK>
__device__ __forceinline__ void bulk_scale_consume(BulkRing<STAGES, CHUNK>& r, float* out, const float* in,
                                                   int64_t len, const Divisor& dv, int ct) {
  if (len <= 0) return;
  constexpr int64_t CF = CHUNK / 4;
  static_assert(CHUNK % (32 * BK_CONSUMERS) == 0, "whole 8-float groups per consumer");
  int64_t head, nchunks;
  bulk_split<CF>(in, len, &head, &nchunks);
  float* ob = out + head;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    mbar_wait(&r.full[r.stage], r.phase);
    const float4* q = reinterpret_cast<const float4*>(r.buf + (size_t)r.stage * CHUNK);
    float* oc = ob + c * CF;
#pragma unroll
    for (int k = 0; k < CHUNK / 32 / BK_CONSUMERS; ++k) {
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

// ---- dynamically scheduled, deterministic streaming sum ----------------------
// The hoisted `sum` over up to NSEG segments (streamed in segment order, each
// with its own L2 policy) through the BK ring.  Chunk u of the concatenated
// chunk space: the first `ns` are dealt grid-strided (they feed this CTA's
// partial `acc`), the last `dyn` form tasks of `tc` consecutive chunks that CTAs
// claim from *task_ctr as they run dry (claimed one ahead, so the atomic's round
// trip overlaps the loads).  A task's sum does not depend on which CTA runs it:
// each consumer thread adds its 8-float groups of the task's chunks in chunk
// order, a warp butterfly combines the lanes, and whichever warp finishes the
// task last adds the 8 warp sums in warp order into task_sums[t].  tc >=
// BK_STAGES bounds how far warps drift apart (at most one task), so two task
// slots suffice.  Why: per-SM streaming rates differ by 1-2 % at random, and
// with every chunk dealt statically the last CTA finished ~20-40 us after the
// median at n = 2^32 (scripts/reduce_timeline.cu).  The caller combines
// per-CTA partials and task sums in index order, and resets *task_ctr once
// every CTA is done claiming.
constexpr int kDynMinTC = BK_STAGES;

struct DynSeg {
  const float* p;
  int64_t len;
  uint64_t pol;
  int hint;  // 1: cp.async.bulk with the L2 policy `pol`
};

struct DynSmem {  // shared-memory state of dyn_stream_sum
  int64_t stage_chunk[BK_STAGES];
  double slot[2][BK_CONSUMERS / 32];
  unsigned slot_cnt[2];
};

template <int NSEG>
struct DynGeo {
  const float* body[NSEG];
  int64_t head[NSEG], nch[NSEG];
  int64_t total;
  __device__ __forceinline__ DynGeo(const DynSeg* seg) : total(0) {
    constexpr int64_t CF = BK_CHUNK / 4;
#pragma unroll
    for (int i = 0; i < NSEG; ++i) {
      if (seg[i].len > 0) {
        bulk_split<CF>(seg[i].p, seg[i].len, &head[i], &nch[i]);
      } else {
        head[i] = 0;
        nch[i] = 0;
      }
      body[i] = seg[i].p + head[i];
      total += nch[i];
    }
  }
  __device__ __forceinline__ const float* chunk(int64_t u, int* si) const {
    constexpr int64_t CF = BK_CHUNK / 4;
#pragma unroll
    for (int i = 0; i < NSEG - 1; ++i) {
      if (u < nch[i]) {
        *si = i;
        return body[i] + u * CF;
      }
      u -= nch[i];
    }
    *si = NSEG - 1;
    return body[NSEG - 1] + u * CF;
  }
};

template <int NSEG>
__device__ __forceinline__ void dyn_issue(BulkRing<BK_STAGES, BK_CHUNK>& r, const DynGeo<NSEG>& g,
                                          const DynSeg* seg, int64_t u, DynSmem& sm, bool tag) {
  int si;
  const float* src = g.chunk(u, &si);
  if (r.issued >= BK_STAGES) stage_acquire(&r.empty[r.stage], r.phase ^ 1);
  if (tag) sm.stage_chunk[r.stage] = u;
  mbar_arrive_expect_tx(&r.full[r.stage], BK_CHUNK);
  void* dst = r.buf + (size_t)r.stage * BK_CHUNK;
  uint64_t pol = seg[0].pol;  // select without dynamic indexing (keeps seg in registers)
  int hint = seg[0].hint;
#pragma unroll
  for (int i = 1; i < NSEG; ++i)
    if (si == i) {
      pol = seg[i].pol;
      hint = seg[i].hint;
    }
  if (hint) bulk_g2s_hint(dst, src, BK_CHUNK, &r.full[r.stage], pol);
  else bulk_g2s(dst, src, BK_CHUNK, &r.full[r.stage]);
  ++r.issued;
  r.advance();
}

__device__ __forceinline__ double dyn_chunk_sum(const BulkRing<BK_STAGES, BK_CHUNK>& r, int ct) {
  const float4* q = reinterpret_cast<const float4*>(r.buf + (size_t)r.stage * BK_CHUNK);
  double a = 0.0;
#pragma unroll
  for (int k = 0; k < BK_CHUNK / 32 / BK_CONSUMERS; ++k) {
    const int i = k * BK_CONSUMERS + ct;
    const float4 x = q[2 * i], y = q[2 * i + 1];
    a += sum8(f8{{x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w}});
  }
  return a;
}

// Called by every thread of a BK_THREADS CTA (warp 0 lane 0 produces, warps 1..8
// consume); returns this thread's share of the CTA's static partial.  `sm` must
// have slot_cnt zeroed before the ring's init barrier.
template <int NSEG>
__device__ __forceinline__ double dyn_stream_sum(BulkRing<BK_STAGES, BK_CHUNK>& r, const DynSeg* seg,
                                                 int64_t dyn, int tc, unsigned* task_ctr,
                                                 double* task_sums, DynSmem& sm, int64_t* ntasks_out) {
  const DynGeo<NSEG> g(seg);
  if (dyn > g.total) dyn = g.total;
  const int64_t ns = g.total - dyn;
  const int64_t ntasks = (dyn + tc - 1) / tc;
  *ntasks_out = ntasks;
  double acc = 0.0;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      for (int64_t u = blockIdx.x; u < ns; u += gridDim.x) dyn_issue<NSEG>(r, g, seg, u, sm, false);
      int64_t next = ntasks > 0 ? (int64_t)atomicAdd(task_ctr, 1u) : ntasks;
      while (next < ntasks) {
        const int64_t t = next;
        next = (int64_t)atomicAdd(task_ctr, 1u);
        const int64_t u0 = ns + t * tc, u1 = u0 + tc < g.total ? u0 + tc : g.total;
        for (int64_t u = u0; u < u1; ++u) dyn_issue<NSEG>(r, g, seg, u, sm, true);
      }
      if (r.issued >= BK_STAGES) stage_acquire(&r.empty[r.stage], r.phase ^ 1);
      sm.stage_chunk[r.stage] = -1;  // end marker: completes with no bytes
      mbar_arrive(&r.full[r.stage]);
    }
    return 0.0;
  }
  const int ct = threadIdx.x - 32, w = ct >> 5, lane = ct & 31;
  for (int64_t u = blockIdx.x; u < ns; u += gridDim.x) {
    mbar_wait(&r.full[r.stage], r.phase);
    acc += dyn_chunk_sum(r, ct);
    stage_release(&r.empty[r.stage]);
    r.advance();
  }
  double tacc = 0.0;
  unsigned done = 0;  // tasks this warp has finished (the same sequence in every warp)
  for (;;) {
    mbar_wait(&r.full[r.stage], r.phase);
    const int64_t u = *(volatile int64_t*)&sm.stage_chunk[r.stage];
    if (u < 0) break;
    tacc += dyn_chunk_sum(r, ct);
    stage_release(&r.empty[r.stage]);
    r.advance();
    const int64_t d = u - ns;
    if ((d + 1) % tc == 0 || u + 1 == g.total) {  // last chunk of task d / tc
      const double v = warp_sum(tacc);
      tacc = 0.0;
      const unsigned p = done++ & 1u;
      if (lane == 0) {
        sm.slot[p][w] = v;
        __threadfence_block();
        if (atomicAdd(&sm.slot_cnt[p], 1u) == BK_CONSUMERS / 32 - 1) {
          __threadfence_block();
          double t = 0.0;
#pragma unroll
          for (int k = 0; k < BK_CONSUMERS / 32; ++k) t += *(volatile double*)&sm.slot[p][k];
          task_sums[d / tc] = t;
          __threadfence();  // before this CTA's ticket / grid barrier
          sm.slot_cnt[p] = 0u;
        }
      }
    }
  }
  // each segment's remainder (< one chunk) and head: plain loads, static
  constexpr int64_t CF = BK_CHUNK / 4;
#pragma unroll
  for (int i = 0; i < NSEG; ++i) {
    const float* p = seg[i].p;
    const int64_t len = seg[i].len;
    if (len <= 0) continue;
    for (int64_t e = g.head[i] + g.nch[i] * CF + (int64_t)blockIdx.x * BK_CONSUMERS + ct; e < len;
         e += (int64_t)gridDim.x * BK_CONSUMERS)
      acc += (double)p[e];
    if (blockIdx.x == 0 && ct < g.head[i]) acc += (double)p[ct];
  }
  return acc;
}

// ---- rank partials (multi-GPU) ---------------------------------------------
// Fused exchange: the rank's partial goes straight from the reduce's last CTA into
// slot [epoch & 1][rank] of every rank's mailbox (peer stores through NVLink),
// then one system-scope fence and the epoch flags (release).  Parity double
// buffering makes a fast rank's next epoch unable to overwrite a slot that a slow
// rank has not read yet (the next epoch's reduce needs this epoch's scale done).
// Warp-cooperative (call from all 32 lanes of ONE warp, S the same in every
// lane): lane r stores the rank partial into rank r's mailbox, fences, then
// release-stores rank r's flag, so the W remote stores and fences of a W-rank
// exchange overlap instead of running one after another (one NVLink round trip
// instead of W).  A reader that acquires rank r's flag needs only the value
// store that precedes that flag's release in the same lane.
__device__ __forceinline__ void publish_partial_warp(const PeerPost& post, double S) {
  if (!post.mail) return;
  const int lane = threadIdx.x & 31;
  const size_t slot = ((size_t)(post.epoch & 1) * post.world + post.rank) * 2;
  for (int r = lane; r < post.world; r += 32) st_relaxed_sys_f64(post.mail[r] + slot, S);
  __threadfence_system();
  for (int r = lane; r < post.world; r += 32)
    st_release_sys_u64(reinterpret_cast<unsigned long long*>(post.mail[r] + slot + 1), post.epoch);
}

// s = (float)(S_parts[0] + ... + S_parts[nparts-1]) in that fixed order; with
// epoch != 0, S_parts is this rank's mailbox: wait (acquire, system scope, ~30 s
// timeout -> NaN) for every slot of parity epoch & 1 to carry `epoch`, then
// combine the slots in rank order.  *S_full receives the fp64 sum.
// Warp-cooperative (call from all 32 lanes of ONE warp; every lane returns the
// same value): lane r waits for / loads rank r's slot, so the W flag and value
// round trips overlap; the sum is then taken in rank order through shuffles --
// the same additions in the same order as a sequential loop, hence the same bits.
__device__ __forceinline__ float combine_parts_warp(const double* S_parts, int nparts, double* S_full,
                                                   unsigned long long epoch = 0) {
  const int lane = threadIdx.x & 31;
  const double* box = epoch == 0 ? S_parts : S_parts + (size_t)(epoch & 1) * nparts * 2;
  const int stride = epoch == 0 ? 1 : 2;
  bool ok = true;
  if (epoch != 0) {
    // mailbox: wait for every rank's slot of this epoch (peer stores over NVLink)
    const unsigned long long t0 = globaltimer_ns();
    for (int r = lane; r < nparts && ok; r += 32) {
      const unsigned long long* flag = reinterpret_cast<const unsigned long long*>(box + 2 * r + 1);
      while (ld_acquire_sys_u64(flag) != epoch) {
        if (globaltimer_ns() - t0 > 30000000000ull) { ok = false; break; }  // peer lost: no hang
        __nanosleep(64);
      }
    }
    ok = __all_sync(0xffffffffu, ok);
  }
  double S = 0.0;
  for (int base = 0; base < nparts; base += 32) {
    const int r = base + lane;
    double v = 0.0;
    if (r < nparts) v = epoch == 0 ? __ldcg(box + r) : ld_relaxed_sys_f64(box + (size_t)stride * r);
    const int m = nparts - base < 32 ? nparts - base : 32;
    for (int j = 0; j < m; ++j) {  // fixed (rank / chunk) order
      const double x = __shfl_sync(0xffffffffu, v, j);
      S = (base == 0 && j == 0) ? x : S + x;
    }
  }
  if (!ok) S = __longlong_as_double(0x7ff8000000000000ll);
  *S_full = S;
  return (float)S;  // RN to binary32
}

template <typename Kern, typename... Args>
static inline cudaError_t launch_maybe_pdl_smem(Kern k, int grid, int block, size_t smem, bool pdl,
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
static inline cudaError_t launch_maybe_pdl(Kern k, int grid, int block, bool pdl, cudaStream_t st,
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

}  // namespace lnorm
