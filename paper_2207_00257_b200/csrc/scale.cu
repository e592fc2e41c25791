// scale.cu — the kernel body of Fig. 1 after LICM:
// out[i] = in[i] / s for i in the covered set C(n), other outputs untouched.
// TMA-bulk load ring (large, co-aligned), LDG.E.256 or scalar (otherwise),
// residue coverage (literal n <= 992), and the one-CTA small path.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include "stream_common.cuh"

namespace lnorm {

#ifdef NORM_TIMELINE  // probe builds only (scripts/pdl_timeline.py): per-CTA %globaltimer stamps
__device__ unsigned long long g_scale_ts[4096 * 5];
#define SCL_STAMP(k) g_scale_ts[blockIdx.x * 5 + (k)] = globaltimer_ns();
extern "C" __attribute__((visibility("default"))) int norm_debug_scale_timeline(unsigned long long* host,
                                                                                 int n) {
  return (int)cudaMemcpyFromSymbol(host, g_scale_ts, (size_t)n * sizeof(unsigned long long));
}
#else
#define SCL_STAMP(k)
#endif

// ---------------------------------------------------------------- scale
template <bool VEC, bool ALIAS>
__global__ void __launch_bounds__(SC_THREADS)
    scale_kernel(float* out, const float* in, int64_t len, const double* __restrict__ S_parts,
                 int nparts, float* sum_out, double* sum_out_f64, unsigned long long epoch) {
  __shared__ float s_sh;
  pdl_wait();  // S_parts are complete and visible; `in` is no longer being read
  if (threadIdx.x < 32) {
    double S;
    const float s = combine_parts_warp(S_parts, nparts, &S, epoch);
    if (threadIdx.x == 0) {
      s_sh = s;
      if (blockIdx.x == 0) {
        if (sum_out) *sum_out = s;
        if (sum_out_f64) *sum_out_f64 = S;
      }
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
// ctr != NULL: chunks are dealt from a queue (the producer claims the next chunk
// with an atomic, one ahead) instead of grid-strided, so SMs that stream faster
// take more chunks and the grid finishes together; every output element is the
// same quotient whoever computes it, so this changes no bits.  The last producer
// to run dry resets the queue for the next call.
__global__ void __launch_bounds__(BK_THREADS, 1)
    scale_bulk_kernel(float* out, const float* in, int64_t len, const double* __restrict__ S_parts,
                      int nparts, float* sum_out, double* sum_out_f64, unsigned long long epoch,
                      unsigned* ctr) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[SB_STAGES], empty[SB_STAGES];
  __shared__ int64_t stage_chunk[SB_STAGES];
  __shared__ float s_sh;
  auto r = bulk_ring_init<SB_STAGES, SB_CHUNK>(ring, full, empty);
  constexpr int64_t CF = SB_CHUNK / 4;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      SCL_STAMP(0);  // producer entry (before griddepcontrol.wait: PDL lets it start early)
      if (!ctr) {
        bulk_produce<false>(r, in, len, 0);
      } else {
        int64_t head, nchunks;
        bulk_split<CF>(in, len, &head, &nchunks);
        const float* body = in + head;
        int64_t next = (int64_t)atomicAdd(ctr, 1u);
        for (;;) {
          const int64_t c = next;
          if (c >= nchunks) break;
          next = (int64_t)atomicAdd(ctr, 1u);
          if (r.issued >= SB_STAGES) stage_acquire(&r.empty[r.stage], r.phase ^ 1);
          stage_chunk[r.stage] = c;
          mbar_arrive_expect_tx(&r.full[r.stage], SB_CHUNK);
          bulk_g2s(r.buf + (size_t)r.stage * SB_CHUNK, body + c * CF, SB_CHUNK, &r.full[r.stage]);
#ifdef NORM_TIMELINE
          if (r.issued == 0) SCL_STAMP(1);  // first TMA chunk issued
#endif
          ++r.issued;
          r.advance();
        }
        __threadfence();  // this CTA's claims on ctr[0] precede its count on ctr[1]
        if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {  // every producer has claimed its last chunk
          __threadfence();  // every other CTA's claims are visible before the reset
          ctr[0] = 0u;
          ctr[1] = 0u;
        }
        if (r.issued >= SB_STAGES) stage_acquire(&r.empty[r.stage], r.phase ^ 1);
        stage_chunk[r.stage] = -1;  // end marker: completes with no bytes
        mbar_arrive(&r.full[r.stage]);
      }
    }
    return;
  }
  const int ct = threadIdx.x - 32;
  pdl_wait();
  if (ct < 32) {  // consumer warp 0
    if (ct == 0) SCL_STAMP(2);  // griddepcontrol.wait returned: the reduce grid is complete
    double S;
    const float s = combine_parts_warp(S_parts, nparts, &S, epoch);
    if (ct == 0) {
      s_sh = s;
      if (blockIdx.x == 0) {
        if (sum_out) *sum_out = s;
        if (sum_out_f64) *sum_out_f64 = S;
      }
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(BK_CONSUMERS) : "memory");  // consumers only
  const Divisor dv = make_divisor(s_sh);
#ifdef NORM_TIMELINE
  bool first = true;
#endif
  if (!ctr) {
    bulk_scale_consume(r, out, in, len, dv, ct);
    return;
  }
  int64_t head, nchunks;
  bulk_split<CF>(in, len, &head, &nchunks);
  float* ob = out + head;
  for (;;) {
    mbar_wait(&r.full[r.stage], r.phase);
    const int64_t c = *(volatile int64_t*)&stage_chunk[r.stage];
    if (c < 0) break;
    const float4* q = reinterpret_cast<const float4*>(r.buf + (size_t)r.stage * SB_CHUNK);
    float* oc = ob + c * CF;
#pragma unroll
    for (int k = 0; k < SB_CHUNK / 32 / BK_CONSUMERS; ++k) {
      const int i = k * BK_CONSUMERS + ct;
      const float4 a = q[2 * i], b = q[2 * i + 1];
      st8_stream(oc + (int64_t)i * 8, div8_fchk(f8{{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w}}, dv));
    }
#ifdef NORM_TIMELINE
    if (first && ct == 0) SCL_STAMP(3);  // first chunk divided and stored
    first = false;
#endif
    stage_release(&r.empty[r.stage]);
    r.advance();
  }
#ifdef NORM_TIMELINE
  if (ct == 0) SCL_STAMP(4);  // last chunk stored
#endif
  const int64_t rbeg = head + nchunks * CF;  // remainder, then the head
  for (int64_t i = rbeg + (int64_t)blockIdx.x * BK_CONSUMERS + ct; i < len;
       i += (int64_t)gridDim.x * BK_CONSUMERS)
    out[i] = div_rn(in[i], dv);
  if (blockIdx.x == 0 && ct < head) out[ct] = div_rn(in[ct], dv);
}

// Scale, one-tile-per-CTA variant (the default for out/in co-aligned mod 32 B):
// a NON-persistent grid of (len - head) / TILE_F CTAs, each loading one
// contiguous TILE_F-float tile with 256-bit loads (one per thread) BEFORE
// griddepcontrol.wait -- `in` is not written by the preceding reduce -- then
// reading s, dividing and storing.  The hardware block scheduler hands tiles out
// in index order as CTAs retire, so the reads and writes of the whole GPU sweep
// the buffers as one contiguous wavefront; this measured 6.99 TB/s (n = 2^32,
// IEEE division) against 6.69-6.78 for the persistent TMA ring above and 5.8-6.0
// for persistent grid-stride loops of the same loads
// (scripts/microbench_scale2.cu, profiles/round2/mb_scale2_*.txt).  CTA index
// `ntiles` (the grid's last) takes the unaligned head and the ragged remainder.
// ALIAS (out == in): coherent loads instead of the read-only path; each element
// is read and written by the same thread, so aliasing needs nothing else.
constexpr int TILE_THREADS = 256;
constexpr int64_t TILE_F = (int64_t)TILE_THREADS * 8;
template <bool ALIAS>
__global__ void __launch_bounds__(TILE_THREADS)
    scale_tile_kernel(float* out, const float* in, int64_t len, int64_t head, int64_t ntiles,
                      const double* __restrict__ S_parts, int nparts, float* sum_out, double* sum_out_f64,
                      unsigned long long epoch) {
  __shared__ float s_sh;
  const bool body = (int64_t)blockIdx.x < ntiles;
  const int64_t off = head + (int64_t)blockIdx.x * TILE_F + (int64_t)threadIdx.x * 8;
  f8 v;
  if (body) v = ALIAS ? ld8(in + off) : ld8_stream(in + off);
  pdl_wait();
  if (threadIdx.x < 32) {
    double S;
    const float s = combine_parts_warp(S_parts, nparts, &S, epoch);
    if (threadIdx.x == 0) {
      s_sh = s;
      if (blockIdx.x == 0) {
        if (sum_out) *sum_out = s;
        if (sum_out_f64) *sum_out_f64 = S;
      }
    }
  }
  __syncthreads();
  const Divisor dv = make_divisor(s_sh);
  if (body) {
    st8_stream(out + off, div8_fchk(v, dv));
    return;
  }
  for (int64_t i = threadIdx.x; i < head; i += TILE_THREADS) out[i] = div_rn(in[i], dv);
  for (int64_t i = head + ntiles * TILE_F + threadIdx.x; i < len; i += TILE_THREADS)
    out[i] = div_rn(in[i], dv);
}

__global__ void __launch_bounds__(256)
    scale_residue_kernel(float* out, const float* in, int64_t len, int64_t gbegin, int64_t G,
                         const double* __restrict__ S_parts, int nparts, float* sum_out,
                         double* sum_out_f64, unsigned long long epoch) {
  __shared__ float s_sh;
  pdl_wait();
  if (threadIdx.x < 32) {
    double S;
    const float s = combine_parts_warp(S_parts, nparts, &S, epoch);
    if (threadIdx.x == 0) {
      s_sh = s;
      if (blockIdx.x == 0) {
        if (sum_out) *sum_out = s;
        if (sum_out_f64) *sum_out_f64 = S;
      }
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
  // Launched as a programmatic dependent of whatever precedes it on the stream
  // (back-to-back latency-bound calls: the next call's CTA is resident while
  // this one runs): wait for the predecessor's completion and memory before
  // touching anything, then let the next call launch.
  pdl_wait();
  pdl_launch_dependents();
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

cudaError_t launch_scale(float* out, const float* in, int64_t len, const double* S_parts,
                         int nparts, float* sum_out, double* sum_out_f64, const DeviceInfo& d,
                         bool pdl, cudaStream_t st, unsigned long long epoch, unsigned* ctr) {
  const int64_t per_chunk = (int64_t)SC_THREADS * SC_UNROLL * 8;
  int64_t g = (len + per_chunk - 1) / per_chunk;
  const int64_t gmax = (int64_t)d.sms * SC_CTAS_PER_SM;
  if (g > gmax) g = gmax;
  if (g < 1) g = 1;
  const bool vec = ((reinterpret_cast<uintptr_t>(out) - reinterpret_cast<uintptr_t>(in)) & 31u) == 0;
  const bool alias = out == in;
  // NORM_SCALE_KERNEL=tile (default) | bulk | grid: which co-aligned scale kernel
  // (A/B runs only; every choice gives the same bits).
  static const int which = [] {
    const char* e = getenv("NORM_SCALE_KERNEL");
    if (e && !strcmp(e, "bulk")) return 1;
    if (e && !strcmp(e, "grid")) return 2;
    return 0;
  }();
  if (vec && which == 0) {
    int64_t head = (int64_t)(((32u - (reinterpret_cast<uintptr_t>(in) & 31u)) & 31u) / 4u);
    if (head > len) head = len;
    const int64_t ntiles = (len - head) / TILE_F;
    if (ntiles + 1 > 0x7fffffffll) return cudaErrorInvalidConfiguration;
    if (alias)
      return launch_maybe_pdl(scale_tile_kernel<true>, (int)(ntiles + 1), TILE_THREADS, pdl, st, out, in,
                              len, head, ntiles, S_parts, nparts, sum_out, sum_out_f64, epoch);
    return launch_maybe_pdl(scale_tile_kernel<false>, (int)(ntiles + 1), TILE_THREADS, pdl, st, out, in,
                            len, head, ntiles, S_parts, nparts, sum_out, sum_out_f64, epoch);
  }
  if (vec && len >= kBulkMinN && which == 1) {
    static int configured[64] = {0};
    if (d.device < 64 && !configured[d.device]) {
      cudaError_t e = cudaFuncSetAttribute(scale_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)SB_SMEM);
      if (e != cudaSuccess) return e;
      configured[d.device] = 1;
    }
    static const bool queue = [] {
      const char* e = getenv("NORM_SCALE_QUEUE");
      return !(e && !strcmp(e, "0"));
    }();
    return launch_maybe_pdl_smem(scale_bulk_kernel, d.sms, BK_THREADS, SB_SMEM, pdl, st, out, in,
                                 len, S_parts, nparts, sum_out, sum_out_f64, epoch,
                                 queue ? ctr : (unsigned*)nullptr);
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
  return launch_maybe_pdl(small_kernel, 1, SMALL_THREADS, pdl_chain(), st, out, in, cov.n, (int)cov.kind,
                          cov.L, cov.G, sum_out, sum_out_f64);
}

}  // namespace lnorm
