// rows.cu — batched per-row normalize (reading R10, BASELINE configs[4]):
// TMA-staged warp-per-row kernel for sparsely covered rows, register-resident
// CTA-per-row kernel for dense rows, and a generic fallback.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include "stream_common.cuh"

namespace lnorm {

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

// ctr != NULL: rows come from a queue instead of r, r + grid, ...: thread 0
// claims the row after next with an atomic while the current row is finished (the
// claim's round trip overlaps the row) and publishes it through shared memory
// across the row's barrier; CTAs on faster SMs take more rows, so the grid ends
// together.  Each row's result is independent of which CTA computes it.  The
// last CTA to run dry resets the queue.
template <bool ALIAS, int MAXV>
__global__ void __launch_bounds__(ROW_THREADS, row_ctas_per_sm(MAXV))
    rows_vec_kernel(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                    int64_t ld_in, int64_t L, int64_t G, float* sum_out, double* sum_out_f64,
                    unsigned* ctr) {
  __shared__ double red[2][ROW_THREADS / 32];  // alternated by row: one barrier per row
  __shared__ int64_t claim[2];
  const int nvr = (int)(cols >> 3);
  const int64_t step = gridDim.x;
  f8 a[MAXV], b[MAXV];
  int64_t r, rn;
  if (ctr) {
    if (threadIdx.x == 0) {
      claim[0] = (int64_t)atomicAdd(ctr, 1u);
      claim[1] = claim[0] < rows ? (int64_t)atomicAdd(ctr, 1u) : rows;
    }
    __syncthreads();
    r = claim[0];
    rn = claim[1];
  } else {
    r = blockIdx.x;
    rn = r + step;
  }
  // the row after rn: claimed by thread 0 before row_finish's barrier, read after it
  auto next_after = [&](int64_t cur_next, int slot) -> int64_t {
    if (!ctr) return cur_next + step;
    return claim[slot];
  };
  auto claim_ahead = [&](int64_t cur_next, int slot) {
    if (ctr && threadIdx.x == 0) claim[slot] = cur_next < rows ? (int64_t)atomicAdd(ctr, 1u) : rows;
  };
  if (r < rows) row_load<ALIAS, MAXV>(in + r * ld_in, nvr, a);
  while (r < rows) {
    if (rn < rows) row_load<ALIAS, MAXV>(in + rn * ld_in, nvr, b);
    claim_ahead(rn, 0);
    row_finish<MAXV>(out + r * ld_out, nvr, a, r, L, G, red[0], sum_out, sum_out_f64);
    int64_t rnn = next_after(rn, 0);
    r = rn;
    rn = rnn;
    if (r >= rows) break;
    if (rn < rows) row_load<ALIAS, MAXV>(in + rn * ld_in, nvr, a);
    claim_ahead(rn, 1);
    row_finish<MAXV>(out + r * ld_out, nvr, b, r, L, G, red[1], sum_out, sum_out_f64);
    rnn = next_after(rn, 1);
    r = rn;
    rn = rnn;
  }
  if (ctr && threadIdx.x == 0) __threadfence();  // claims on ctr[0] precede the count
  if (ctr && threadIdx.x == 0 && atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {  // all CTAs done claiming
    __threadfence();  // every other CTA's claims are visible before the reset
    ctr[0] = 0u;
    ctr[1] = 0u;
  }
}

// Batched rows, TMA-staged, one WARP per row (rows of <= 48 KiB, 16-byte aligned
// with cols % 4 == 0).  One CTA per SM: lane 0 of warp 0 streams whole rows
// into a ring of S shared-memory stages with cp.async.bulk; consumer warp w
// (W warps, W divides S) owns stages w, w + W, ... and processes this CTA's
// rows k = w, w + W, ...: sum
// the row out of shared memory, warp-shuffle reduce (no block barrier on the
// per-row critical path), then scale the covered elements out of shared memory
// into `out`.  Up to S rows are in flight per SM, so HBM stays busy while each
// warp finishes its row.
constexpr int RB_MAX_STAGES = 16, RB_MAX_WARPS = 16;
#ifndef NORM_RB_BUDGET_KIB  // probe builds only (ring depth A/B): -DNORM_RB_BUDGET_KIB=128
#define NORM_RB_BUDGET_KIB 200
#endif
constexpr size_t RB_SMEM_BUDGET = (size_t)NORM_RB_BUDGET_KIB * 1024;

// ctr != NULL: the producer takes its grid-strided share of the first 97 % of the
// rows, then claims rows of the rest from a queue (one ahead), tagging each stage
// with its row (stage_row); after the last row it posts an end marker to each
// consumer warp's next stage; the last producer to run dry resets the queue.
__global__ void __launch_bounds__(32 * (1 + RB_MAX_WARPS), 1)
    rows_bulk_kernel(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                     int64_t ld_in, int64_t L, int64_t G, int S, int W, float* sum_out,
                     double* sum_out_f64, unsigned* ctr) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[RB_MAX_STAGES], empty[RB_MAX_STAGES];
  __shared__ int64_t stage_row[RB_MAX_STAGES];
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
      if (!ctr) {
        for (int64_t r = blockIdx.x; r < rows; r += step, ++k) {
          const int st = (int)(k % S);
          if (k >= S) stage_acquire(&empty[st], (unsigned)(((k / S) - 1) & 1));
          mbar_arrive_expect_tx(&full[st], row_bytes);
          bulk_g2s(ring + st * stage_bytes, in + r * ld_in, row_bytes, &full[st]);
        }
      } else {
        // rows [0, rs) grid-strided, then rows [rs, rows) from the queue, one
        // claim ahead (a claim per row for every row capped the single producer
        // at about one row per atomic round trip)
        const int64_t dyn = rows * 3 / 100 > 8 * step ? rows * 3 / 100 : 8 * step;
        const int64_t rs = rows > dyn ? rows - dyn : 0;
        auto issue = [&](int64_t r) {
          const int st = (int)(k % S);
          if (k >= S) stage_acquire(&empty[st], (unsigned)(((k / S) - 1) & 1));
          stage_row[st] = r;
          mbar_arrive_expect_tx(&full[st], row_bytes);
          bulk_g2s(ring + st * stage_bytes, in + r * ld_in, row_bytes, &full[st]);
          ++k;
        };
        int64_t next = rs + (int64_t)atomicAdd(ctr, 1u);
        for (int64_t r = blockIdx.x; r < rs; r += step) issue(r);
        while (next < rows) {
          const int64_t r = next;
          next = rs + (int64_t)atomicAdd(ctr, 1u);
          issue(r);
        }
        __threadfence();  // this CTA's claims on ctr[0] precede its count on ctr[1]
        if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {  // every producer has claimed its last row
          __threadfence();  // every other CTA's claims are visible before the reset
          ctr[0] = 0u;
          ctr[1] = 0u;
        }
        for (int j = 0; j < W; ++j, ++k) {  // end marker in each consumer warp's next stage
          const int st = (int)(k % S);
          if (k >= S) stage_acquire(&empty[st], (unsigned)(((k / S) - 1) & 1));
          stage_row[st] = -1;
          mbar_arrive(&full[st]);
        }
      }
    }
    return;
  }
  const int w = warp - 1;
  const int nq = (int)(cols >> 2);  // float4s per row
  const bool vst = ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) && (ld_out % 4 == 0);
  for (int64_t k = w; ctr || blockIdx.x + k * step < rows; k += W) {
    const int st = (int)(k % S);
    mbar_wait(&full[st], (unsigned)((k / S) & 1));
    const int64_t r = ctr ? *(volatile int64_t*)&stage_row[st] : blockIdx.x + k * step;
    if (r < 0) break;
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

cudaError_t launch_rows(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                        int64_t ld_in, const Coverage& rc, float* sum_out, double* sum_out_f64,
                        const DeviceInfo& d, cudaStream_t st, unsigned* row_ctr) {
  static const bool queue = [] {
    const char* e = getenv("NORM_ROWS_QUEUE");
    return !(e && !strcmp(e, "0"));
  }();
  unsigned* rq = queue && rows < (1ll << 31) ? row_ctr : nullptr;  // 32-bit claim counter
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
  static const bool no_bulk = [] {  // A/B knob: NORM_ROWS_NO_BULK=1 forces the register kernel
    const char* e = getenv("NORM_ROWS_NO_BULK");
    return e && strcmp(e, "0") != 0 && e[0] != '\0';
  }();
  if (bulk_ok && !no_bulk) {
    const size_t stage_bytes = ((size_t)cols * 4 + 127) & ~(size_t)127;
    int S = (int)(RB_SMEM_BUDGET / stage_bytes);
    if (S > RB_MAX_STAGES) S = RB_MAX_STAGES;
    S &= ~1;
    // Consumer warps: warp w takes rows k = w, w + W, ... in stage k % S, and its
    // mbarrier parity waits are only safe if the previous use of that stage was
    // its own (so it has landed): W must divide S.  One stage per warp (W = S)
    // measured best for 16 KiB rows (204 vs 209 us with W = S / 2); W = 8 with
    // S = 12 aliased phases and read stale rows.  NORM_ROWS_BULK_WARPS: A/B knob,
    // honoured only if it divides S.
    static const int warps_env = [] {
      const char* e = getenv("NORM_ROWS_BULK_WARPS");
      return e ? atoi(e) : 0;
    }();
    int W = S;
    if (warps_env > 0 && S % warps_env == 0) W = warps_env;
    if (W > RB_MAX_WARPS) W = RB_MAX_WARPS;
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
      rows_bulk_kernel<<<(int)gb, 32 * (1 + W), (size_t)S * stage_bytes, st>>>(
          out, in, rows, cols, ld_out, ld_in, L, rc.G, S, W, sum_out, sum_out_f64, rq);
      return cudaGetLastError();
    }
  }
#define NORM_ROWS(A, M)                                                                           \
  rows_vec_kernel<A, M><<<(int)g, ROW_THREADS, 0, st>>>(out, in, rows, cols, ld_out, ld_in, L, rc.G, \
                                                       sum_out, sum_out_f64, rq)
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
