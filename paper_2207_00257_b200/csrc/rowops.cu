// rowops.cu — SURVEY §8(f) NEXT-2: the reduce->elementwise PyTorch kernels the
// paper transpiles next to `normalize`: row Softmax /
// LogSoftmax ("aggregation operations like Softmax") and ClassNLLCriterion
// updateOutput / updateGradInput (the NLL loss "uses CUDA's __syncthreads()").
//
// Softmax reuses the rows skeleton of rows.cu: one row per CTA held in
// registers (256-bit loads), the next row prefetched before the current row's
// reductions, block max -> exp -> fp64 block sum -> scale, one HBM read and one
// write per element.  NLL forward is a gather + deterministic two-level
// reduction (per-CTA partials, last-CTA ticket); NLL backward is a write stream
// (zeros plus one value per row).
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "device_common.cuh"
#include "norm_internal.h"

namespace lnorm {

constexpr int SM_THREADS = 256;

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block max (exact, order-independent); NaN propagation is handled by the caller.
__device__ __forceinline__ float block_max(float v, float* redf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) redf[warp] = v;
  __syncthreads();
  float t = lane < nw ? redf[lane] : -INFINITY;
  return warp_max(t);
}

// exp(d) for d = x - m <= 0 as 2^(d * log2 e) on the SFU (MUFU.EX2).  Relative
// error <= |d|·2^-24 (rounding of d, then of d·log2 e) + 2^-22 (ex2.approx):
// below 5.1e-6 for |d| <= 80; smaller results are below 1.8e-35.
__device__ __forceinline__ float exp_shifted(float d) {
  float y;
  asm("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(d * 1.4426950408889634f));
  return y;
}

template <int MAXV>
__device__ __forceinline__ void sm_load(const float* src, int nvr, f8* v) {
#pragma unroll
  for (int k = 0; k < MAXV; ++k) {
    const int idx = k * SM_THREADS + threadIdx.x;
    if (idx < nvr) v[k] = ld8_stream(src + (int64_t)idx * 8);
  }
}

// softmax / log-softmax of one register-resident row.
template <bool LOG, int MAXV>
__device__ __forceinline__ void sm_finish(float* dst, int nvr, f8* v, float* redf, double* redd) {
  // two single-barrier block reductions per row (max, then sum), on distinct
  // buffers, so each row costs two __syncthreads; NaN propagates through max.NaN
  float m = -INFINITY;
#pragma unroll
  for (int k = 0; k < MAXV; ++k)
    if (k * SM_THREADS + (int)threadIdx.x < nvr)
#pragma unroll
      for (int j = 0; j < 8; ++j) m = fmax_nan(m, v[k].v[j]);
  m = block_max_1b(m, redf);
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < MAXV; ++k)
    if (k * SM_THREADS + (int)threadIdx.x < nvr) {
      f8 e;
#pragma unroll
      for (int j = 0; j < 8; ++j) e.v[j] = exp_shifted(v[k].v[j] - m);
      acc += sum8(e);
      if (!LOG) v[k] = e;
    }
  const double S = block_sum_1b(acc, redd);
  if (LOG) {
    const float lse = (float)log(S);
#pragma unroll
    for (int k = 0; k < MAXV; ++k) {
      const int idx = k * SM_THREADS + threadIdx.x;
      if (idx < nvr) {
        f8 y;
#pragma unroll
        for (int j = 0; j < 8; ++j) y.v[j] = (v[k].v[j] - m) - lse;
        st8_stream(dst + (int64_t)idx * 8, y);
      }
    }
  } else {
    // y = e * (1/S): one rounding of 1/S and one of the product (< 1.2e-7 relative)
    const float rs = (float)(1.0 / S);
#pragma unroll
    for (int k = 0; k < MAXV; ++k) {
      const int idx = k * SM_THREADS + threadIdx.x;
      if (idx < nvr) {
        f8 y;
#pragma unroll
        for (int j = 0; j < 8; ++j) y.v[j] = v[k].v[j] * rs;
        st8_stream(dst + (int64_t)idx * 8, y);
      }
    }
  }
}

#ifndef NORM_SM_CTAS  // probe builds only (occupancy A/B): -DNORM_SM_CTAS=5
#define NORM_SM_CTAS 5
#endif
__host__ __device__ constexpr int sm_ctas_per_sm(int maxv) { return maxv >= 4 ? 2 : NORM_SM_CTAS; }

// ctr != NULL: rows from a queue, as rows_vec_kernel (rows.cu): thread 0 claims
// the row after next while the current row is finished and publishes it across
// the row's barriers; the last CTA to run dry resets the queue.
template <bool LOG, int MAXV>
__global__ void __launch_bounds__(SM_THREADS, sm_ctas_per_sm(MAXV))
    softmax_vec_kernel(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                       int64_t ld_in, unsigned* ctr) {
  __shared__ float redf[SM_THREADS / 32];
  __shared__ double redd[SM_THREADS / 32];
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
  auto claim_ahead = [&](int64_t cur_next, int slot) {
    if (ctr && threadIdx.x == 0) claim[slot] = cur_next < rows ? (int64_t)atomicAdd(ctr, 1u) : rows;
  };
  auto next_after = [&](int64_t cur_next, int slot) -> int64_t { return ctr ? claim[slot] : cur_next + step; };
  if (r < rows) sm_load<MAXV>(in + r * ld_in, nvr, a);
  while (r < rows) {
    if (rn < rows) sm_load<MAXV>(in + rn * ld_in, nvr, b);
    claim_ahead(rn, 0);
    sm_finish<LOG, MAXV>(out + r * ld_out, nvr, a, redf, redd);
    int64_t rnn = next_after(rn, 0);
    r = rn;
    rn = rnn;
    if (r >= rows) break;
    if (rn < rows) sm_load<MAXV>(in + rn * ld_in, nvr, a);
    claim_ahead(rn, 1);
    sm_finish<LOG, MAXV>(out + r * ld_out, nvr, b, redf, redd);
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

// Any shape / alignment / in-place: three sweeps over the row from memory.
template <bool LOG>
__global__ void __launch_bounds__(SM_THREADS)
    softmax_generic_kernel(float* out, const float* in, int64_t rows, int64_t cols,
                           int64_t ld_out, int64_t ld_in) {
  __shared__ float redf[SM_THREADS / 32];
  __shared__ double redd[SM_THREADS / 32];
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const float* x = in + r * ld_in;
    float* y = out + r * ld_out;
    float m = -INFINITY;
    int nan = 0;
    for (int64_t i = threadIdx.x; i < cols; i += SM_THREADS) {
      const float xi = x[i];
      m = fmaxf(m, xi);
      nan |= isnan(xi);
    }
    m = block_max(m, redf);
    if (__syncthreads_or(nan)) m = __int_as_float(0x7fffffff);
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < cols; i += SM_THREADS) acc += (double)exp_shifted(x[i] - m);
    const double S = block_sum(acc, redd);  // barrier: every read precedes every write
    const float rs = (float)(1.0 / S), lse = (float)log(S);
    for (int64_t i = threadIdx.x; i < cols; i += SM_THREADS) {
      const float d = x[i] - m;
      y[i] = LOG ? d - lse : exp_shifted(d) * rs;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ NLL
constexpr int NLL_THREADS = 256;

__global__ void __launch_bounds__(NLL_THREADS)
    nll_forward_kernel(const float* __restrict__ logp, const int64_t* __restrict__ target,
                       const float* __restrict__ weight, int64_t N, int64_t C, int64_t ld,
                       int reduction, int64_t ignore_index, float* loss, float* total_weight,
                       double* partials, unsigned* ticket) {
  __shared__ double red[NLL_THREADS / 32];
  __shared__ unsigned is_last;
  double num = 0.0, den = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * NLL_THREADS + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * NLL_THREADS) {
    const int64_t t = target[i];
    double li = 0.0;
    if (t != ignore_index) {
      if (t < 0 || t >= C) {
        li = __longlong_as_double(0x7ff8000000000000ll);  // reading R17: invalid target -> NaN
      } else {
        const double w = weight ? (double)weight[t] : 1.0;
        li = -w * (double)logp[i * ld + t];
        den += w;
      }
    }
    if (reduction == NORM_REDUCTION_NONE) loss[i] = (float)li;
    num += li;
  }
  const double bn = block_sum(num, red);
  const double bd = block_sum(den, red);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = bn;
    partials[2 * blockIdx.x + 1] = bd;
    __threadfence();
    is_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double vn = 0.0, vd = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += NLL_THREADS) {
    vn += __ldcg(partials + 2 * i);
    vd += __ldcg(partials + 2 * i + 1);
  }
  const double Sn = block_sum(vn, red);
  const double Sd = block_sum(vd, red);
  if (threadIdx.x == 0) {
    if (reduction == NORM_REDUCTION_SUM) loss[0] = (float)Sn;
    if (reduction == NORM_REDUCTION_MEAN) loss[0] = (float)(Sn / Sd);
    if (total_weight) *total_weight = (float)Sd;
    *ticket = 0u;
  }
}

// grad[i, :] = 0 except grad[i, t_i] = -w[t_i] * g_i / (MEAN ? total_weight : 1).
template <bool VEC>
__global__ void __launch_bounds__(256)
    nll_backward_kernel(float* __restrict__ grad, const float* __restrict__ grad_out,
                        const int64_t* __restrict__ target, const float* __restrict__ weight,
                        const float* __restrict__ total_weight, int64_t N, int64_t C, int64_t ld,
                        int reduction, int64_t ignore_index) {
  const double tw = reduction == NORM_REDUCTION_MEAN ? (double)*total_weight : 1.0;
  const double g0 = reduction == NORM_REDUCTION_NONE ? 0.0 : (double)grad_out[0];
  // the next row's target (and grad_out) are loaded one row ahead, so the row's
  // write stream does not wait on a dependent load each time
  int64_t r = blockIdx.x;
  int64_t t_next = r < N ? target[r] : 0;
  double go_next = (reduction == NORM_REDUCTION_NONE && r < N) ? (double)grad_out[r] : g0;
  for (; r < N; r += gridDim.x) {
    const int64_t t = t_next;
    const double go = go_next;
    const int64_t rn = r + gridDim.x;
    if (rn < N) {
      t_next = target[rn];
      if (reduction == NORM_REDUCTION_NONE) go_next = (double)grad_out[rn];
    }
    const bool hit = t != ignore_index && t >= 0 && t < C;
    float val = 0.0f;
    if (hit) {
      const double w = weight ? (double)weight[t] : 1.0;
      val = (float)(-w * go / tw);
    }
    float* row = grad + r * ld;
    if constexpr (VEC) {
      const int64_t nv = C >> 3;
      for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) {
        f8 z;
#pragma unroll
        for (int j = 0; j < 8; ++j) z.v[j] = (hit && v * 8 + j == t) ? val : 0.0f;
        st8_stream(row + v * 8, z);
      }
    } else {
      for (int64_t c = threadIdx.x; c < C; c += blockDim.x) row[c] = (hit && c == t) ? val : 0.0f;
    }
  }
}

// The same gradient in two launches (C % 8 == 0, 32 B-aligned rows): a zero
// fill of the [N, C] tile with no loads at all -- one 2048-float tile of one row
// per CTA on a non-persistent grid, so the block scheduler sweeps the gradient
// as one contiguous write wavefront (the scale_tile_kernel pattern) -- then one
// thread per row stores its one nonzero value over the zeros.  The scatter is
// the fill's programmatic dependent: it loads target / weight / grad_out before
// griddepcontrol.wait and stores after it.  Same fp64 arithmetic as
// nll_backward_kernel, so the same bits.
__global__ void __launch_bounds__(256)
    nll_zero_tile_kernel(float* __restrict__ grad, int64_t C, int64_t ld, int64_t tiles_per_row) {
  pdl_launch_dependents();  // the scatter may be scheduled as the last tiles drain
  const int64_t r = blockIdx.x / tiles_per_row;
  const int64_t c0 = (int64_t)(blockIdx.x % tiles_per_row) * 2048 + (int64_t)threadIdx.x * 8;
  if (c0 >= C) return;
  f8 z;
#pragma unroll
  for (int j = 0; j < 8; ++j) z.v[j] = 0.0f;
  st8_stream(grad + r * ld + c0, z);
}

__global__ void __launch_bounds__(256)
    nll_scatter_kernel(float* __restrict__ grad, const float* __restrict__ grad_out,
                       const int64_t* __restrict__ target, const float* __restrict__ weight,
                       const float* __restrict__ total_weight, int64_t N, int64_t C, int64_t ld,
                       int reduction, int64_t ignore_index) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool hit = false;
  float val = 0.0f;
  int64_t t = 0;
  if (r < N) {  // inputs are not written by the zero fill: load them before the wait
    t = target[r];
    hit = t != ignore_index && t >= 0 && t < C;
    if (hit) {
      const double tw = reduction == NORM_REDUCTION_MEAN ? (double)*total_weight : 1.0;
      const double go = reduction == NORM_REDUCTION_NONE ? (double)grad_out[r] : (double)grad_out[0];
      const double w = weight ? (double)weight[t] : 1.0;
      val = (float)(-w * go / tw);
    }
  }
  pdl_wait();  // the zero fill of `grad` is complete
  if (hit) grad[r * ld + t] = val;
}

// ============================================================ launchers

cudaError_t launch_softmax_rows(float* out, const float* in, int64_t rows, int64_t cols,
                                int64_t ld_out, int64_t ld_in, bool log, const DeviceInfo& d,
                                cudaStream_t st, unsigned* row_ctr) {
  static const bool queue = [] {
    const char* e = getenv("NORM_ROWS_QUEUE");
    return !(e && !strcmp(e, "0"));
  }();
  unsigned* rq = queue && rows < (1ll << 31) ? row_ctr : nullptr;  // 32-bit claim counter
  const bool aligned = ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(in)) & 31u) == 0 &&
                       (ld_out % 8) == 0 && (ld_in % 8) == 0 && (cols % 8) == 0;
  const bool vec = aligned && out != in && cols <= (int64_t)SM_THREADS * 8 * 4;
  const int maxv = cols <= SM_THREADS * 8 ? 1 : (cols <= SM_THREADS * 16 ? 2 : 4);
  int64_t g = (int64_t)d.sms * (vec ? sm_ctas_per_sm(maxv) : 8);
  if (rows < g) g = rows;
#define NORM_SM(LG, M) \
  softmax_vec_kernel<LG, M><<<(int)g, SM_THREADS, 0, st>>>(out, in, rows, cols, ld_out, ld_in, rq)
  if (!vec) {
    if (log) softmax_generic_kernel<true><<<(int)g, SM_THREADS, 0, st>>>(out, in, rows, cols, ld_out, ld_in);
    else softmax_generic_kernel<false><<<(int)g, SM_THREADS, 0, st>>>(out, in, rows, cols, ld_out, ld_in);
  } else if (log) {
    if (maxv == 1) NORM_SM(true, 1);
    else if (maxv == 2) NORM_SM(true, 2);
    else NORM_SM(true, 4);
  } else {
    if (maxv == 1) NORM_SM(false, 1);
    else if (maxv == 2) NORM_SM(false, 2);
    else NORM_SM(false, 4);
  }
#undef NORM_SM
  return cudaGetLastError();
}

cudaError_t launch_nll_forward(float* loss, float* total_weight, const float* logp,
                               const int64_t* target, const float* weight, int64_t N, int64_t C,
                               int64_t ld, int reduction, int64_t ignore_index,
                               const Workspace& ws, const DeviceInfo& d, cudaStream_t st) {
  int64_t g = (N + NLL_THREADS - 1) / NLL_THREADS;
  if (g > (int64_t)d.sms * 4) g = (int64_t)d.sms * 4;
  if (g > kMaxGrid / 2) g = kMaxGrid / 2;
  if (g < 1) g = 1;
  nll_forward_kernel<<<(int)g, NLL_THREADS, 0, st>>>(logp, target, weight, N, C, ld, reduction,
                                                     ignore_index, loss, total_weight,
                                                     ws.partials, ws.ticket);
  return cudaGetLastError();
}

cudaError_t launch_nll_backward(float* grad, const float* grad_out, const int64_t* target,
                                const float* weight, const float* total_weight, int64_t N,
                                int64_t C, int64_t ld, int reduction, int64_t ignore_index,
                                const DeviceInfo& d, cudaStream_t st) {
  const bool vec = (reinterpret_cast<uintptr_t>(grad) & 31u) == 0 && ld % 8 == 0 && C % 8 == 0;
  // NORM_NLL_TILE=0: the persistent row loop below instead of the tile grid (A/B)
  static const bool tile = [] {
    const char* e = getenv("NORM_NLL_TILE");
    return !(e && !strcmp(e, "0"));
  }();
  const int64_t tpr = (C + 2047) / 2048;
  if (vec && tile && N > 0 && N <= 0x7fffffffll / tpr) {
    const int threads = C < 2048 ? (int)((C / 8 + 31) / 32 * 32) : 256;
    nll_zero_tile_kernel<<<(unsigned)(N * tpr), threads, 0, st>>>(grad, C, ld, tpr);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};  // the scatter as the fill's programmatic dependent
    cfg.gridDim = dim3((unsigned)((N + 255) / 256));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_mode() != PDL_OFF ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, nll_scatter_kernel, grad, grad_out, target, weight, total_weight, N, C, ld,
                              reduction, ignore_index);
  }
  int64_t g = (int64_t)d.sms * 8;
  if (N < g) g = N;
  int threads = (int)((vec ? C / 8 : C) < 256 ? ((vec ? C / 8 : C) + 31) / 32 * 32 : 256);
  if (threads < 32) threads = 32;
  if (vec)
    nll_backward_kernel<true><<<(int)g, threads, 0, st>>>(grad, grad_out, target, weight,
                                                          total_weight, N, C, ld, reduction,
                                                          ignore_index);
  else
    nll_backward_kernel<false><<<(int)g, threads, 0, st>>>(grad, grad_out, target, weight,
                                                           total_weight, N, C, ld, reduction,
                                                           ignore_index);
  return cudaGetLastError();
}

}  // namespace lnorm
