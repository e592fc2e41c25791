// backward.cu — gradients of the forward ops, for PyTorch autograd of the
// torch.library ops (the paper runs PyTorch *training*
// through its transpiled kernels, so Softmax and the
// normalize of Fig. 1 need their backward passes too).  Each gradient has the
// forward's shape: one reduction, then an elementwise pass.
//
//   normalize (functional form: covered y_i = x_i / s, uncovered y_j = x_j):
//     D = sum_{i in C} g_i y_i / s,   gx_j = ([j in C] ? g_j / s : g_j) - D
//   softmax:      D = sum_k g_k y_k,  gx_j = y_j (g_j - D)
//   log-softmax:  D = sum_k g_k,      gx_j = g_j - exp(y_j) D
//
// Sums in fp64 over fixed partitions (per-thread, warp butterfly, block in warp
// order, per-CTA partials in index order): bit-identical run to run.  HBM
// traffic: read g and y (of the covered set, for the vector normalize's sum)
// once, write gx once; the row kernels' second sweep over a row re-reads it
// from L2.
#include <cuda_runtime.h>
#include <math.h>

#include <stdlib.h>
#include <string.h>

#include "stream_common.cuh"

namespace lnorm {

constexpr int BW_THREADS = 256;
#ifndef NORM_BW_MINB  // probe builds only (occupancy A/B)
#define NORM_BW_MINB 4
#endif
#ifndef NORM_BW_ROW_CTAS
#define NORM_BW_ROW_CTAS 8
#endif
constexpr int BW_ROW_CTAS_PER_SM = NORM_BW_ROW_CTAS;
// Register-resident rows kernel where it applies (rows of <= 4096 floats, 32-byte
// aligned), 3 CTAs per SM, rows from a queue (NORM_ROWS_QUEUE=0: grid-strided;
// same box: softmax / log-softmax / rows-normalize backward 457 / 457 / 492 us vs
// 495 / 496 / 509, profiles/round2/backward/ab_row_queue.txt);
// NORM_BW_REG=0 / NORM_BW_REG_MINB: probe builds only.
// Same box, 65536 x 4096, us per call (profiles/round2/backward/ab_bwreg*.txt):
// softmax / log-softmax / rows-normalize backward 499 / 468 / 505 at 3 CTAs/SM vs
// 503 / 478 / ~548 for the two-sweep kernel (4 CTAs/SM: 513 / 511 / 486; 5: 502 /
// 506 / 508-551).
#ifndef NORM_BW_REG
#define NORM_BW_REG 1
#endif
#ifndef NORM_BW_REG_MINB
#define NORM_BW_REG_MINB 3
#endif

__device__ __forceinline__ bool bw_cov(int64_t i, int64_t L, int64_t G) {
  return L >= 0 ? i < L : (i % 32) < G;
}

// the reduction's term of element (g, y); `cov` only matters for normalize
template <int KIND>
__device__ __forceinline__ double bw_term(float g, float y, bool cov) {
  if (KIND == BW_LOG_SOFTMAX) return (double)g;
  if (KIND == BW_NORMALIZE && !cov) return 0.0;
  return (double)g * (double)y;  // exact in fp64
}

// exp(y) for log-softmax outputs y <= 0 as 2^(y log2 e) on the SFU (MUFU.EX2), as
// the forward softmax does: relative error <= |y| 2^-24 + 2^-22 (< 5.5e-6 for
// y >= -87; below that exp(y) < 1.7e-38).
__device__ __forceinline__ float bw_exp(float y) {
  float r;
  asm("ex2.approx.f32 %0, %1;" : "=f"(r) : "f"(y * 1.4426950408889634f));
  return r;
}

// g / s through the hoisted reciprocal (div_rn: bit-identical to __fdiv_rn,
// exhaustively checked, tests/test_gpu_division.py)
template <int KIND>
__device__ __forceinline__ float bw_out(float g, float y, bool cov, float D, const Divisor& dv) {
  if (KIND == BW_SOFTMAX) return y * (g - D);
  if (KIND == BW_LOG_SOFTMAX) return g - bw_exp(y) * D;
  return (cov ? div_rn(g, dv) : g) - D;
}

// Four outputs of one float4; for normalize the four quotients take one window
// test together (as the forward's div8), the rare out-of-window vector goes
// element by element through div_rn.
template <int KIND>
__device__ __forceinline__ float4 bw_out4(const float4& a, const float4& b, int64_t e, int64_t L, int64_t G,
                                          float D, const Divisor& dv) {
  if (KIND == BW_NORMALIZE && L >= e + 4) {  // all four covered
    const float x[4] = {a.x, a.y, a.z, a.w};
    float q[4];
    bool ok = true;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float q0 = __fmul_rn(x[k], dv.r);
      q[k] = __fmaf_rn(dv.r, __fmaf_rn(-q0, dv.s, x[k]), q0);
      const float ax = fabsf(x[k]);
      ok &= (ax >= dv.lo) & (ax <= dv.hi);
    }
    if (ok) return make_float4(q[0] - D, q[1] - D, q[2] - D, q[3] - D);
  }
  return make_float4(bw_out<KIND>(a.x, b.x, bw_cov(e, L, G), D, dv), bw_out<KIND>(a.y, b.y, bw_cov(e + 1, L, G), D, dv),
                     bw_out<KIND>(a.z, b.z, bw_cov(e + 2, L, G), D, dv), bw_out<KIND>(a.w, b.w, bw_cov(e + 3, L, G), D, dv));
}

// ------------------------------------------------------------------ rows
// Persistent grid, one row per CTA at a time (rows r = blockIdx.x, + grid, ...):
// sweep 1 reduces the row, sweep 2 (same element-to-thread map, so gx may alias
// g or y) writes it.  VEC: float4 accesses (16-byte aligned rows, cols % 4 == 0).
template <int KIND, bool VEC>
__global__ void __launch_bounds__(BW_THREADS, NORM_BW_MINB)
    rows_bwd_kernel(float* gx, const float* g, const float* y, const float* s_rows, int64_t rows,
                    int64_t cols, int64_t ld, int64_t L, int64_t G) {
  __shared__ double red[2][BW_THREADS / 32];
  int par = 0;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x, par ^= 1) {
    const float* gr = g + r * ld;
    const float* yr = y + r * ld;
    float* xr = gx + r * ld;
    double acc = 0.0;
    if (VEC) {
      const int64_t n4 = cols >> 2;
      const float4* g4 = reinterpret_cast<const float4*>(gr);
      const float4* y4 = reinterpret_cast<const float4*>(yr);
#pragma unroll 4
      for (int64_t j = threadIdx.x; j < n4; j += BW_THREADS) {
        const float4 a = g4[j], b = y4[j];
        const int64_t e = 4 * j;
        if (KIND == BW_LOG_SOFTMAX)  // sweep 2 reads y: start its HBM read now
          asm volatile("prefetch.global.L2 [%0];" ::"l"(y4 + j));
        acc += bw_term<KIND>(a.x, b.x, bw_cov(e, L, G)) + bw_term<KIND>(a.y, b.y, bw_cov(e + 1, L, G)) +
               bw_term<KIND>(a.z, b.z, bw_cov(e + 2, L, G)) + bw_term<KIND>(a.w, b.w, bw_cov(e + 3, L, G));
      }
    } else {
      for (int64_t j = threadIdx.x; j < cols; j += BW_THREADS) acc += bw_term<KIND>(gr[j], yr[j], bw_cov(j, L, G));
    }
    const double Dsum = block_sum_1b(acc, red[par]);  // alternating buffers: one barrier per row
    float s = 1.0f, D;
    if (KIND == BW_NORMALIZE) {
      s = s_rows[r];
      D = (float)(Dsum / (double)s);
    } else {
      D = (float)Dsum;
    }
    const Divisor dv = make_divisor(s);
    if (VEC) {
      const int64_t n4 = cols >> 2;
      const float4* g4 = reinterpret_cast<const float4*>(gr);
      const float4* y4 = reinterpret_cast<const float4*>(yr);
      float4* x4 = reinterpret_cast<float4*>(xr);
#pragma unroll 4
      for (int64_t j = threadIdx.x; j < n4; j += BW_THREADS) {
        const float4 a = g4[j], b = y4[j];
        const int64_t e = 4 * j;
        __stcs(x4 + j, bw_out4<KIND>(a, b, e, L, G, D, dv));
      }
    } else {
      for (int64_t j = threadIdx.x; j < cols; j += BW_THREADS)
        xr[j] = bw_out<KIND>(gr[j], yr[j], bw_cov(j, L, G), D, dv);
    }
  }
}

// Register-resident rows (32-byte aligned, cols % 8 == 0, cols <= 2048 MAXV): the
// row's g and y are loaded once with 256-bit loads and kept in registers across
// the block reduction, so the elementwise pass re-reads nothing.
template <int KIND, int MAXV>
__global__ void __launch_bounds__(BW_THREADS, NORM_BW_REG_MINB)
    rows_bwd_reg_kernel(float* gx, const float* g, const float* y, const float* s_rows, int64_t rows,
                        int64_t cols, int64_t ld, int64_t L, int64_t G, unsigned* ctr) {
  // ctr != NULL: rows from a queue (as the forward rows kernels): thread 0 claims
  // the next row before the current row's barrier and publishes it across it,
  // so CTAs on faster SMs take more rows; the last CTA to run dry resets it.
  __shared__ double red[2][BW_THREADS / 32];
  __shared__ int64_t claim[2];
  const int nv = (int)(cols >> 3);
  int par = 0;
  int64_t r = blockIdx.x;
  if (ctr) {
    if (threadIdx.x == 0) claim[0] = (int64_t)atomicAdd(ctr, 1u);
    __syncthreads();
    r = claim[0];
  }
  while (r < rows) {
    const float* gr = g + r * ld;
    const float* yr = y + r * ld;
    f8 a[MAXV], b[MAXV];
#pragma unroll
    for (int k = 0; k < MAXV; ++k) {
      const int idx = k * BW_THREADS + threadIdx.x;
      if (idx < nv) {
        a[k] = ld8(gr + (int64_t)idx * 8);
        b[k] = ld8(yr + (int64_t)idx * 8);
      }
    }
    if (ctr && threadIdx.x == 0) claim[par ^ 1] = r < rows ? (int64_t)atomicAdd(ctr, 1u) : rows;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < MAXV; ++k) {
      const int idx = k * BW_THREADS + threadIdx.x;
      if (idx < nv) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) t += bw_term<KIND>(a[k].v[j], b[k].v[j], bw_cov((int64_t)idx * 8 + j, L, G));
        acc += t;
      }
    }
    const double Dsum = block_sum_1b(acc, red[par]);  // its barrier also publishes claim[par ^ 1]
    float s = 1.0f, D;
    if (KIND == BW_NORMALIZE) {
      s = s_rows[r];
      D = (float)(Dsum / (double)s);
    } else {
      D = (float)Dsum;
    }
    const Divisor dv = make_divisor(s);
    float* xr = gx + r * ld;
#pragma unroll
    for (int k = 0; k < MAXV; ++k) {
      const int idx = k * BW_THREADS + threadIdx.x;
      if (idx < nv) {
        const int64_t e = (int64_t)idx * 8;
        const float4 lo = bw_out4<KIND>(make_float4(a[k].v[0], a[k].v[1], a[k].v[2], a[k].v[3]),
                                        make_float4(b[k].v[0], b[k].v[1], b[k].v[2], b[k].v[3]), e, L, G, D, dv);
        const float4 hi = bw_out4<KIND>(make_float4(a[k].v[4], a[k].v[5], a[k].v[6], a[k].v[7]),
                                        make_float4(b[k].v[4], b[k].v[5], b[k].v[6], b[k].v[7]), e + 4, L, G, D, dv);
        st8_stream(xr + e, f8{{lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w}});
      }
    }
    r = ctr ? claim[par ^ 1] : r + gridDim.x;
    par ^= 1;
  }
  if (ctr && threadIdx.x == 0) {
    __threadfence();  // this CTA's claims on ctr[0] precede its count on ctr[1]
    if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {
      __threadfence();  // every other CTA's claims are visible before the reset
      ctr[0] = 0u;
      ctr[1] = 0u;
    }
  }
}

// ---------------------------------------------------------------- vector
// normalize backward over one vector: D = sum_{i in C} g_i y_i / s by a
// persistent grid (per-CTA partials, last-CTA ticket, index order), then the
// elementwise pass over all n.
template <bool VEC>
__global__ void __launch_bounds__(BW_THREADS, 4)
    vec_bwd_dot_kernel(const float* g, const float* y, int64_t n, int64_t L, int64_t G, const float* s,
                       double* partials, unsigned* ticket, double* D_out) {
  __shared__ double red[BW_THREADS / 32];
  __shared__ unsigned is_last;
  const int64_t len = L >= 0 ? L : n;  // prefix coverage: [0, L); residue: test every index
  const int64_t tid = (int64_t)blockIdx.x * BW_THREADS + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * BW_THREADS;
  double acc = 0.0;
  if (VEC) {
    const int64_t n4 = len >> 2;
    const float4* g4 = reinterpret_cast<const float4*>(g);
    const float4* y4 = reinterpret_cast<const float4*>(y);
#pragma unroll 4
    for (int64_t j = tid; j < n4; j += nth) {
      const float4 a = __ldcs(g4 + j), b = __ldcs(y4 + j);
      acc += (double)a.x * (double)b.x + (double)a.y * (double)b.y + (double)a.z * (double)b.z +
             (double)a.w * (double)b.w;
    }
    if (blockIdx.x == 0 && threadIdx.x < (len & 3)) {
      const int64_t e = 4 * n4 + threadIdx.x;
      acc += (double)g[e] * (double)y[e];
    }
  } else {
    for (int64_t j = tid; j < len; j += nth) acc += bw_term<BW_NORMALIZE>(g[j], y[j], bw_cov(j, L, G));
  }
  pdl_launch_dependents();  // the tile kernel may start loading g (this kernel never writes it)
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
  for (int i = threadIdx.x; i < (int)gridDim.x; i += BW_THREADS) v += __ldcg(partials + i);
  const double Dsum = block_sum(v, red);
  if (threadIdx.x == 0) {
    *D_out = Dsum / (double)*s;
    *ticket = 0u;  // leave the workspace reusable
  }
}

template <bool VEC>
__global__ void __launch_bounds__(BW_THREADS, 4)
    vec_bwd_apply_kernel(float* gx, const float* g, int64_t n, int64_t L, int64_t G, const float* s,
                         const double* D_in) {
  const Divisor dv = make_divisor(*s);
  const float D = (float)__ldcg(D_in);
  const int64_t tid = (int64_t)blockIdx.x * BW_THREADS + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * BW_THREADS;
  if (VEC) {
    const int64_t n4 = n >> 2;
    const float4* g4 = reinterpret_cast<const float4*>(g);
    float4* x4 = reinterpret_cast<float4*>(gx);
    // four float4 loads in flight per thread before their stores (gx may alias g:
    // each element is loaded before it is stored, by the same thread)
    int64_t j = tid;
    for (; j + 3 * nth < n4; j += 4 * nth) {
      float4 a[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) a[k] = __ldcs(g4 + j + k * nth);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        __stcs(x4 + j + k * nth, bw_out4<BW_NORMALIZE>(a[k], a[k], 4 * (j + k * nth), L, G, D, dv));
    }
    for (; j < n4; j += nth) {
      const float4 a = __ldcs(g4 + j);
      __stcs(x4 + j, bw_out4<BW_NORMALIZE>(a, a, 4 * j, L, G, D, dv));
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
      const int64_t e = 4 * n4 + threadIdx.x;
      gx[e] = bw_out<BW_NORMALIZE>(g[e], 0.f, bw_cov(e, L, G), D, dv);
    }
  } else {
    for (int64_t j = tid; j < n; j += nth) gx[j] = bw_out<BW_NORMALIZE>(g[j], 0.f, bw_cov(j, L, G), D, dv);
  }
}

// Elementwise pass as the forward's scale_tile_kernel: a non-persistent grid of
// one 2048-float tile per CTA (one 256-bit load per thread, issued before
// griddepcontrol.wait: the dot kernel does not write g), the last CTA takes the
// unaligned head and the ragged tail.  Prefix coverage [0, L); g and gx
// co-aligned mod 32 bytes.
constexpr int BWT_THREADS = 256;
constexpr int64_t BWT_F = (int64_t)BWT_THREADS * 8;

template <bool ALIAS>
__global__ void __launch_bounds__(BWT_THREADS)
    vec_bwd_tile_kernel(float* gx, const float* g, int64_t n, int64_t L, int64_t head, int64_t ntiles,
                        const float* s, const double* D_in) {
  const bool body = (int64_t)blockIdx.x < ntiles;
  const int64_t off = head + (int64_t)blockIdx.x * BWT_F + (int64_t)threadIdx.x * 8;
  f8 v;
  if (body) v = ALIAS ? ld8(g + off) : ld8_stream(g + off);
  pdl_wait();
  const Divisor dv = make_divisor(*s);
  const float D = (float)__ldcg(D_in);
  if (body) {
    f8 o;
    if (off + 8 <= L) {
      o = div8(v, dv);
#pragma unroll
      for (int j = 0; j < 8; ++j) o.v[j] -= D;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) o.v[j] = bw_out<BW_NORMALIZE>(v.v[j], 0.f, off + j < L, D, dv);
    }
    st8_stream(gx + off, o);
    return;
  }
  for (int64_t i = threadIdx.x; i < head; i += BWT_THREADS) gx[i] = bw_out<BW_NORMALIZE>(g[i], 0.f, i < L, D, dv);
  for (int64_t i = head + ntiles * BWT_F + threadIdx.x; i < n; i += BWT_THREADS)
    gx[i] = bw_out<BW_NORMALIZE>(g[i], 0.f, i < L, D, dv);
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

cudaError_t launch_normalize_backward(float* gx, const float* g, const float* y, const float* s,
                                      const Coverage& cov, const Workspace& ws, const DeviceInfo& d,
                                      cudaStream_t st) {
  const int64_t L = cov.kind == COV_PREFIX ? cov.L : -1;
  const bool vec = L >= 0 && aligned16(gx) && aligned16(g) && aligned16(y);
  int64_t gd = (int64_t)d.sms * 4;
  if (gd > kMaxGrid) gd = kMaxGrid;
  double* D = ws.S + 2;  // S[2]: this pass's D (S[0] / S[1] belong to the forward paths)
  if (vec)
    vec_bwd_dot_kernel<true><<<(int)gd, BW_THREADS, 0, st>>>(g, y, cov.n, L, cov.G, s, ws.partials, ws.ticket, D);
  else
    vec_bwd_dot_kernel<false><<<(int)gd, BW_THREADS, 0, st>>>(g, y, cov.n, L, cov.G, s, ws.partials, ws.ticket, D);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // tile kernel when g and gx are co-aligned mod 32 B (the common case)
  const uintptr_t pg = reinterpret_cast<uintptr_t>(g), px = reinterpret_cast<uintptr_t>(gx);
  if (vec && ((pg ^ px) & 31u) == 0) {
    int64_t head = (int64_t)(((32u - (pg & 31u)) & 31u) / 4);
    if (head > cov.n) head = cov.n;
    const int64_t ntiles = (cov.n - head) / BWT_F;
    if (ntiles + 1 <= 2147483647LL) {
      return gx == g ? launch_maybe_pdl(vec_bwd_tile_kernel<true>, (int)(ntiles + 1), BWT_THREADS, true, st, gx,
                                        g, cov.n, L, head, ntiles, s, (const double*)D)
                     : launch_maybe_pdl(vec_bwd_tile_kernel<false>, (int)(ntiles + 1), BWT_THREADS, true, st, gx,
                                        g, cov.n, L, head, ntiles, s, (const double*)D);
    }
  }
  const int64_t ga = (int64_t)d.sms * 8;
  if (vec)
    vec_bwd_apply_kernel<true><<<(int)ga, BW_THREADS, 0, st>>>(gx, g, cov.n, L, cov.G, s, D);
  else
    vec_bwd_apply_kernel<false><<<(int)ga, BW_THREADS, 0, st>>>(gx, g, cov.n, L, cov.G, s, D);
  return cudaGetLastError();
}

cudaError_t launch_rows_backward(float* gx, const float* g, const float* y, const float* s_rows,
                                 int64_t rows, int64_t cols, int64_t ld, int kind, const Coverage& rc,
                                 const DeviceInfo& d, cudaStream_t st, unsigned* row_ctr) {
  static const bool queue = [] {  // NORM_ROWS_QUEUE=0: grid-strided rows (A/B knob)
    const char* e = getenv("NORM_ROWS_QUEUE");
    return !(e && !strcmp(e, "0"));
  }();
  unsigned* rq = queue && rows < (1ll << 31) ? row_ctr : nullptr;  // 32-bit claim counter
  const int64_t L = kind != BW_NORMALIZE ? cols : (rc.kind == COV_PREFIX ? rc.L : -1);
  const bool vec = aligned16(gx) && aligned16(g) && aligned16(y) && (cols % 4) == 0 && (ld % 4) == 0;
  int64_t gd = (int64_t)d.sms * BW_ROW_CTAS_PER_SM;
  if (rows < gd) gd = rows;
#if NORM_BW_REG
  const bool reg = ((reinterpret_cast<uintptr_t>(gx) | reinterpret_cast<uintptr_t>(g) |
                     reinterpret_cast<uintptr_t>(y)) & 31u) == 0 && (cols % 8) == 0 && (ld % 8) == 0 &&
                   cols <= BW_THREADS * 8 * 2;
  if (reg) {
    int64_t gr = (int64_t)d.sms * NORM_BW_REG_MINB;
    if (rows < gr) gr = rows;
    const bool two = cols > BW_THREADS * 8;
#define NORM_BWR(K)                                                                                 \
  (two ? rows_bwd_reg_kernel<K, 2><<<(int)gr, BW_THREADS, 0, st>>>(gx, g, y, s_rows, rows, cols, ld, L, rc.G, rq) \
       : rows_bwd_reg_kernel<K, 1><<<(int)gr, BW_THREADS, 0, st>>>(gx, g, y, s_rows, rows, cols, ld, L, rc.G, rq))
    if (kind == BW_NORMALIZE) NORM_BWR(BW_NORMALIZE);
    else if (kind == BW_SOFTMAX) NORM_BWR(BW_SOFTMAX);
    else NORM_BWR(BW_LOG_SOFTMAX);
#undef NORM_BWR
    return cudaGetLastError();
  }
#endif
#define NORM_BW(K, V) \
  rows_bwd_kernel<K, V><<<(int)gd, BW_THREADS, 0, st>>>(gx, g, y, s_rows, rows, cols, ld, L, rc.G)
  if (kind == BW_NORMALIZE) {
    if (vec) NORM_BW(BW_NORMALIZE, true);
    else NORM_BW(BW_NORMALIZE, false);
  } else if (kind == BW_SOFTMAX) {
    if (vec) NORM_BW(BW_SOFTMAX, true);
    else NORM_BW(BW_SOFTMAX, false);
  } else {
    if (vec) NORM_BW(BW_LOG_SOFTMAX, true);
    else NORM_BW(BW_LOG_SOFTMAX, false);
  }
#undef NORM_BW
  return cudaGetLastError();
}

}  // namespace lnorm
