/*
 * oracle/norm_oracle.c — CPU oracle for Fig. 1 `normalize` (arxiv 2207.00257).
 *
 * TEST INFRASTRUCTURE ONLY (see norm_oracle.h).  Compiled with
 * -O2 -ffp-contract=off -fno-fast-math; no SIMD intrinsics, no threads.
 *
 * What the oracle computes (Fig. 1, and §2.1):
 *   for every (blockIdx b, threadIdx t) of normalize<<<(n+31)/32, 32>>>:
 *       tid = b + 32 t                (literal index)
 *       val = sum(in, n)              (`sum` elided at :100)
 *       if (tid < n) out[tid] = in[tid] / val
 * Form 1 evaluates `sum` per thread (as written), form 2 once per block (the
 * commented shared-memory variant), form 3 once before the
 * grid (after parallel LICM).
 */
#include "norm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define FIG1_BLOCK 32 /* blockDim.x of the launch */

/* ------------------------------------------------------------------ launch */

int64_t oracle_grid_blocks(int64_t n) { return (n + 31) / 32; /* PAPER.md:113 */ }

int64_t oracle_tid(int64_t b, int64_t t, int mode) {
  if (mode == ORACLE_LITERAL) return b + (int64_t)FIG1_BLOCK * t;
  return b * (int64_t)FIG1_BLOCK + t;                             /* reading R1   */
}

/* ---------------------------------------------------------------- coverage */

int oracle_coverage_brute(int64_t n, int mode, uint32_t* mult) {
  if (n < 0 || (n > 0 && !mult)) return 1;
  if (n > 0) memset(mult, 0, (size_t)n * sizeof(uint32_t));
  int64_t G = oracle_grid_blocks(n);
  for (int64_t b = 0; b < G; ++b)
    for (int64_t t = 0; t < FIG1_BLOCK; ++t) {
      int64_t tid = oracle_tid(b, t, mode);
      if (tid < n) mult[tid] += 1; /* `if (tid < n)` */
    }
  return 0;
}

/* Closed form: tid = b + 32t with 0 <= b < G, 0 <= t < 32.
 *  G >= 32: the b-range spans every residue mod 32, so tids fill [0, G-1+992]
 *           without gaps; C(n) = [0, min(n, G+992)).
 *  G <  32: tid mod 32 = b, so C(n) = {x < n : x mod 32 < G}.            */
int oracle_is_covered(int64_t n, int mode, int64_t i) {
  if (i < 0 || i >= n) return 0;
  if (mode != ORACLE_LITERAL) return 1;
  int64_t G = oracle_grid_blocks(n);
  if (G >= 32) return i < G + 992;
  return (i % 32) < G;
}

int oracle_coverage_closed(int64_t n, int mode, int64_t* count, int64_t* prefix_len) {
  if (n < 0 || !count || !prefix_len) return 1;
  if (n == 0) { *count = 0; *prefix_len = 0; return 0; }
  if (mode != ORACLE_LITERAL) { *count = n; *prefix_len = n; return 0; }
  int64_t G = oracle_grid_blocks(n);
  if (G >= 32) {
    int64_t L = n < G + 992 ? n : G + 992;
    *count = L;
    *prefix_len = L;
    return 0;
  }
  int64_t rem = n % 32;
  *count = (n / 32) * G + (rem < G ? rem : G);
  *prefix_len = (n <= 32) ? 1 : -1; /* C = {0} when G == 1 */
  return 0;
}

/* -------------------------------------------------------------------- sums */

/* Reading R2: sum(data, n) = sum_{i<n} data[i], PAPER.md:100 (body elided). */
double oracle_sum_seq(const float* x, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += (double)x[i];
  return s;
}

/* Exact superaccumulator.  A finite binary32 value is mant * 2^(k - 149) with
 * integer mant < 2^24 and k in [0, 253]; the accumulator holds the integer
 * sum_i (+-mant_i << k_i) in 32-bit digits stored in int64 limbs (headroom for
 * 2^30 additions between carry normalisations). */
#define ACC_LIMBS 12
typedef struct {
  int64_t limb[ACC_LIMBS];
  int64_t pending;
  int64_t nposinf, nneginf, nnan, nterms, nnegzero;
} acc_t;

static void acc_norm(acc_t* a) {
  for (int j = 0; j < ACC_LIMBS - 1; ++j) {
    int64_t low = a->limb[j] & 0xFFFFFFFFll;
    int64_t carry = (a->limb[j] - low) / 4294967296ll; /* exact: divisible */
    a->limb[j] = low;
    a->limb[j + 1] += carry;
  }
  a->pending = 0;
}

static void acc_add(acc_t* a, float f, int absolute) {
  uint32_t u;
  memcpy(&u, &f, sizeof u);
  uint32_t sign = u >> 31, e = (u >> 23) & 0xFFu, m = u & 0x7FFFFFu;
  if (absolute) sign = 0;
  a->nterms++;
  if (e == 0xFFu) {
    if (m) a->nnan++;
    else if (sign) a->nneginf++;
    else a->nposinf++;
    return;
  }
  if (e == 0 && m == 0 && sign) a->nnegzero++;
  uint64_t mant = e ? (m | 0x800000u) : m;
  int k = e ? (int)e - 1 : 0;
  uint64_t v = mant << (k % 32);
  int j = k / 32;
  int64_t lo = (int64_t)(v & 0xFFFFFFFFull), hi = (int64_t)(v >> 32);
  if (sign) { a->limb[j] -= lo; a->limb[j + 1] -= hi; }
  else      { a->limb[j] += lo; a->limb[j + 1] += hi; }
  if (++a->pending == (1ll << 30)) acc_norm(a);
}

static int acc_bit(const int64_t* d, int p) { return (int)((d[p / 32] >> (p % 32)) & 1); }

/* Round the exact integer (times 2^-149) to the nearest double, ties to even. */
static double acc_result(acc_t* a) {
  if (a->nnan || (a->nposinf && a->nneginf)) return NAN; /* reading R7 */
  if (a->nposinf) return INFINITY;
  if (a->nneginf) return -INFINITY;
  acc_norm(a);
  int neg = a->limb[ACC_LIMBS - 1] < 0;
  if (neg) {
    for (int j = 0; j < ACC_LIMBS; ++j) a->limb[j] = -a->limb[j];
    acc_norm(a);
  }
  int top = -1;
  for (int p = 32 * ACC_LIMBS - 1; p >= 0; --p)
    if (acc_bit(a->limb, p)) { top = p; break; }
  if (top < 0) /* exact zero: -0 only if every term was -0 (IEEE sum) */
    return (a->nterms > 0 && a->nnegzero == a->nterms) ? -0.0 : 0.0;
  uint64_t M = 0;
  int low = top - 52 > 0 ? top - 52 : 0;
  for (int p = top; p >= low; --p) M = (M << 1) | (uint64_t)acc_bit(a->limb, p);
  if (low > 0) {
    int round = acc_bit(a->limb, low - 1), sticky = 0;
    for (int p = low - 2; p >= 0 && !sticky; --p) sticky = acc_bit(a->limb, p);
    if (round && (sticky || (M & 1))) M += 1; /* 2^53 is still exact */
  }
  double r = ldexp((double)M, low - 149);
  return neg ? -r : r;
}

static double exact_sum(const float* x, int64_t n, int absolute) {
  acc_t a;
  memset(&a, 0, sizeof a);
  for (int64_t i = 0; i < n; ++i) acc_add(&a, x[i], absolute);
  return acc_result(&a);
}

double oracle_sum_exact(const float* x, int64_t n) { return exact_sum(x, n, 0); }
double oracle_sum_abs_exact(const float* x, int64_t n) { return exact_sum(x, n, 1); }

/* The oracle's `sum`: the exact S rounded once to fp64 (reading R2/R3). */
static double fig1_sum(const float* data, int64_t n, uint64_t* adds) {
  if (adds) *adds += (uint64_t)n; /* one add per element: O(n) per call */
  return oracle_sum_exact(data, n);
}

/* out[tid] = in[tid] / val, quotient rounded once to fp32. */
static float fig1_div(float a, double val) { return (float)((double)a / val); }

/* ------------------------------------------------------------------- forms */

/* Form 1, as written: `float val = sum(in, n);` in every thread. */
int oracle_form_thread(float* out, const float* in, int64_t n, int mode, uint64_t* adds) {
  if (n < 0 || (n > 0 && (!out || !in)) || (n > 0 && out == in)) return 1;
  int64_t G = oracle_grid_blocks(n);
  for (int64_t b = 0; b < G; ++b)
    for (int64_t t = 0; t < FIG1_BLOCK; ++t) {
      double val = fig1_sum(in, n, adds);
      int64_t tid = oracle_tid(b, t, mode);
      if (tid < n) out[tid] = fig1_div(in[tid], val);
    }
  return 0;
}

/* Form 2, the commented per-block variant:
 *   __shared__ val; if (threadIdx.x == 0) val = sum(in, n); __syncthreads();  */
int oracle_form_block(float* out, const float* in, int64_t n, int mode, uint64_t* adds) {
  if (n < 0 || (n > 0 && (!out || !in)) || (n > 0 && out == in)) return 1;
  int64_t G = oracle_grid_blocks(n);
  for (int64_t b = 0; b < G; ++b) {
    double val = fig1_sum(in, n, adds); /* thread 0 of block b, then barrier */
    for (int64_t t = 0; t < FIG1_BLOCK; ++t) {
      int64_t tid = oracle_tid(b, t, mode);
      if (tid < n) out[tid] = fig1_div(in[tid], val);
    }
  }
  return 0;
}

/* Form 3, after parallel LICM: `sum` hoisted before the launch (PAPER.md:117,
 * 226-230, 592-598).  out == in is allowed under the paper's lock-step reading
 * (every thread executes instruction k before any thread executes
 * instruction k+1), so every load of in[tid] precedes every store to out[tid];
 * the literal index writes an element up to 32 times, so an in-place run reads
 * from a snapshot of `in` (reading R9). */
int oracle_form_hoisted(float* out, const float* in, int64_t n, int mode, uint64_t* adds) {
  if (n < 0 || (n > 0 && (!out || !in))) return 1;
  if (n == 0) return 0;
  float* snapshot = NULL;
  if (out == in) {
    snapshot = (float*)malloc((size_t)n * sizeof(float));
    if (!snapshot) return 2;
    memcpy(snapshot, in, (size_t)n * sizeof(float));
    in = snapshot;
  }
  double val = fig1_sum(in, n, adds);
  int64_t G = oracle_grid_blocks(n);
  for (int64_t b = 0; b < G; ++b)
    for (int64_t t = 0; t < FIG1_BLOCK; ++t) {
      int64_t tid = oracle_tid(b, t, mode);
      if (tid < n) out[tid] = fig1_div(in[tid], val);
    }
  free(snapshot);
  return 0;
}

/* Form 3 on T host threads, for timing the oracle on all of the host's cores
 * (the cpu_baseline of bench.py).  Same arithmetic as
 * oracle_form_hoisted: thread k accumulates the contiguous chunk
 * [k n / T, (k+1) n / T) of `in` EXACTLY into its own superaccumulator; the T
 * accumulators are merged in chunk order (integer limb addition: exact, so the
 * merged value is the exact sum of all n terms whatever T is) and rounded once
 * to fp64 -> val.  After a join (every load of the sum precedes every store,
 * PAPER.md:598), thread k writes out[i] = in[i] / val for the covered i of its
 * chunk (i in C(n) <=> some (b, t) of the launch has tid == i, PAPER.md:103,
 * 109, 113).  Bit-identical to oracle_form_hoisted for every T (pinned). */
typedef struct {
  const float* in;
  float* out;
  int64_t lo, hi, n;
  int mode;
  double val;
  acc_t acc;
} mt_task_t;

static void* mt_sum(void* arg) {
  mt_task_t* k = (mt_task_t*)arg;
  memset(&k->acc, 0, sizeof k->acc);
  for (int64_t i = k->lo; i < k->hi; ++i) acc_add(&k->acc, k->in[i], 0);
  acc_norm(&k->acc);
  return NULL;
}

static void* mt_scale(void* arg) {
  mt_task_t* k = (mt_task_t*)arg;
  for (int64_t i = k->lo; i < k->hi; ++i)
    if (oracle_is_covered(k->n, k->mode, i)) k->out[i] = fig1_div(k->in[i], k->val);
  return NULL;
}

static int mt_run(mt_task_t* t, int T, void* (*fn)(void*)) {
  pthread_t th[256];
  int started = 0, rc = 0;
  for (int k = 1; k < T; ++k) {
    if (pthread_create(&th[k], NULL, fn, &t[k]) != 0) { rc = 3; break; }
    started = k;
  }
  if (rc) { /* could not start every thread: run the rest here */
    for (int k = started + 1; k < T; ++k) fn(&t[k]);
    rc = 0;
  }
  fn(&t[0]);
  for (int k = 1; k <= started; ++k) pthread_join(th[k], NULL);
  return rc;
}

int oracle_form_hoisted_mt(float* out, const float* in, int64_t n, int mode, int threads,
                           uint64_t* adds) {
  if (n < 0 || (n > 0 && (!out || !in)) || threads < 1 || threads > 256) return 1;
  if (n == 0) return 0;
  mt_task_t* t = (mt_task_t*)calloc((size_t)threads, sizeof(mt_task_t));
  if (!t) return 2;
  for (int k = 0; k < threads; ++k) {
    t[k].in = in;
    t[k].out = out;
    t[k].lo = n * k / threads;
    t[k].hi = n * (k + 1) / threads;
    t[k].n = n;
    t[k].mode = mode;
  }
  mt_run(t, threads, mt_sum);
  acc_t all;
  memset(&all, 0, sizeof all);
  for (int k = 0; k < threads; ++k) { /* chunk order; exact integer addition */
    for (int j = 0; j < ACC_LIMBS; ++j) all.limb[j] += t[k].acc.limb[j];
    all.nposinf += t[k].acc.nposinf;
    all.nneginf += t[k].acc.nneginf;
    all.nnan += t[k].acc.nnan;
    all.nterms += t[k].acc.nterms;
    all.nnegzero += t[k].acc.nnegzero;
  }
  if (adds) *adds += (uint64_t)n;
  const double val = acc_result(&all);
  for (int k = 0; k < threads; ++k) t[k].val = val;
  mt_run(t, threads, mt_scale);
  free(t);
  return 0;
}

/* The exact sum of x[0, n) on T threads (same chunking and exact merge as
 * oracle_form_hoisted_mt), correctly rounded to fp64: == oracle_sum_exact. */
double oracle_sum_exact_mt(const float* x, int64_t n, int threads) {
  if (n <= 0) return 0.0;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  mt_task_t* t = (mt_task_t*)calloc((size_t)threads, sizeof(mt_task_t));
  if (!t) return oracle_sum_exact(x, n);
  for (int k = 0; k < threads; ++k) {
    t[k].in = x;
    t[k].lo = n * k / threads;
    t[k].hi = n * (k + 1) / threads;
  }
  mt_run(t, threads, mt_sum);
  acc_t all;
  memset(&all, 0, sizeof all);
  for (int k = 0; k < threads; ++k) {
    for (int j = 0; j < ACC_LIMBS; ++j) all.limb[j] += t[k].acc.limb[j];
    all.nposinf += t[k].acc.nposinf;
    all.nneginf += t[k].acc.nneginf;
    all.nnan += t[k].acc.nnan;
    all.nterms += t[k].acc.nterms;
    all.nnegzero += t[k].acc.nnegzero;
  }
  free(t);
  return acc_result(&all);
}

/* Exact per-row sums (the oracle's `sum` of each row, reading R10): S[r] = the
 * exact sum of row r, correctly rounded to fp64. */
int oracle_rows_sum_exact(double* S, const float* in, int64_t rows, int64_t cols, int64_t ld) {
  if (rows < 0 || cols < 0 || ld < cols || (rows > 0 && (!S || (cols > 0 && !in)))) return 1;
  for (int64_t r = 0; r < rows; ++r) S[r] = oracle_sum_exact(in + r * ld, cols);
  return 0;
}

int oracle_rows(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                int64_t ld_in, int mode) {
  if (rows < 0 || cols < 0 || ld_out < cols || ld_in < cols) return 1;
  for (int64_t r = 0; r < rows; ++r) {
    int rc = oracle_form_hoisted(out + r * ld_out, in + r * ld_in, cols, mode, NULL);
    if (rc) return rc;
  }
  return 0;
}

int oracle_replay(float* out, const float* in, int64_t n, int mode, float s) {
  if (n < 0 || (n > 0 && (!out || !in))) return 1;
  for (int64_t i = 0; i < n; ++i)
    if (oracle_is_covered(n, mode, i)) out[i] = in[i] / s; /* binary32 RN */
  return 0;
}

/* ================================================================ NEXT-2
 * Row softmax / log-softmax and ClassNLLCriterion (the PyTorch
 * CUDA kernels MocCUDA transpiles: "aggregation operations like Softmax" and the
 * NLL loss that uses __syncthreads).  Textbook definitions in fp64. */

static int rowop_args(int64_t rows, int64_t cols, int64_t ld_out, int64_t ld_in, const void* a,
                      const void* b) {
  if (rows < 0 || cols < 0 || ld_out < cols || ld_in < cols) return 1;
  if (rows > 0 && cols > 0 && (!a || !b)) return 1;
  return 0;
}

/* max over the row; NaN if any element is NaN (IEEE maximum propagating NaN). */
static double row_max(const float* x, int64_t cols) {
  double m = -INFINITY;
  for (int64_t i = 0; i < cols; ++i) {
    if (isnan(x[i])) return NAN;
    if ((double)x[i] > m) m = (double)x[i];
  }
  return m;
}

int oracle_softmax_rows(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                        int64_t ld_in) {
  if (rowop_args(rows, cols, ld_out, ld_in, out, in)) return 1;
  for (int64_t r = 0; r < rows; ++r) {
    const float* x = in + r * ld_in;
    float* y = out + r * ld_out;
    const double m = row_max(x, cols);
    double S = 0.0;
    for (int64_t i = 0; i < cols; ++i) S += exp((double)x[i] - m);
    for (int64_t i = 0; i < cols; ++i) y[i] = (float)(exp((double)x[i] - m) / S);
  }
  return 0;
}

int oracle_log_softmax_rows(float* out, const float* in, int64_t rows, int64_t cols,
                            int64_t ld_out, int64_t ld_in) {
  if (rowop_args(rows, cols, ld_out, ld_in, out, in)) return 1;
  for (int64_t r = 0; r < rows; ++r) {
    const float* x = in + r * ld_in;
    float* y = out + r * ld_out;
    const double m = row_max(x, cols);
    double S = 0.0;
    for (int64_t i = 0; i < cols; ++i) S += exp((double)x[i] - m);
    const double lse = log(S);
    for (int64_t i = 0; i < cols; ++i) y[i] = (float)(((double)x[i] - m) - lse);
  }
  return 0;
}

int oracle_nll_forward(double* loss, double* total_weight, const float* logp, const int64_t* target,
                       const float* weight, int64_t N, int64_t C, int64_t ld, int reduction,
                       int64_t ignore_index) {
  if (N < 0 || C < 1 || ld < C || !loss || !total_weight || (N > 0 && (!logp || !target))) return 1;
  if (reduction < ORACLE_RED_NONE || reduction > ORACLE_RED_SUM) return 1;
  double num = 0.0, den = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    const int64_t t = target[i];
    double li;
    if (t == ignore_index) {
      li = 0.0;
    } else if (t < 0 || t >= C) {
      li = NAN;
    } else {
      const double w = weight ? (double)weight[t] : 1.0;
      li = -w * (double)logp[i * ld + t];
      den += w;
    }
    if (reduction == ORACLE_RED_NONE) loss[i] = li;
    num += li;
  }
  *total_weight = den;
  if (reduction == ORACLE_RED_SUM) loss[0] = num;
  if (reduction == ORACLE_RED_MEAN) loss[0] = num / den; /* 0/0 -> NaN when all ignored */
  return 0;
}

int oracle_nll_backward(double* grad, const double* grad_out, const int64_t* target,
                        const float* weight, double total_weight, int64_t N, int64_t C, int64_t ld,
                        int reduction, int64_t ignore_index) {
  if (N < 0 || C < 1 || ld < C || (N > 0 && (!grad || !grad_out || !target))) return 1;
  if (reduction < ORACLE_RED_NONE || reduction > ORACLE_RED_SUM) return 1;
  for (int64_t i = 0; i < N; ++i) {
    for (int64_t c = 0; c < C; ++c) grad[i * ld + c] = 0.0;
    const int64_t t = target[i];
    if (t == ignore_index || t < 0 || t >= C) continue;
    const double w = weight ? (double)weight[t] : 1.0;
    const double g = grad_out[reduction == ORACLE_RED_NONE ? i : 0];
    grad[i * ld + t] = -w * g / (reduction == ORACLE_RED_MEAN ? total_weight : 1.0);
  }
  return 0;
}

/* ------------------------------------------------------------ gradients
 * For PyTorch autograd of the forward ops above (the training the paper runs
 * through MocCUDA).  Plain derivatives, fp64 in and out.
 *
 * normalize (functional form y = normalize(x): covered y_i = x_i / S with
 * S = sum_{k<n} x_k; uncovered y_j = x_j): with g = dL/dy and
 * y_i = x_i / S,  dy_i/dx_j = [i == j]/S - x_i/S^2 for i in C(n), so
 *   gx_j = [j in C] g_j / S + [j not in C] g_j - D,   D = sum_{i in C} g_i y_i / S. */
int oracle_normalize_backward(double* gx, const double* g, const double* y, double S, int64_t n,
                              int mode) {
  if (n < 0 || (n > 0 && (!gx || !g || !y))) return 1;
  double D = 0.0;
  for (int64_t i = 0; i < n; ++i)
    if (oracle_is_covered(n, mode, i)) D += g[i] * y[i];
  D /= S;
  for (int64_t j = 0; j < n; ++j) gx[j] = (oracle_is_covered(n, mode, j) ? g[j] / S : g[j]) - D;
  return 0;
}

/* softmax: y = exp(x - m) / sum exp(x - m)  ->  gx_j = y_j (g_j - sum_k g_k y_k);
 * log-softmax: y = x - m - log sum exp(x - m)  ->  gx_j = g_j - exp(y_j) sum_k g_k. */
int oracle_softmax_backward_rows(double* gx, const double* g, const double* y, int64_t rows,
                                 int64_t cols, int log_softmax) {
  if (rows < 0 || cols < 0 || (rows > 0 && cols > 0 && (!gx || !g || !y))) return 1;
  for (int64_t r = 0; r < rows; ++r) {
    const double* gr = g + r * cols;
    const double* yr = y + r * cols;
    double D = 0.0;
    for (int64_t k = 0; k < cols; ++k) D += log_softmax ? gr[k] : gr[k] * yr[k];
    for (int64_t j = 0; j < cols; ++j)
      gx[r * cols + j] = log_softmax ? gr[j] - exp(yr[j]) * D : yr[j] * (gr[j] - D);
  }
  return 0;
}

/* ================================================================ NEXT-4
 * bpnn_layerforward of Rodinia backprop as printed in Fig. backprop
 * (PAPER.md:553-579).  The printed listing elides the index expressions and
 * garbles the tree condition (`if( ty ` ...); reading R18 takes them from the
 * Rodinia kernel the figure reproduces: index = (hid+1)*HEIGHT*by + (hid+1)*ty
 * + tx + 1 + (hid+1), index_in = HEIGHT*by + ty + 1, condition ty % 2^i == 0.
 * Executed block by block; within a block every phase between barriers runs
 * for all threads before the next (the barrier semantics of PAPER.md:314-351). */
#define BP_H 16
int oracle_bpnn_layerforward(const float* input, float* hidden, float* output, int64_t in,
                             int64_t hid) {
  if (hid != BP_H || in < 0 || in % BP_H || (in > 0 && (!input || !hidden || !output))) return 1;
  const int64_t blocks = in / BP_H;
  for (int64_t by = 0; by < blocks; ++by) {
    float node[BP_H], w[BP_H][BP_H];
    for (int ty = 0; ty < BP_H; ++ty) node[ty] = input[BP_H * by + ty + 1]; /* tx == 0 */
    for (int ty = 0; ty < BP_H; ++ty)
      for (int tx = 0; tx < BP_H; ++tx)
        w[ty][tx] = hidden[(hid + 1) * BP_H * by + (hid + 1) * ty + tx + 1 + (hid + 1)];
    for (int ty = 0; ty < BP_H; ++ty)
      for (int tx = 0; tx < BP_H; ++tx) w[ty][tx] = w[ty][tx] * node[ty];
    for (int i = 1; i <= 4; ++i) { /* log2(HEIGHT) steps */
      const int p = 1 << i;
      for (int ty = 0; ty < BP_H; ++ty)
        if (ty % p == 0)
          for (int tx = 0; tx < BP_H; ++tx) w[ty][tx] = w[ty][tx] + w[ty + p / 2][tx];
    }
    for (int ty = 0; ty < BP_H; ++ty)
      for (int tx = 0; tx < BP_H; ++tx)
        hidden[(hid + 1) * BP_H * by + (hid + 1) * ty + tx + 1 + (hid + 1)] = w[ty][tx];
    for (int ty = 0; ty < BP_H; ++ty) output[by * hid + ty] = w[0][ty]; /* tx == 0: weights[tx][ty] */
  }
  return 0;
}
