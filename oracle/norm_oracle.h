/*
 * oracle/norm_oracle.h — CPU oracle for Fig. 1 `normalize` (arxiv 2207.00257).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header or constant with the CUDA path (paper_2207_00257_b200/ and
 * include/), and the product path never calls it.
 *
 * Plain, slow, obviously-correct C in fp64 (plus an exact integer
 * superaccumulator).  Each function cites the passage it follows.  Readings of
 * the paper where it is silent/garbled are listed in DESIGN.md §3 (R1..R12).
 *
 * Parity status:
 *   coverage (brute + closed)  pinned: hand-derived golden cases, brute force.
 *   oracle_sum_exact           pinned: math.fsum, integer closed forms.
 *   forms thread/block/hoisted pinned: mutual bit agreement, op counts of
 *                              PAPER.md:117 / SPEC.md:617, 1/n, sum-to-1.
 *   oracle_replay              pinned: exact rational RN32 via fractions.
 *   the exact fp32 bits of the GPU divisor s: parity unpinned (any fp32
 *   within 1e-6 of S is correct; PAPER.md:100 elides `sum`).
 */
#ifndef NORM_ORACLE_H
#define NORM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_LITERAL = 0, ORACLE_DENSE = 1 };

/* Fig. 1 launch: normalize<<<(n+31)/32, 32>>>. */
int64_t oracle_grid_blocks(int64_t n);
/* Fig. 1 index: tid = blockIdx.x + blockDim.x * threadIdx.x [LITERAL];
 * the conventional blockIdx.x * blockDim.x + threadIdx.x [DENSE, reading R1]. */
int64_t oracle_tid(int64_t b, int64_t t, int mode);

/* Enumerate every (blockIdx, threadIdx) of the launch; mult[tid]++ for tid < n. */
int oracle_coverage_brute(int64_t n, int mode, uint32_t* mult);
/* Closed form of the covered set C(n).  count = |C(n)|;
 * prefix_len = L if C(n) == [0, L), else -1. */
int oracle_coverage_closed(int64_t n, int mode, int64_t* count, int64_t* prefix_len);
int oracle_is_covered(int64_t n, int mode, int64_t i);

/* Sequential fp64 sum in index order (reading R2 of the elided `sum`). */
double oracle_sum_seq(const float* x, int64_t n);
/* Exact sum of the n fp32 values, correctly rounded to fp64 (superaccumulator).
 * Non-finite classification follows a plain IEEE sum (reading R7). */
double oracle_sum_exact(const float* x, int64_t n);
/* Exact sum of |x_i|, correctly rounded to fp64 (tolerance scale for signed inputs). */
double oracle_sum_abs_exact(const float* x, int64_t n);

/* The three forms of Fig. 1 (PAPER.md:100-114 and caption 117).  out != in is
 * required for forms 1 and 2 (reading R9); *adds receives the number of
 * additions performed by `sum` calls.  Return 0 ok, nonzero on bad arguments. */
int oracle_form_thread(float* out, const float* in, int64_t n, int mode, uint64_t* adds);
int oracle_form_block(float* out, const float* in, int64_t n, int mode, uint64_t* adds);
int oracle_form_hoisted(float* out, const float* in, int64_t n, int mode, uint64_t* adds);

/* Form 3 on `threads` host threads (1..256): contiguous chunks accumulated
 * exactly, merged in chunk order, one rounding -> bit-identical to
 * oracle_form_hoisted.  For timing the oracle on all host cores (cpu_baseline). */
int oracle_form_hoisted_mt(float* out, const float* in, int64_t n, int mode, int threads,
                           uint64_t* adds);
/* The exact sum on `threads` threads (exact merge): == oracle_sum_exact. */
double oracle_sum_exact_mt(const float* x, int64_t n, int threads);
/* S[r] = exact sum of row r (in[r*ld + 0 .. cols)), correctly rounded to fp64. */
int oracle_rows_sum_exact(double* S, const float* in, int64_t rows, int64_t cols, int64_t ld);

/* Batched variant (reading R10): row r == oracle_form_hoisted on row r. */
int oracle_rows(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                int64_t ld_in, int mode);

/* Replay given a divisor s: out[i] = in[i] / s in binary32 RN for i in C(n). */
int oracle_replay(float* out, const float* in, int64_t n, int mode, float s);

/* ---- the PyTorch kernels the paper transpiles next to
 * normalize — "aggregation operations like Softmax" and ClassNLLCriterion
 * (PAPER.md:747-750).  fp64 throughout; parity pins in tests/test_oracle_rowops.py. */

/* Row softmax: out = exp(x - max) / sum exp(x - max), fp64, then rounded once. */
int oracle_softmax_rows(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                        int64_t ld_in);
/* Row log-softmax: out = (x - max) - log(sum exp(x - max)). */
int oracle_log_softmax_rows(float* out, const float* in, int64_t rows, int64_t cols,
                            int64_t ld_out, int64_t ld_in);

enum { ORACLE_RED_NONE = 0, ORACLE_RED_MEAN = 1, ORACLE_RED_SUM = 2 };
/* ClassNLLCriterion_updateOutput: per sample i with t = target[i] != ignore_index,
 * l_i = -w[t] * logp[i*ld + t] (w = 1 without weights).  NONE: loss[i] = l_i (0 if
 * ignored); SUM: loss[0] = sum l_i; MEAN: loss[0] = sum l_i / sum w[t_i] (NaN if
 * the weight sum is 0).  *total_weight = sum w[t_i].  A target outside [0, C) that
 * is not ignore_index gives NaN (reading R17). */
/* Gradients (fp64): y = normalize(x) in its functional form (uncovered y_j = x_j),
 * given g = dL/dy, y and S: gx_j = [j in C] g_j / S + [j not in C] g_j - sum_{i in C} g_i y_i / S. */
int oracle_normalize_backward(double* gx, const double* g, const double* y, double S, int64_t n,
                              int mode);
/* softmax: gx = y (g - sum g y); log-softmax: gx = g - exp(y) sum g (rows x cols, contiguous). */
int oracle_softmax_backward_rows(double* gx, const double* g, const double* y, int64_t rows,
                                 int64_t cols, int log_softmax);
int oracle_nll_forward(double* loss, double* total_weight, const float* logp, const int64_t* target,
                       const float* weight, int64_t N, int64_t C, int64_t ld, int reduction,
                       int64_t ignore_index);
/* ClassNLLCriterion_updateGradInput: grad[i*ld + c] = 0 except
 * grad[i*ld + t_i] = -w[t_i] * g_i / (MEAN ? total_weight : 1), g_i = grad_out[NONE ? i : 0]. */
int oracle_nll_backward(double* grad, const double* grad_out, const int64_t* target,
                        const float* weight, double total_weight, int64_t N, int64_t C, int64_t ld,
                        int reduction, int64_t ignore_index);

/* ---- Rodinia backprop bpnn_layerforward (Fig. backprop,
 * PAPER.md:549-584), HEIGHT = WIDTH = hid = 16, in a multiple of 16 (reading R18).
 * Step by step in binary32 with the printed statement order and the printed
 * shared-memory tree (no contraction):
 *   node[ty] = input[16 by + ty + 1]
 *   w[ty][tx] = hidden[17 (16 by + ty + 1) + tx + 1] * node[ty]
 *   for i = 1..4: if (ty % 2^i == 0) w[ty][tx] += w[ty + 2^(i-1)][tx]
 *   hidden[...] = w[ty][tx];   output[16 by + ty] = w[0][ty]
 * input: fp32[in + 1]; hidden: fp32[(in + 1) * 17] (in/out); output: fp32[in]. */
int oracle_bpnn_layerforward(const float* input, float* hidden, float* output, int64_t in,
                             int64_t hid);

#ifdef __cplusplus
}
#endif
#endif
