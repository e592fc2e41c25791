/*
 * include/libnorm.h — C ABI of libnorm: Fig. 1 `normalize` of arxiv 2207.00257
 * ("High-Performance GPU-to-CPU Transpilation and Optimization via High-Level
 * Parallel Constructs") after parallel loop-invariant code motion, on B200
 * (sm_100a).
 *
 * The operation (Fig. 1, and §2.1):
 *
 *     __global__ void normalize(float *out, float* in, int n) {
 *       int tid = blockIdx.x + blockDim.x * threadIdx.x;
 *       float val = sum(in, n);
 *       if (tid < n) out[tid] = in[tid] / val;
 *     }
 *     void launch(... d_out, ... d_in, int n) {
 *       normalize<<<(n+31)/32, 32>>>(d_out, d_in, n);
 *     }
 *
 * with `sum` (elided at PAPER.md:100) hoisted out of the kernel by parallel LICM
 * (PAPER.md:117, 592-598), so every call is:  S = sum_{i<n} in[i] (one global
 * reduction over ALL n elements), then out[i] = in[i] / s for every i in the
 * covered set C(n) of the launch, where s is an fp32 within 1e-6 relative of S.
 * Elements outside C(n) are left untouched.
 *
 * Coverage C(n), G = ceil(n/32):
 *   NORM_INDEX_LITERAL (default; tid = b + 32 t as printed at PAPER.md:103):
 *       G >= 32: C(n) = [0, min(n, G + 992))
 *       G <  32: C(n) = { x < n : x mod 32 < G }
 *   NORM_INDEX_DENSE (tid = 32 b + t, the caption's "normalizes a vector"):
 *       C(n) = [0, n)
 * The readings taken where the paper is silent are DESIGN.md §3 (R1..R15).
 *
 * Conventions for every entry point:
 *   - returns norm_status_t; never aborts, throws or prints.  norm_last_error()
 *     returns a thread-local detail string for the last failing call.
 *   - device entries are stream-ordered and return after enqueue, like the
 *     kernel launch of Fig. 1; asynchronous device faults surface at the
 *     caller's next synchronisation.  They never synchronise the device.
 *   - the caller owns all memory it passes (in, out, sum_out*, workspace);
 *     libnorm never frees caller memory.  Pointers are device pointers unless
 *     the name says `host`.  Float pointers must be 4-byte aligned.
 *   - `out == in` (exact alias) is allowed (reading R9: all loads of `in`
 *     precede every store under the paper's lock-step semantics);
 *     partial overlap returns NORM_ERR_OVERLAP.
 *   - n == 0 (or rows == 0 / cols == 0) is a no-op returning NORM_OK (R8).
 *   - a zero or non-finite sum is not an error: IEEE results (R7).
 *   - results are bitwise deterministic run to run for the same arguments
 *     (same n, index mode, path, pointer alignment mod 32 B and world size).
 */
#ifndef LIBNORM_H
#define LIBNORM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LIBNORM_VERSION_MAJOR 0
#define LIBNORM_VERSION_MINOR 1

typedef enum {
  NORM_OK = 0,
  NORM_ERR_INVALID_VALUE = 1, /* n < 0, NULL with work to do, misaligned, bad enum, ld < cols */
  NORM_ERR_OVERLAP = 2,       /* out and in overlap without being identical */
  NORM_ERR_CUDA = 3,          /* CUDA runtime / launch error (detail in norm_last_error) */
  NORM_ERR_NCCL = 4,          /* NCCL error */
  NORM_ERR_WORKSPACE = 5,     /* caller workspace too small, or device allocation failed */
  NORM_ERR_UNSUPPORTED = 6    /* not an sm_100 device, or literal grid > 2^31-1 blocks */
} norm_status_t;

typedef enum {
  NORM_INDEX_LITERAL = 0, /* Fig. 1 as printed: tid = blockIdx.x + blockDim.x*threadIdx.x */
  NORM_INDEX_DENSE = 1    /* tid = blockIdx.x*blockDim.x + threadIdx.x: all of [0, n)      */
} norm_index_t;

typedef enum {
  NORM_PATH_AUTO = 0,     /* small n: small; L2-sized: mid; input > L2 but covered prefix
                             fits: fused; else two-pass                    */
  NORM_PATH_TWO_PASS = 1, /* reduce kernel, then scale kernel (PDL-chained)               */
  NORM_PATH_FUSED = 2,    /* one cooperative kernel: reduce, grid barrier, scale from L2  */
  NORM_PATH_SMALL = 3,    /* one CTA does everything (any n; intended for n <= 2^17)       */
  NORM_PATH_MID = 4,      /* one cooperative kernel of 256-bit-load CTAs, one per SM:
                             reduce, grid barrier, scale (L2-sized inputs)                 */
  NORM_PATH_CLUSTER = 5   /* one thread-block cluster (16 CTAs): reduce, DSMEM combine,
                             scale -- no workspace (L2-sized inputs, e.g. 2^20 + 7)        */
} norm_path_t;

/* Options of every device entry point.  `index` and `path` carry norm_index_t /
 * norm_path_t values but are declared int32_t: the width of a C enum is
 * implementation-defined, and a fixed-width field keeps this struct's layout
 * identical for every compiler and FFI (ctypes, Rust, ...).  Out-of-range values
 * return NORM_ERR_INVALID_VALUE. */
typedef struct {
  void* stream;         /* cudaStream_t to enqueue on; NULL = legacy default stream       */
  int32_t index;        /* norm_index_t value, default NORM_INDEX_LITERAL                  */
  int32_t path;         /* norm_path_t value, default NORM_PATH_AUTO                       */
  float* sum_out;       /* optional device ptr: receives s, the fp32 divisor used.
                           norm_rows: array of `rows` floats, one divisor per row          */
  double* sum_out_f64;  /* optional device ptr: receives S as accumulated (fp64).
                           norm_rows: array of `rows` doubles                              */
  void* workspace;      /* optional caller-owned device scratch (>= norm_workspace_bytes),
                           zero-filled before its first use; libnorm leaves it reusable.
                           NULL = an internal cache keyed by (device, stream).  Calls that
                           may run concurrently must not share a workspace.                */
  size_t workspace_bytes;
  uint32_t flags;       /* NORM_FLAG_* bits; 0 = all checks                                */
  uint32_t reserved;    /* must be 0                                                       */
} norm_opts_t;

/* The caller guarantees that every pointer it passes (in, out, sum_out,
 * sum_out_f64) is device memory of the CURRENT device.  libnorm then skips its
 * per-pointer cudaPointerGetAttributes checks (about 0.3-1 us of host time
 * each; they exist to turn a host pointer into NORM_ERR_INVALID_VALUE instead of
 * a sticky device fault).  For launch-bound callers (configs 1-2: n = 1024,
 * 2^20 + 7).  A wrong pointer under this flag is a device fault. */
#define NORM_FLAG_TRUSTED_PTRS 1u

/* Designated defaults: literal index, AUTO path, default stream, no outputs. */
#define NORM_OPTS_INIT {NULL, NORM_INDEX_LITERAL, NORM_PATH_AUTO, NULL, NULL, NULL, 0, 0u, 0u}

/* ---------------------------------------------------------------- vector */

/* Fig. 1 `launch(d_out, d_in, n)` after LICM: literal index,
 * legacy default stream, AUTO path.  out, in: device fp32[n]. */
norm_status_t norm_launch(float* out, const float* in, int64_t n);

/* As norm_launch with options (NULL o = NORM_OPTS_INIT). */
norm_status_t norm_launch_ex(float* out, const float* in, int64_t n, const norm_opts_t* o);

/* A call captured once as a CUDA graph (its 1-2 kernels and their programmatic
 * dependency) with its own workspace; every norm_graph_launch replays it on
 * `stream` with one cudaGraphLaunch (launch-bound sizes: ~1 host launch instead
 * of two).  Pointers, n and opts are fixed at creation (o->stream and the event
 * fields are ignored).  Launches of one graph must be stream-ordered with
 * respect to each other (they share the workspace). */
typedef struct norm_graph norm_graph_t;
norm_status_t norm_graph_create(norm_graph_t** graph, float* out, const float* in, int64_t n,
                                const norm_opts_t* o);
norm_status_t norm_graph_launch(norm_graph_t* graph, void* stream);
norm_status_t norm_graph_destroy(norm_graph_t* graph);

/* End-to-end variant on HOST buffers: out_host/in_host are host fp32[n] (pinned
 * memory gives asynchronous, overlapped copies; pageable memory works but the
 * copies serialise).  libnorm streams `in` to the device in chunks, reduces each
 * chunk as it lands, keeps only the covered elements resident, scales them and
 * copies back only out_host[C(n)] — uncovered host outputs are untouched.
 * Enqueued on o->stream; the caller synchronises that stream before reading
 * out_host.  o->workspace is ignored (device staging is internal, per stream).
 * Same s bit-for-bit as long as the chunk partition is unchanged. */
norm_status_t norm_launch_host(float* out_host, const float* in_host, int64_t n,
                               const norm_opts_t* o);

/* ------------------------------------------------ before LICM (NEXT-1) */

typedef enum {
  NORM_FORM_HOISTED = 0,    /* after parallel LICM: one O(N) sum (== norm_launch_ex)      */
  NORM_FORM_PER_BLOCK = 1,  /* thread 0 of each block sums, O(N^2/B)    */
  NORM_FORM_PER_THREAD = 2  /* PAPER.md:108, as printed: every thread sums, O(N^2)        */
} norm_form_t;

/* Fig. 1 in the given form, for timing the LICM before/after on the GPU
 * (PAPER.md:117, 226-228).  The un-hoisted forms run the printed launch
 * normalize<<<(n+31)/32, 32>>> with the index of o->index and a sequential fp64
 * `sum` in every summing thread; o->path is ignored for them.  out == in is
 * rejected for the un-hoisted forms (they race as printed; reading R9), and
 * n > 2^24 is rejected for them (NORM_ERR_UNSUPPORTED: O(N^2) work). */
norm_status_t norm_launch_form(float* out, const float* in, int64_t n, int32_t form,
                               const norm_opts_t* o);

/* ------------------------------------------------------------------ rows */

/* Batched per-row variant (reading R10; BASELINE configs[4]): for each row r,
 * out[r*ld_out + i] = in[r*ld_in + i] / s_r for i in C(cols), s_r ~ sum of row r.
 * Row r is exactly norm_launch_ex(out + r*ld_out, in + r*ld_in, cols, o).
 * o->sum_out / sum_out_f64, when set, receive one value per row.  o->workspace
 * holds the row queue (CTAs take rows dynamically; each row's result does not
 * depend on which CTA computes it). */
norm_status_t norm_rows(float* out, const float* in, int64_t rows, int64_t cols,
                        int64_t ld_out, int64_t ld_in, const norm_opts_t* o);

/* ------------------------------------------- row ops (NEXT-2) */
/* The PyTorch CUDA kernels the paper transpiles beside normalize: "aggregation
 * operations like Softmax" and ClassNLLCriterion.  Same
 * conventions as above; o->stream / o->workspace are used, the other opts fields
 * are ignored.  Tolerances: DESIGN.md §9. */

typedef enum { NORM_SOFTMAX = 0, NORM_LOG_SOFTMAX = 1 } norm_softmax_t;

/* out[r, i] = exp(x - m_r) / sum_j exp(x_j - m_r)  (softmax), or
 * (x - m_r) - log(sum_j exp(x_j - m_r))             (log-softmax), m_r = max of row r.
 * A row containing NaN gives NaN; rows are [rows][ld], ld >= cols; out == in with
 * equal ld is allowed (in place); partial overlap -> NORM_ERR_OVERLAP. */
norm_status_t norm_softmax_rows(float* out, const float* in, int64_t rows, int64_t cols,
                                int64_t ld_out, int64_t ld_in, int32_t kind,
                                const norm_opts_t* o);

typedef enum { NORM_REDUCTION_NONE = 0, NORM_REDUCTION_MEAN = 1, NORM_REDUCTION_SUM = 2 } norm_reduction_t;

/* ClassNLLCriterion_updateOutput.  logp: [N][ld] log-probabilities, target: int64[N],
 * weight: optional fp32[C] (NULL = 1).  Sample i with t = target[i] != ignore_index
 * contributes l_i = -w[t] * logp[i, t]; a target outside [0, C) that is not
 * ignore_index contributes NaN (reading R17).  NONE: loss[i] = l_i (0 if ignored),
 * loss is fp32[N]; SUM / MEAN: loss[0] = sum l_i (/ sum w[t_i]).  total_weight
 * (optional, fp32[1]) = sum w[t_i].  Deterministic (fixed-order fp64 reduction). */
norm_status_t norm_nll_forward(float* loss, float* total_weight, const float* logp,
                               const int64_t* target, const float* weight, int64_t N, int64_t C,
                               int64_t ld, int32_t reduction, int64_t ignore_index,
                               const norm_opts_t* o);

/* ClassNLLCriterion_updateGradInput: writes the whole [N][ld] grad (cols [0, C)):
 * zeros except grad[i, t_i] = -w[t_i] * g_i / (MEAN ? *total_weight : 1), with
 * g_i = grad_out[NONE ? i : 0].  total_weight (device fp32[1]) is required for MEAN. */
norm_status_t norm_nll_backward(float* grad, const float* grad_out, const int64_t* target,
                                const float* weight, const float* total_weight, int64_t N,
                                int64_t C, int64_t ld, int32_t reduction, int64_t ignore_index,
                                const norm_opts_t* o);

/* ------------------------------------------- gradients (autograd of the ops above)
 * The paper runs PyTorch training through its transpiled kernels (MocCUDA,
 * PAPER.md:710-753); these are the backward passes of the forward entries, used
 * by the torch.library ops' autograd.  Each is one fp64 reduction (fixed order,
 * bit-identical run to run) and one elementwise fp32 pass.  g = dL/dy, y = the
 * forward's output; gx may be g or y itself (exact alias), partial overlap of gx
 * with g or y -> NORM_ERR_OVERLAP.  All pointers are device memory of the current
 * device; stream-ordered on o->stream like the forward calls.
 *
 * Functional normalize, y = x with y[C(n)] = x[C(n)] / s (the forward on a copy
 * of x, or in place; o->index selects C(n)), s = the forward's divisor (device
 * fp32[1], e.g. its sum_out), PAPER.md:108-110:
 *   gx_j = ([j in C] ? g_j / s : g_j) - D,   D = sum_{i in C} g_i y_i / s. */
norm_status_t norm_launch_backward(float* gx, const float* g, const float* y, const float* s,
                                   int64_t n, const norm_opts_t* o);
/* The same per row of a [rows][ld] matrix (C(cols) per row), s = fp32[rows] divisors
 * (norm_rows's sum_out). */
norm_status_t norm_rows_backward(float* gx, const float* g, const float* y, const float* s,
                                 int64_t rows, int64_t cols, int64_t ld, const norm_opts_t* o);
/* Row softmax: gx = y (g - sum_k g_k y_k); log-softmax (kind NORM_LOG_SOFTMAX):
 * gx = g - exp(y) sum_k g_k.  [rows][ld] matrices (PyTorch's _softmax_backward_data). */
norm_status_t norm_softmax_rows_backward(float* gx, const float* g, const float* y, int64_t rows,
                                         int64_t cols, int64_t ld, int32_t kind,
                                         const norm_opts_t* o);

/* ------------------------------- backprop layerforward (NEXT-4) */
typedef enum {
  NORM_BP_PRINTED = 0,     /* Fig. backprop as printed: shared memory, 8 barriers             */
  NORM_BP_ELIMINATED = 1,  /* §4.1/§4.2 by hand: barriers #1, #2 removed, store/load forwarded */
  NORM_BP_REGISTER = 2,    /* one thread per (block, column), tree in registers, 0 barriers    */
  NORM_BP_TMA = 3          /* REGISTER's arithmetic on tiles streamed by TMA (runs of 15
                              blocks + their inputs, 4-stage ring, 2 CTAs/SM, run queue)     */
} norm_bp_variant_t;

/* Rodinia backprop bpnn_layerforward (the kernel of Fig. backprop):
 * for every 16-row block `by` of the input layer and column c < 16:
 *   w[ty][c] = hidden[(16 by + ty + 1)(hid + 1) + c + 1] * input[16 by + ty + 1]
 *   tree: for i = 1..4, rows ty % 2^i == 0 add row ty + 2^(i-1)   (fp32, this order)
 *   hidden[...] <- w[ty][c];  output[16 by + c] <- w[0][c]
 * input: device fp32[in + 1]; hidden: device fp32[(in + 1) * (hid + 1)], updated in
 * place as the Rodinia kernel does; output: device fp32[in].  hid must be 16 and in a
 * multiple of 16 (else NORM_ERR_UNSUPPORTED).  All variants are bitwise identical
 * (reading R18).  o->stream and o->workspace (the TMA form's run queue) are used. */
norm_status_t norm_bpnn_layerforward(const float* input, float* hidden, float* output, int64_t in,
                                     int64_t hid, int32_t variant, const norm_opts_t* o);

/* ------------------------------------------------------------ host-only */

/* Size of C(n) for the index mode; *prefix_len = L if C(n) == [0, L), else -1.
 * Pure host function (no CUDA call). */
norm_status_t norm_coverage(int64_t n, int32_t index, int64_t* count, int64_t* prefix_len);

/* Bytes of device workspace a call with (n, o) needs if the caller supplies one
 * (the per-CTA partials and queue counters of the reduce and
 * scale kernels; independent of n today).  Host-only. */
norm_status_t norm_workspace_bytes(int64_t n, const norm_opts_t* o, size_t* bytes);

/* The path (norm_path_t) a call takes on the CURRENT device: `requested` if not
 * AUTO, else the AUTO rule of DESIGN.md §4 for n elements whose covered set is
 * [0, covered_prefix) (covered_prefix = -1: not a prefix).  The sharded peer
 * path applies it per rank to the local buffer.  Reads the device's L2 size
 * (NORM_ERR_CUDA / NORM_ERR_UNSUPPORTED without an sm_100 device). */
norm_status_t norm_choose_path(int64_t n, int64_t covered_prefix, int32_t requested, int32_t* chosen);

/* Algorithmic HBM bytes of one call (the roofline numerator):
 * two-pass 4n + 8|C(n)|.  Pure host function. */
norm_status_t norm_algorithmic_bytes(int64_t n, int32_t index, int64_t* bytes);

/* --------------------------------------------------------- multi-GPU (NCCL) */
/* The paper's method has one cross-thread dependency, the hoisted `sum`
 * (PAPER.md:108, 117); sharded over W GPUs it becomes a local partial per rank
 * plus an exchange of those 8-byte partials.  The paper itself scales only by
 * MPI ranks under Horovod; the contiguous shards, the
 * coverage-balanced plan and the "one NCCL all-reduce of a scalar" are the
 * north_star's (BASELINE.json) and SURVEY.md §8(b)/(e)'s design, DESIGN.md §6. */

/* Opaque: owns an ncclComm_t on the device current at init, plus device scratch
 * for the per-rank partial sums. One process per GPU. */
typedef struct norm_comm norm_comm_t;

/* Global index ranges owned by one rank, in ascending order.  The rank's local
 * buffers hold its ranges concatenated in this order. */
typedef struct {
  int32_t nranges;  /* 0, 1 or 2 */
  int64_t begin[2];
  int64_t len[2];
} norm_shard_t;

/* Rank 0 creates the NCCL unique id (128 bytes); the caller broadcasts it
 * (the Python binding uses the torch.distributed store). */
norm_status_t norm_comm_unique_id(unsigned char id[128]);
/* Collective over all `world` ranks; binds to the current CUDA device. */
norm_status_t norm_comm_init(norm_comm_t** comm, int32_t world, int32_t rank,
                             const unsigned char id[128]);
norm_status_t norm_comm_destroy(norm_comm_t* comm);

/* How norm_launch_sharded exchanges the partials:
 *   NORM_COMM_ALLGATHER (default): ncclAllGather of the W fp64 partials, summed in
 *     rank order by every rank -> bit-identical s on all ranks, order pinned;
 *   NORM_COMM_ALLREDUCE: ncclAllReduce(sum) of the fp64 partial (the north_star's
 *     "NCCL all-reduce of a scalar"); NCCL's reduction order, identical on all
 *     ranks for a given communicator. */
typedef enum { NORM_COMM_ALLGATHER = 0, NORM_COMM_ALLREDUCE = 1 } norm_comm_mode_t;
norm_status_t norm_comm_set_mode(norm_comm_t* comm, int32_t mode);

/* Partition [0, n) over `world` ranks (pure host function; plan[world]);
 * SURVEY.md §8(e)(i)/(ii), north_star "partitioned ... by contiguous shards".
 * DENSE, or coverage_balanced == 0: one contiguous range per rank, boundaries
 * rounded to 8 elements.  LITERAL with coverage_balanced != 0 and a prefix
 * coverage [0, L): each rank gets a slice of [0, L) and a slice of [L, n), so
 * the post-collective scale work is balanced. */
norm_status_t norm_plan_shards(int64_t n, int32_t world, int32_t index,
                               int32_t coverage_balanced, norm_shard_t* plan);

/* Sharded normalize of a global vector of n_global elements: every rank calls it
 * with its own shard `mine` (from norm_plan_shards) and local buffers
 * in_local/out_local of sum(mine->len) elements.  Local reduce -> one NCCL
 * all-gather of an 8-byte partial per rank on o->stream -> fixed rank-order
 * combine (identical s on every rank) -> scale of the locally covered elements.
 * o->index selects the coverage of the GLOBAL index. */
norm_status_t norm_launch_sharded(norm_comm_t* comm, float* out_local, const float* in_local,
                                  const norm_shard_t* mine, int64_t n_global,
                                  const norm_opts_t* o);

/* The same path split in two so that any collective can carry the exchange
 * (e.g. torch.distributed, or a caller-fused kernel):
 *   norm_shard_partial: *partial (device fp64[1]) <- sum of in_local[0, n_local)
 *   <caller all-gathers the W partials, in rank order, into a device fp64[W]>
 *   norm_shard_finish:  s = RN32(partials[0] + ... + partials[W-1]) (rank order),
 *                       then the scale of the locally covered elements.
 * norm_launch_sharded == partial + ncclAllGather + finish.  opts as above. */
norm_status_t norm_shard_partial(double* partial, const float* in_local, int64_t n_local,
                                 const norm_opts_t* o);
norm_status_t norm_shard_finish(float* out_local, const float* in_local, const norm_shard_t* mine,
                                int64_t n_global, const double* partials, int32_t world,
                                const norm_opts_t* o);

/* Fused exchange over peer memory (no collective launch on the data path): the
 * reduce kernel's last CTA stores the rank's 8-byte partial straight into every
 * rank's mailbox (CUDA IPC mappings of device memory; NVLink/NVSwitch stores on a
 * multi-GPU box) and releases an epoch flag; the scale kernel's prologue waits
 * for all W flags of the epoch (acquire, system scope; ~30 s timeout gives s =
 * NaN instead of a hang) and combines the partials in rank order -- the same
 * bits as norm_launch_sharded.  Set-up (one process per GPU, collective):
 *   norm_peer_create -> 64-byte IPC handle of this rank's mailbox
 *   <caller all-gathers the W handles in rank order>
 *   norm_peer_connect(handles[W*64]) -> maps the peers' mailboxes
 * Calls on one norm_peer_t must be issued in the same order on every rank.
 * o->path: AUTO applies norm_choose_path per rank to the local buffer; FUSED (or
 * AUTO choosing it) runs ONE cooperative kernel per rank when the locally
 * covered elements are a prefix of the local buffer: reduce, grid barrier,
 * publish + mailbox wait, scale (the covered part read last, from L2 where it
 * fits); TWO_PASS (or a non-prefix local coverage) runs reduce -> scale.  Each
 * path is deterministic; their local partials differ only in summation order
 * (bit-identical whenever the fp64 accumulation is exact, e.g. grid-valued
 * inputs).
 * Failure: if a call fails after this rank's publishing kernel was enqueued, the
 * handle's epoch can no longer match its peers'; every later call on it returns
 * NORM_ERR_CUDA ("peer handle broken") instead of waiting -- destroy and
 * recreate the handles on every rank.  A call that fails before enqueueing
 * anything leaves the handle usable. */
typedef struct norm_peer norm_peer_t;
norm_status_t norm_peer_create(norm_peer_t** peer, int32_t world, int32_t rank,
                               unsigned char handle[64]);
norm_status_t norm_peer_connect(norm_peer_t* peer, const unsigned char* handles);
norm_status_t norm_peer_destroy(norm_peer_t* peer);
norm_status_t norm_launch_sharded_peer(norm_peer_t* peer, float* out_local, const float* in_local,
                                       const norm_shard_t* mine, int64_t n_global,
                                       const norm_opts_t* o);

/* -------------------------------------------------------- instrumentation */
/* Not part of the operation: for timing the dominant kernel (bench.py's
 * roofline).  begin / end are cudaEvent_t (or NULL).  Until called again, every
 * vector or sharded call made on THIS host thread records `begin` on its stream
 * immediately before its dominant kernel -- on two-pass paths the reduce, or on
 * one GPU the scale when it moves more algorithmic bytes (8|C| > 4n, e.g. the
 * dense index); the one kernel on the small, mid, cluster and fused paths -- and
 * `end` immediately after it.
 * (NULL, NULL) turns it off.  Ignored inside norm_graph_create. */
norm_status_t norm_debug_set_events(void* begin, void* end);

/* --------------------------------------------------------------- caches */
/* Frees libnorm's internal per-(device, stream) caches: the ~161 KB workspaces and
 * the norm_launch_host staging buffers (resident covered prefix, 3 x 128 MiB ring).
 * Synchronises every device that owns a cache entry.  Later calls re-create them.
 * Note for CUDA-graph capture: the internal workspace of a (device, stream) is
 * allocated on its first use, which is not capturable -- make one call on the
 * stream before capturing, or pass o->workspace. */
norm_status_t norm_cache_release(void);

/* -------------------------------------------------------------- errors */
const char* norm_status_string(norm_status_t s);
const char* norm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* LIBNORM_H */
