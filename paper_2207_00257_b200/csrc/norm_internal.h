// norm_internal.h — host-side internals of libnorm shared by the C ABI (libnorm.cpp),
// the NCCL / peer layer (comm.cpp) and the kernel launchers (reduce.cu, scale.cu,
// fused.cu, rows.cu, rowops.cu, unhoisted.cu, backprop.cu).  Not installed.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <nvtx3/nvToolsExt.h>

#include <string>

#include "libnorm.h"

namespace lnorm {

// NVTX range on the host thread for the lifetime of the object (the enqueue of
// one step of the path: "reduce", "exchange:...", "scale", ...).  Header-only
// NVTX v3: a no-op unless a tool (nsys, ncu --nvtx) is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Covered set C(n) of Fig. 1's launch, DESIGN.md §3.1.
enum CovKind { COV_EMPTY = 0, COV_PREFIX = 1, COV_RESIDUE = 2 };
struct Coverage {
  int kind;
  int64_t n;      // vector length
  int64_t count;  // |C(n)|
  int64_t L;      // COV_PREFIX: C(n) = [0, L)
  int64_t G;      // blocks of the literal launch; COV_RESIDUE: C = {x < n : x % 32 < G}
};
Coverage coverage_of(int64_t n, int index);

// Device workspace (one per (device, stream) in the internal cache, or carved
// from the caller's buffer).  Must be zero-filled before first use; every
// kernel that uses the counters returns them to zero.
constexpr int kMaxGrid = 4096;   // max CTAs of any persistent reduce grid
constexpr int kMaxTasks = 16384; // max dynamically scheduled tasks of the bulk reduce
struct Workspace {
  double* partials;    // [kMaxGrid] per-CTA partial sums
  double* S;           // [4] fp64 sum slots (S[0]: vector sum; S[1]: sharded local partial)
  unsigned* ticket;    // [1] last-block ticket of the reduce kernel
  unsigned* task_ctr;  // [1] next task of the bulk reduce's dynamic tail
  unsigned* scale_ctr; // [2] {next chunk, producers done} of the bulk scale's chunk queue
  unsigned* row_ctr;   // [2] {next row, CTAs done} of the register rows kernel's row queue
  unsigned* bp_ctr;    // [2] {next tile run, producers done} of the TMA backprop kernel
  unsigned long long* arrivals;  // [1] fused kernel's grid barrier: CTA arrivals, never reset
  double* task_sums;   // [kMaxTasks] per-task sums of the dynamic tail
};
size_t workspace_bytes();
Workspace workspace_carve(void* base);
// o->workspace if given (checked), else the internal (device, stream) cache.
norm_status_t get_workspace(const norm_opts_t* o, int dev, cudaStream_t st, Workspace* ws);

struct DeviceInfo {
  int device;
  int sms;
  int cc_major, cc_minor;
  size_t l2_bytes;
};
// Cached per device; returns false (with detail) if the device is unusable.
bool device_info(DeviceInfo* out, std::string* err);

enum PdlMode { PDL_OFF = 0, PDL_EARLY = 1, PDL_LATE = 2 };
int pdl_mode();  // NORM_PDL env knob, read once (reduce.cu)
bool pdl_chain();  // NORM_PDL_CHAIN: small / mid kernels as programmatic dependents (reduce.cu)

// ---- kernel launchers.  All return the launch's cudaError_t. ----
// Tuning constants live next to the kernels.
int reduce_grid(const DeviceInfo& d, int64_t n);

// S_out <- sum of in[0, n) (fp64), via per-CTA partials and a last-block ticket.
// Peer-memory publication of a rank's partial (fused exchange, comm.cpp).  When
// `mail` is set, the reduce's last CTA also stores S into slot [epoch & 1][rank]
// of every rank's mailbox (mail[r] = rank r's mailbox, mapped here) and then
// releases the slot's epoch flag at system scope.  Mailbox layout (fp64 pairs):
// [2 parities][world ranks] x {partial, epoch as u64}.
struct PeerPost {
  double* const* mail;
  int rank, world;
  unsigned long long epoch;
};

// n >= 2^22: TMA-bulk kernel (one CTA per SM); smaller n: LDG.E.256 kernel.
cudaError_t launch_reduce(const float* in, int64_t n, const Workspace& ws, double* S_out,
                          const DeviceInfo& d, cudaStream_t st, PeerPost post = PeerPost{nullptr, 0, 0, 0});

// out[i] = in[i] / s for i in [0, len), s = (float)(S_parts[0] + ... + S_parts[nparts-1])
// (fixed order).  Launched as a PDL dependent of the preceding kernel when pdl.
// Block 0 writes sum_out / sum_out_f64 when non-null (also when len == 0).
// epoch != 0: S_parts is this rank's mailbox; the prologue waits (acquire, system
// scope, ~30 s timeout -> NaN) until all nparts slots of parity epoch & 1 carry
// `epoch`, then combines them in rank order.
// ctr (Workspace::scale_ctr, zeroed; left zeroed): the bulk kernel deals its
// chunks from a queue instead of grid-strided (NULL: grid-strided).
cudaError_t launch_scale(float* out, const float* in, int64_t len, const double* S_parts,
                         int nparts, float* sum_out, double* sum_out_f64,
                         const DeviceInfo& d, bool pdl, cudaStream_t st,
                         unsigned long long epoch = 0, unsigned* ctr = nullptr);

// Residue coverage (literal, G < 32): local element j is global index gbegin + j;
// written iff (gbegin + j) % 32 < G.
cudaError_t launch_scale_residue(float* out, const float* in, int64_t len, int64_t gbegin,
                                 int64_t G, const double* S_parts, int nparts, float* sum_out,
                                 double* sum_out_f64, bool pdl, cudaStream_t st,
                                 unsigned long long epoch = 0);

// One CTA: reduce, then scale C(n).  For small n (one launch, no workspace).
cudaError_t launch_small(float* out, const float* in, const Coverage& cov, float* sum_out,
                         double* sum_out_f64, cudaStream_t st);

// One cooperative persistent kernel: reduce (covered prefix last, L2 evict_last),
// grid barrier, scale from L2.  Requires COV_PREFIX.
// Chunks of an n-element stream that the bulk reduce / fused kernel hand out
// dynamically (NORM_DYN_PCT / NORM_DYN_TC; reduce.cu), and the task size.
int64_t dyn_chunks(int64_t n, int grid, int* tc);

// post.mail set: multi-GPU, the rank partial is published into every rank's
// mailbox after the grid barrier and `mailbox` (this rank's) is waited on.
cudaError_t launch_fused(float* out, const float* in, const Coverage& cov, const Workspace& ws,
                         float* sum_out, double* sum_out_f64, const DeviceInfo& d,
                         cudaStream_t st, PeerPost post = PeerPost{nullptr, 0, 0, 0},
                         const double* mailbox = nullptr);

// One cooperative LDG.E.256 kernel (one CTA per SM): reduce, grid barrier, scale of
// the covered prefix from L2 (NORM_PATH_MID: L2-sized inputs).  Requires COV_PREFIX.
cudaError_t launch_mid(float* out, const float* in, const Coverage& cov, const Workspace& ws,
                       float* sum_out, double* sum_out_f64, const DeviceInfo& d, cudaStream_t st,
                       PeerPost post = PeerPost{nullptr, 0, 0, 0}, const double* mailbox = nullptr);

// The whole call in one thread-block cluster (16 CTAs, DSMEM combine; NORM_PATH_
// CLUSTER, cluster.cu).  Requires COV_PREFIX.  No workspace.
cudaError_t launch_cluster(float* out, const float* in, const Coverage& cov, float* sum_out,
                           double* sum_out_f64, const DeviceInfo& d, cudaStream_t st);

// Batched rows: one CTA per row (grid-strided), row held in registers when it fits.
// row_ctr (Workspace::row_ctr, zeroed; left zeroed) or NULL: rows dealt from a
// queue or grid-strided.
cudaError_t launch_rows(float* out, const float* in, int64_t rows, int64_t cols, int64_t ld_out,
                        int64_t ld_in, const Coverage& row_cov, float* sum_out,
                        double* sum_out_f64, const DeviceInfo& d, cudaStream_t st,
                        unsigned* row_ctr = nullptr);

// Fig. 1 before LICM (unhoisted.cu): the printed launch <<<(n+31)/32, 32>>> with
// `sum` per thread (NORM_FORM_PER_THREAD) or per block (NORM_FORM_PER_BLOCK).
cudaError_t launch_unhoisted(float* out, const float* in, int64_t n, int index, int form,
                             float* sum_out, double* sum_out_f64, cudaStream_t st);

// NEXT-2 row ops (rowops.cu)
cudaError_t launch_softmax_rows(float* out, const float* in, int64_t rows, int64_t cols,
                                int64_t ld_out, int64_t ld_in, bool log, const DeviceInfo& d,
                                cudaStream_t st, unsigned* row_ctr = nullptr);
cudaError_t launch_nll_forward(float* loss, float* total_weight, const float* logp,
                               const int64_t* target, const float* weight, int64_t N, int64_t C,
                               int64_t ld, int reduction, int64_t ignore_index,
                               const Workspace& ws, const DeviceInfo& d, cudaStream_t st);
cudaError_t launch_nll_backward(float* grad, const float* grad_out, const int64_t* target,
                                const float* weight, const float* total_weight, int64_t N,
                                int64_t C, int64_t ld, int reduction, int64_t ignore_index,
                                const DeviceInfo& d, cudaStream_t st);
// Gradients (backward.cu): normalize's functional form and row softmax / log-softmax.
enum BwKind { BW_NORMALIZE = 0, BW_SOFTMAX = 1, BW_LOG_SOFTMAX = 2 };
cudaError_t launch_normalize_backward(float* gx, const float* g, const float* y, const float* s,
                                      const Coverage& cov, const Workspace& ws, const DeviceInfo& d,
                                      cudaStream_t st);
cudaError_t launch_rows_backward(float* gx, const float* g, const float* y, const float* s_rows,
                                 int64_t rows, int64_t cols, int64_t ld, int kind, const Coverage& rc,
                                 const DeviceInfo& d, cudaStream_t st, unsigned* row_ctr);

// NEXT-4 backprop layerforward (backprop.cu)
cudaError_t launch_bpnn(const float* input, float* hidden, float* output, int64_t in, int64_t hid,
                        int variant, cudaStream_t st, const DeviceInfo& d, unsigned* ctr);

// The AUTO path for a call over n elements whose covered set is [0, L) (prefix)
// or not a prefix (libnorm.cpp; also used per rank by the sharded peer path).
int auto_path(int64_t n, int64_t L, bool prefix, const DeviceInfo& d);

// Argument checks shared by the C ABI entry points (libnorm.cpp).
norm_status_t check_device(DeviceInfo* d);  // current device, must be sm_100
norm_status_t check_opts(const norm_opts_t* o);
norm_status_t check_out_ptrs(const norm_opts_t* o, const DeviceInfo& d);  // sum_out, sum_out_f64
norm_status_t check_io_ptrs(const float* out, const float* in, const norm_opts_t* o,
                            const DeviceInfo& d);  // + in, out

// norm_debug_set_events instrumentation: record this thread's begin / end event
// (if set, and not while a graph is being captured) on `st`.
void ev_begin(cudaStream_t st);
void ev_end(cudaStream_t st);

// thread-local error detail
void set_error(const std::string& s);
norm_status_t fail(norm_status_t st, const std::string& s);
norm_status_t cuda_fail(cudaError_t e, const char* what);

}  // namespace lnorm
