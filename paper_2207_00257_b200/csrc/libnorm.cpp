// libnorm.cpp — the C ABI of include/libnorm.h: argument validation, the launch
// plan (coverage of Fig. 1's grid, path choice, grid sizes), workspace
// management, dispatch to the kernels, and the host-buffer (end-to-end) entry.
#include <cuda_runtime.h>
#include <string.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "libnorm.h"
#include "norm_internal.h"

#define NORM_API extern "C" __attribute__((visibility("default")))

namespace lnorm {

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

void set_error(const std::string& s) { g_last_error = s; }
norm_status_t fail(norm_status_t st, const std::string& s) {
  set_error(s);
  return st;
}
norm_status_t cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  return NORM_ERR_CUDA;
}

// ------------------------------------------------ instrumentation (bench only)
// norm_debug_set_events: events recorded around the dominant kernel of every
// call on this host thread; suppressed while norm_graph_create captures.
static thread_local cudaEvent_t g_ev_begin = nullptr, g_ev_end = nullptr;
static thread_local bool g_capturing = false;

void ev_begin(cudaStream_t st) {
  if (g_ev_begin && !g_capturing) cudaEventRecord(g_ev_begin, st);
}
void ev_end(cudaStream_t st) {
  if (g_ev_end && !g_capturing) cudaEventRecord(g_ev_end, st);
}

// ---------------------------------------------------------------- coverage
// Fig. 1: normalize<<<(n+31)/32, 32>>> with tid = blockIdx.x + blockDim.x*threadIdx.x
// (PAPER.md:103, 113).  tid = b + 32t, 0 <= b < G, 0 <= t < 32:
//   G >= 32 -> every residue mod 32 occurs among b, tids fill [0, G+991]: C = [0, min(n, G+992))
//   G <  32 -> tid mod 32 == b:  C = {x < n : x mod 32 < G}
// NORM_FAULT: build-time fault injection for the test suite only
// (tests/test_gpu_faults.py builds libnorm_fault<k>.so and checks that the parity
// tests catch each fault).  Never defined in the product build.
#ifndef NORM_FAULT
#define NORM_FAULT 0
#endif

Coverage coverage_of(int64_t n, int index) {
  Coverage c{};
#if NORM_FAULT == 2  // fault: the conventional (dense) index instead of Fig. 1's literal one
  index = NORM_INDEX_DENSE;
#endif
  c.n = n;
  c.G = n > 0 ? (n + 31) / 32 : 0;
  if (n <= 0) {
    c.kind = COV_EMPTY;
    return c;
  }
  if (index == NORM_INDEX_DENSE) {
    c.kind = COV_PREFIX;
    c.L = c.count = n;
    return c;
  }
  if (c.G >= 32) {
    c.kind = COV_PREFIX;
#if NORM_FAULT == 7  // fault: off-by-one in the covered prefix
    c.L = c.count = (n < c.G + 991) ? n : c.G + 991;
#else
    c.L = c.count = (n < c.G + 992) ? n : c.G + 992;
#endif
    return c;
  }
  if (n <= 32) {  // G == 1: only tid 0
    c.kind = COV_PREFIX;
    c.L = c.count = 1;
    return c;
  }
  c.kind = COV_RESIDUE;
  const int64_t rem = n % 32;
  c.count = (n / 32) * c.G + (rem < c.G ? rem : c.G);
  c.L = -1;
  return c;
}

// --------------------------------------------------------------- devices
bool device_info(DeviceInfo* out, std::string* err) {
  static std::mutex mu;
  static std::vector<DeviceInfo> cache;
  static std::vector<bool> valid;
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    *err = std::string("cudaGetDevice: ") + cudaGetErrorString(e);
    return false;
  }
  std::lock_guard<std::mutex> lk(mu);
  if ((int)cache.size() <= dev) {
    cache.resize(dev + 1);
    valid.resize(dev + 1, false);
  }
  if (!valid[dev]) {
    DeviceInfo d{};
    d.device = dev;
    int l2 = 0;
    if (cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess) {
      *err = "cudaDeviceGetAttribute failed";
      return false;
    }
    d.l2_bytes = (size_t)l2;
    cache[dev] = d;
    valid[dev] = true;
  }
  *out = cache[dev];
  return true;
}

norm_status_t check_device(DeviceInfo* d) {
  std::string err;
  if (!device_info(d, &err)) return fail(NORM_ERR_CUDA, err);
  if (d->cc_major != 10 || d->cc_minor != 0)
    return fail(NORM_ERR_UNSUPPORTED, "libnorm is built for sm_100a (B200); device is sm_" +
                                          std::to_string(d->cc_major) + std::to_string(d->cc_minor));
  return NORM_OK;
}

// ------------------------------------------------------------- workspace
static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t workspace_bytes() {
  return align_up(kMaxGrid * sizeof(double), 256) + 256 /* S[4] */ + 256 /* ticket and the queue / barrier counters */ +
         align_up(kMaxTasks * sizeof(double), 256);
}

Workspace workspace_carve(void* base) {
  char* p = static_cast<char*>(base);
  Workspace w;
  w.partials = reinterpret_cast<double*>(p);
  p += align_up(kMaxGrid * sizeof(double), 256);
  w.S = reinterpret_cast<double*>(p);
  p += 256;
  w.ticket = reinterpret_cast<unsigned*>(p);
  w.task_ctr = w.ticket + 4;
  w.scale_ctr = w.ticket + 6;
  w.row_ctr = w.ticket + 8;
  w.bp_ctr = w.ticket + 10;
  w.arrivals = reinterpret_cast<unsigned long long*>(w.ticket + 12);  // 8-byte aligned
  p += 256;
  w.task_sums = reinterpret_cast<double*>(p);
  return w;
}

// Internal cache: one zeroed workspace per (device, stream), a few KB each, kept
// until norm_cache_release().
static std::mutex g_ws_mu;
static std::map<std::pair<int, cudaStream_t>, void*> g_ws_cache;
// Bumped by norm_cache_release; a thread's one-entry memo of its last (device,
// stream) -> workspace lookup is valid only for the generation it was made in
// (saves the mutex + map lookup on back-to-back calls: configs 1-2 are host-bound).
static std::atomic<unsigned long long> g_ws_gen{1};
struct WsMemo {
  int dev = -1;
  cudaStream_t st = nullptr;
  void* p = nullptr;
  unsigned long long gen = 0;
};
static thread_local WsMemo g_ws_memo;

static norm_status_t internal_workspace(int dev, cudaStream_t st, Workspace* ws) {
  WsMemo& m = g_ws_memo;
  if (m.p && m.dev == dev && m.st == st && m.gen == g_ws_gen.load(std::memory_order_acquire)) {
    *ws = workspace_carve(m.p);
    return NORM_OK;
  }
  std::mutex& mu = g_ws_mu;
  auto& cache = g_ws_cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(dev, st);
  auto it = cache.find(key);
  if (it == cache.end()) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, workspace_bytes());
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error(std::string("workspace cudaMalloc: ") + cudaGetErrorString(e));
      return NORM_ERR_WORKSPACE;
    }
    e = cudaMemsetAsync(p, 0, workspace_bytes(), st);
    if (e != cudaSuccess) return cuda_fail(e, "workspace memset");
    it = cache.emplace(key, p).first;
  }
  *ws = workspace_carve(it->second);
  m.dev = dev;
  m.st = st;
  m.p = it->second;
  m.gen = g_ws_gen.load(std::memory_order_acquire);
  return NORM_OK;
}

norm_status_t get_workspace(const norm_opts_t* o, int dev, cudaStream_t st, Workspace* ws) {
  if (o->workspace) {
    if (o->workspace_bytes < workspace_bytes())
      return fail(NORM_ERR_WORKSPACE, "workspace_bytes < norm_workspace_bytes()");
    if (reinterpret_cast<uintptr_t>(o->workspace) & 255u)
      return fail(NORM_ERR_INVALID_VALUE, "workspace must be 256-byte aligned");
    *ws = workspace_carve(o->workspace);
    return NORM_OK;
  }
  return internal_workspace(dev, st, ws);
}

// ------------------------------------------------------------ validation
static bool aligned4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }

norm_status_t check_opts(const norm_opts_t* o) {
  if (o->index != NORM_INDEX_LITERAL && o->index != NORM_INDEX_DENSE)
    return fail(NORM_ERR_INVALID_VALUE, "bad index mode");
  if (o->path < NORM_PATH_AUTO || o->path > NORM_PATH_CLUSTER)
    return fail(NORM_ERR_INVALID_VALUE, "bad path");
  if ((o->flags & ~NORM_FLAG_TRUSTED_PTRS) != 0u || o->reserved != 0u)
    return fail(NORM_ERR_INVALID_VALUE, "unknown flags or nonzero reserved field");
  return NORM_OK;
}

// Byte spans [a, a+na) and [b, b+nb): identical start and length -> alias (ok).
static bool partial_overlap(const void* a, size_t na, const void* b, size_t nb) {
  uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  if (x == y && na == nb) return false;
  return x < y + nb && y < x + na;
}

// A pointer the kernels dereference must be device (or managed) memory of the
// current device: a host pointer, or device memory of another GPU launched on
// from this one, is a sticky device fault, so it is rejected up front.  Skipped
// under NORM_FLAG_TRUSTED_PTRS (the caller vouches; launch-bound callers).
static norm_status_t check_device_ptr(const void* p, const char* name, const DeviceInfo& d,
                                      const norm_opts_t* o) {
  if (o && (o->flags & NORM_FLAG_TRUSTED_PTRS)) return NORM_OK;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_fail(e, "cudaPointerGetAttributes");
  }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
    return fail(NORM_ERR_INVALID_VALUE, std::string(name) +
                                            " is not device memory (use norm_launch_host for host buffers)");
  if (at.type == cudaMemoryTypeDevice && at.device != d.device)
    return fail(NORM_ERR_INVALID_VALUE, std::string(name) + " lives on device " +
                                            std::to_string(at.device) + " but the current device is " +
                                            std::to_string(d.device) + " (cudaSetDevice first)");
  return NORM_OK;
}

norm_status_t check_out_ptrs(const norm_opts_t* o, const DeviceInfo& d) {
  norm_status_t s;
  if (o->sum_out && (s = check_device_ptr(o->sum_out, "sum_out", d, o)) != NORM_OK) return s;
  if (o->sum_out_f64 && (s = check_device_ptr(o->sum_out_f64, "sum_out_f64", d, o)) != NORM_OK) return s;
  return NORM_OK;
}

norm_status_t check_io_ptrs(const float* out, const float* in, const norm_opts_t* o,
                            const DeviceInfo& d) {
  norm_status_t s;
  if ((s = check_device_ptr(in, "in", d, o)) != NORM_OK) return s;
  if (out != in && (s = check_device_ptr(out, "out", d, o)) != NORM_OK) return s;
  return check_out_ptrs(o, d);
}

static norm_status_t check_vector_args(float* out, const float* in, int64_t n) {
  if (n < 0) return fail(NORM_ERR_INVALID_VALUE, "n < 0");
  if (n == 0) return NORM_OK;
  if (!out || !in) return fail(NORM_ERR_INVALID_VALUE, "NULL pointer with n > 0");
  if (!aligned4(out) || !aligned4(in)) return fail(NORM_ERR_INVALID_VALUE, "pointer not 4-byte aligned");
  if (partial_overlap(out, (size_t)n * 4, in, (size_t)n * 4))
    return fail(NORM_ERR_OVERLAP, "out and in partially overlap");
  return NORM_OK;
}

static norm_status_t check_literal_grid(const Coverage& c, int index) {
  if (index == NORM_INDEX_LITERAL && c.G > 2147483647LL)
    return fail(NORM_ERR_UNSUPPORTED, "literal launch needs > 2^31-1 blocks (gridDim.x limit)");
  return NORM_OK;
}

// AUTO path thresholds, measured on B200: device time per call
// from CUDA graphs of back-to-back calls, L2 flushed before each call
// (scripts/path_sweep.py -> profiles/round2/path_sweep*.txt; earlier
// scripts/fused_vs_twopass.py, profiles/r05/fused_*.txt):
//  * n <= 3 x 2^15: one CTA does everything (2.4-4 us; mid 4.4-4.7 us);
//  * covered set a prefix and 4n <= 2 L2 (literal) / 0.6 L2 (dense, whose
//    scale re-reads and writes all of it): mid, one cooperative launch of
//    256-bit-load CTAs -- the TMA kernels' fixed cost (ring set-up, dynamic
//    tail, second launch) dominates below that: literal 2^20+7 / 2^22 / 2^25:
//    mid 8.0 / 9.9 / 29.5 us vs two-pass 8.5 / 14.2 / 33.2 vs fused 12.9 / 14.2 /
//    32.8; 2^26 ties (50.5 / 51.4 / 50.9); dense 2^24: mid 30.7, fused 33.3,
//    two-pass 41.9;
//  * fused (TMA ring, covered prefix read last with evict_last, scaled from L2)
//    for partial coverage with input > 2 L2 and covered bytes <= 3 L2 (literal
//    2^27..2^31: 5-9 us faster than two-pass; at 2^32 the 512 MiB prefix
//    streams from HBM and the two-pass TMA scale wins by 15 us), and for full
//    coverage with 0.6 L2 < 4n <= 2 L2 (dense 2^25 / 2^26: 62.3 / 122.7 us vs
//    two-pass 72.4 / 128.7);
//  * otherwise two-pass (dense 2^27: 242 vs fused 245; 2^28: 469 vs 489).
constexpr int64_t kSmallN = 3 << 15;

int auto_path(int64_t n, int64_t L, bool prefix, const DeviceInfo& d) {
  if (n <= kSmallN) return NORM_PATH_SMALL;
  if (!prefix) return NORM_PATH_TWO_PASS;
  const double bytes = 4.0 * (double)n, l2 = (double)d.l2_bytes;
  const bool full = L >= n;
  if (bytes <= (full ? 0.6 : 2.0) * l2) return NORM_PATH_MID;
  if (!full && (double)L * 4.0 <= 3.0 * l2) return NORM_PATH_FUSED;
  if (full && bytes <= 2.0 * l2) return NORM_PATH_FUSED;
  return NORM_PATH_TWO_PASS;
}

static int choose_path(const Coverage& cov, const norm_opts_t* o, const DeviceInfo& d) {
  if (o->path != NORM_PATH_AUTO) return o->path;
  return auto_path(cov.n, cov.L, cov.kind == COV_PREFIX, d);
}

static norm_status_t launch_vector(float* out, const float* in, const Coverage& cov,
                                   const norm_opts_t* o, const DeviceInfo& d) {
  cudaStream_t st = static_cast<cudaStream_t>(o->stream);
  int path = choose_path(cov, o, d);
  if ((path == NORM_PATH_FUSED || path == NORM_PATH_MID || path == NORM_PATH_CLUSTER) && cov.kind != COV_PREFIX)
    path = NORM_PATH_SMALL;
  cudaError_t e;
  if (path == NORM_PATH_CLUSTER) {
    NvtxRange r("libnorm:cluster");
    ev_begin(st);
    e = launch_cluster(out, in, cov, o->sum_out, o->sum_out_f64, d, st);
    if (e != cudaSuccess) return cuda_fail(e, "cluster_kernel launch");
    ev_end(st);
    return NORM_OK;
  }
  if (path == NORM_PATH_SMALL) {
    NvtxRange r("libnorm:small");
    ev_begin(st);
    e = launch_small(out, in, cov, o->sum_out, o->sum_out_f64, st);
    if (e != cudaSuccess) return cuda_fail(e, "small_kernel launch");
    ev_end(st);
    return NORM_OK;
  }
  Workspace ws;
  norm_status_t s = get_workspace(o, d.device, st, &ws);
  if (s != NORM_OK) return s;
  if (path == NORM_PATH_FUSED) {
    NvtxRange r("libnorm:fused");
    ev_begin(st);
    e = launch_fused(out, in, cov, ws, o->sum_out, o->sum_out_f64, d, st);
    if (e != cudaSuccess) return cuda_fail(e, "fused_kernel cooperative launch");
    ev_end(st);
    return NORM_OK;
  }
  if (path == NORM_PATH_MID) {
    NvtxRange r("libnorm:mid");
    ev_begin(st);
    e = launch_mid(out, in, cov, ws, o->sum_out, o->sum_out_f64, d, st);
    if (e != cudaSuccess) return cuda_fail(e, "mid_kernel cooperative launch");
    ev_end(st);
    return NORM_OK;
  }
  // The step's dominant kernel for norm_debug_set_events: the reduce (4n bytes),
  // or the scale when it moves more (8|C| > 4n: dense and nearly dense coverage).
  const bool scale_dominant = cov.kind == COV_PREFIX && 2 * cov.L > cov.n;
  {
    NvtxRange r("libnorm:reduce");
    if (!scale_dominant) ev_begin(st);
    e = launch_reduce(in, cov.n, ws, ws.S, d, st);
    if (e != cudaSuccess) return cuda_fail(e, "reduce_kernel launch");
    if (!scale_dominant) ev_end(st);
  }
  NvtxRange r("libnorm:scale");
  if (scale_dominant) ev_begin(st);
  if (cov.kind == COV_PREFIX)
    e = launch_scale(out, in, cov.L, ws.S, 1, o->sum_out, o->sum_out_f64, d, true, st, 0, ws.scale_ctr);
  else
    e = launch_scale_residue(out, in, cov.n, 0, cov.G, ws.S, 1, o->sum_out, o->sum_out_f64, true, st);
  if (e != cudaSuccess) return cuda_fail(e, "scale_kernel launch");
  if (scale_dominant) ev_end(st);
  return NORM_OK;
}

// ----------------------------------------------------- host-buffer (e2e) path
// Device staging per (device, stream): resident buffer for the covered elements,
// a ring of chunk buffers for the uncovered remainder, per-chunk sums, a copy
// stream and events.  Grows on demand, never shrinks.
constexpr int64_t kHostChunk = 32ll << 20;  // elements per H2D chunk (128 MiB)
constexpr int kRing = 3;

struct HostStage {
  cudaStream_t copy = nullptr;
  float* resident = nullptr;
  int64_t resident_cap = 0;
  float* ring[kRing] = {};
  double* chunkS = nullptr;
  int64_t chunkS_cap = 0;
  cudaEvent_t landed[2] = {};
  cudaEvent_t slot_free[kRing] = {};
  cudaEvent_t start = nullptr;
  void* ws = nullptr;
};

static std::mutex g_hs_mu;
static std::map<std::pair<int, cudaStream_t>, HostStage*> g_hs_cache;

static norm_status_t host_stage(int dev, cudaStream_t st, int64_t resident, int64_t nchunks,
                                HostStage** out) {
  std::mutex& mu = g_hs_mu;
  auto& cache = g_hs_cache;
  std::lock_guard<std::mutex> lk(mu);
  HostStage*& h = cache[std::make_pair(dev, st)];
  cudaError_t e;
  if (!h) {
    h = new HostStage();
    if ((e = cudaStreamCreateWithFlags(&h->copy, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "copy stream");
    for (auto& ev : h->landed)
      if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "event");
    for (auto& ev : h->slot_free)
      if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "event");
    if ((e = cudaEventCreateWithFlags(&h->start, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "event");
    for (auto& r : h->ring)
      if ((e = cudaMalloc(&r, kHostChunk * 4)) != cudaSuccess) {
        cudaGetLastError();
        return fail(NORM_ERR_WORKSPACE, "staging ring cudaMalloc failed");
      }
    if ((e = cudaMalloc(&h->ws, workspace_bytes())) != cudaSuccess) {
      cudaGetLastError();
      return fail(NORM_ERR_WORKSPACE, "workspace cudaMalloc failed");
    }
    if ((e = cudaMemsetAsync(h->ws, 0, workspace_bytes(), st)) != cudaSuccess)
      return cuda_fail(e, "workspace memset");
  }
  if (resident > h->resident_cap) {
    cudaStreamSynchronize(st);  // the old buffer may still be in use
    cudaFree(h->resident);
    h->resident = nullptr;
    h->resident_cap = 0;
    if ((e = cudaMalloc(&h->resident, (size_t)resident * 4)) != cudaSuccess) {
      cudaGetLastError();
      return fail(NORM_ERR_WORKSPACE, "resident buffer of " + std::to_string(resident * 4) +
                                          " bytes: cudaMalloc failed");
    }
    h->resident_cap = resident;
  }
  if (nchunks > h->chunkS_cap) {
    cudaStreamSynchronize(st);
    cudaFree(h->chunkS);
    h->chunkS = nullptr;
    if ((e = cudaMalloc(&h->chunkS, (size_t)nchunks * sizeof(double))) != cudaSuccess) {
      cudaGetLastError();
      return fail(NORM_ERR_WORKSPACE, "chunk sums cudaMalloc failed");
    }
    h->chunkS_cap = nchunks;
  }
  *out = h;
  return NORM_OK;
}

static norm_status_t launch_host(float* out_host, const float* in_host, const Coverage& cov,
                                 const norm_opts_t* o, const DeviceInfo& d) {
  NvtxRange r("norm_launch_host");
  cudaStream_t st = static_cast<cudaStream_t>(o->stream);
  const int64_t n = cov.n;
  // Elements that must stay on the device until the divisor is known.
  const int64_t R = cov.kind == COV_PREFIX ? cov.L : n;
  // Chunk list: [0, R) in resident chunks, then [R, n) through the ring.
  struct Chunk { int64_t a, b; bool res; };
  std::vector<Chunk> chunks;
  for (int64_t a = 0; a < R; a += kHostChunk) chunks.push_back({a, a + kHostChunk < R ? a + kHostChunk : R, true});
  for (int64_t a = R; a < n; a += kHostChunk) chunks.push_back({a, a + kHostChunk < n ? a + kHostChunk : n, false});
  HostStage* h = nullptr;
  norm_status_t s = host_stage(d.device, st, R, (int64_t)chunks.size(), &h);
  if (s != NORM_OK) return s;
  Workspace ws = workspace_carve(h->ws);
  cudaError_t e;
  // Everything earlier on the caller's stream (e.g. the previous call's D2H out of
  // the resident buffer) happens before this call's first copy.
  if ((e = cudaEventRecord(h->start, st)) != cudaSuccess) return cuda_fail(e, "event record");
  if ((e = cudaStreamWaitEvent(h->copy, h->start, 0)) != cudaSuccess) return cuda_fail(e, "wait");
  int slot = 0;
  for (size_t k = 0; k < chunks.size(); ++k) {
    const Chunk& c = chunks[k];
    const int64_t len = c.b - c.a;
    float* dst;
    int used_slot = -1;
    if (c.res) {
      dst = h->resident + c.a;
    } else {
      used_slot = slot;
      dst = h->ring[slot];
      slot = (slot + 1) % kRing;
      if ((e = cudaStreamWaitEvent(h->copy, h->slot_free[used_slot], 0)) != cudaSuccess)
        return cuda_fail(e, "wait");
    }
    if ((e = cudaMemcpyAsync(dst, in_host + c.a, (size_t)len * 4, cudaMemcpyHostToDevice, h->copy)) != cudaSuccess)
      return cuda_fail(e, "H2D copy");
    cudaEvent_t landed = h->landed[k & 1];
    if ((e = cudaEventRecord(landed, h->copy)) != cudaSuccess) return cuda_fail(e, "event record");
    if ((e = cudaStreamWaitEvent(st, landed, 0)) != cudaSuccess) return cuda_fail(e, "wait");
    if ((e = launch_reduce(dst, len, ws, h->chunkS + k, d, st)) != cudaSuccess)
      return cuda_fail(e, "reduce_kernel launch");
    if (used_slot >= 0 && (e = cudaEventRecord(h->slot_free[used_slot], st)) != cudaSuccess)
      return cuda_fail(e, "event record");
  }
  const int nparts = (int)chunks.size();
  if (cov.kind == COV_PREFIX) {
    e = launch_scale(h->resident, h->resident, cov.L, h->chunkS, nparts, o->sum_out,
                     o->sum_out_f64, d, false, st, 0, ws.scale_ctr);
    if (e != cudaSuccess) return cuda_fail(e, "scale_kernel launch");
    e = cudaMemcpyAsync(out_host, h->resident, (size_t)cov.L * 4, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
  } else {
    e = launch_scale_residue(h->resident, h->resident, n, 0, cov.G, h->chunkS, nparts, o->sum_out,
                             o->sum_out_f64, false, st);
    if (e != cudaSuccess) return cuda_fail(e, "scale_residue launch");
    // covered = columns [0, G) of each 32-wide row: a strided 2-D copy
    const int64_t full = n / 32, rem = n % 32;
    if (full > 0) {
      e = cudaMemcpy2DAsync(out_host, 32 * 4, h->resident, 32 * 4, (size_t)cov.G * 4, (size_t)full,
                            cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
    }
    const int64_t last = rem < cov.G ? rem : cov.G;
    if (last > 0) {
      e = cudaMemcpyAsync(out_host + full * 32, h->resident + full * 32, (size_t)last * 4,
                          cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
    }
  }
  return NORM_OK;
}

}  // namespace lnorm

using namespace lnorm;

static const norm_opts_t kDefaultOpts = NORM_OPTS_INIT;

// ================================================================= C ABI

NORM_API norm_status_t norm_launch_ex(float* out, const float* in, int64_t n, const norm_opts_t* o) {
  NvtxRange r("norm_launch_ex");
  if (!o) o = &kDefaultOpts;
  norm_status_t s;
  if ((s = check_opts(o)) != NORM_OK) return s;
  if ((s = check_vector_args(out, in, n)) != NORM_OK) return s;
  if (n == 0) return NORM_OK;
  const Coverage cov = coverage_of(n, o->index);
  if ((s = check_literal_grid(cov, o->index)) != NORM_OK) return s;
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  if ((s = check_io_ptrs(out, in, o, d)) != NORM_OK) return s;
  return launch_vector(out, in, cov, o, d);
}

// ---- CUDA-graph plans: the whole call (1 or 2 kernels) as one cudaGraphLaunch ----
struct norm_graph {
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap = nullptr;
  void* ws = nullptr;
  int device = -1;
};

NORM_API norm_status_t norm_choose_path(int64_t n, int64_t covered_prefix, int32_t requested,
                                        int32_t* chosen) {
  if (n < 0 || !chosen || requested < NORM_PATH_AUTO || requested > NORM_PATH_CLUSTER ||
      covered_prefix > n)
    return fail(NORM_ERR_INVALID_VALUE, "bad norm_choose_path arguments");
  DeviceInfo d;
  norm_status_t st = check_device(&d);
  if (st != NORM_OK) return st;
  *chosen = requested != NORM_PATH_AUTO ? requested
                                        : auto_path(n, covered_prefix, covered_prefix >= 0, d);
  return NORM_OK;
}

NORM_API norm_status_t norm_graph_create(norm_graph_t** out_g, float* out, const float* in,
                                         int64_t n, const norm_opts_t* o) {
  if (!out_g) return fail(NORM_ERR_INVALID_VALUE, "graph is NULL");
  *out_g = nullptr;
  if (!o) o = &kDefaultOpts;
  norm_status_t s;
  if ((s = check_opts(o)) != NORM_OK) return s;
  if ((s = check_vector_args(out, in, n)) != NORM_OK) return s;
  const Coverage cov = coverage_of(n, o->index);
  if ((s = check_literal_grid(cov, o->index)) != NORM_OK) return s;
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  if (n > 0) {
    if ((s = check_io_ptrs(out, in, o, d)) != NORM_OK) return s;
  }
  norm_graph* g = new norm_graph();
  g->device = d.device;
  auto bail = [&](norm_status_t st) {
    if (g->cap) cudaStreamDestroy(g->cap);
    cudaFree(g->ws);
    delete g;
    return st;
  };
  cudaError_t e = cudaStreamCreateWithFlags(&g->cap, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&g->ws, workspace_bytes());
  if (e == cudaSuccess) e = cudaMemset(g->ws, 0, workspace_bytes());
  if (e != cudaSuccess) {
    cudaGetLastError();
    return bail(cuda_fail(e, "graph set-up"));
  }
  norm_opts_t oc = *o;
  oc.stream = g->cap;
  oc.workspace = g->ws;
  oc.workspace_bytes = workspace_bytes();
  oc.flags |= NORM_FLAG_TRUSTED_PTRS;  // checked above
  if ((e = cudaStreamBeginCapture(g->cap, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
    return bail(cuda_fail(e, "cudaStreamBeginCapture"));
  g_capturing = true;
  s = n > 0 ? launch_vector(out, in, cov, &oc, d) : NORM_OK;
  g_capturing = false;
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(g->cap, &graph);
  if (s != NORM_OK) {
    if (graph) cudaGraphDestroy(graph);
    return bail(s);
  }
  if (e != cudaSuccess) return bail(cuda_fail(e, "cudaStreamEndCapture"));
  e = cudaGraphInstantiate(&g->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return bail(cuda_fail(e, "cudaGraphInstantiate"));
  *out_g = g;
  return NORM_OK;
}

NORM_API norm_status_t norm_graph_launch(norm_graph_t* g, void* stream) {
  if (!g) return fail(NORM_ERR_INVALID_VALUE, "graph is NULL");
  cudaError_t e = cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? NORM_OK : cuda_fail(e, "cudaGraphLaunch");
}

NORM_API norm_status_t norm_graph_destroy(norm_graph_t* g) {
  if (!g) return NORM_OK;
  cudaDeviceSynchronize();
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->cap) cudaStreamDestroy(g->cap);
  cudaFree(g->ws);
  delete g;
  return NORM_OK;
}

NORM_API norm_status_t norm_launch(float* out, const float* in, int64_t n) {
  return norm_launch_ex(out, in, n, nullptr);
}

NORM_API norm_status_t norm_launch_form(float* out, const float* in, int64_t n, int32_t form,
                                        const norm_opts_t* o) {
  if (form == NORM_FORM_HOISTED) return norm_launch_ex(out, in, n, o);
  if (!o) o = &kDefaultOpts;
  if (form != NORM_FORM_PER_BLOCK && form != NORM_FORM_PER_THREAD)
    return fail(NORM_ERR_INVALID_VALUE, "bad form");
  norm_status_t s;
  if ((s = check_opts(o)) != NORM_OK) return s;
  if ((s = check_vector_args(out, in, n)) != NORM_OK) return s;
  if (n == 0) return NORM_OK;
  if (out == in) return fail(NORM_ERR_OVERLAP, "un-hoisted forms race under aliasing (reading R9)");
  if (n > (1ll << 24)) return fail(NORM_ERR_UNSUPPORTED, "un-hoisted forms are O(N^2): n <= 2^24");
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  if ((s = check_io_ptrs(out, in, o, d)) != NORM_OK) return s;
  cudaError_t e = launch_unhoisted(out, in, n, o->index, form, o->sum_out, o->sum_out_f64,
                                   static_cast<cudaStream_t>(o->stream));
  return e == cudaSuccess ? NORM_OK : cuda_fail(e, "unhoisted kernel launch");
}

NORM_API norm_status_t norm_launch_host(float* out_host, const float* in_host, int64_t n,
                                        const norm_opts_t* o) {
  if (!o) o = &kDefaultOpts;
  norm_status_t s;
  if ((s = check_opts(o)) != NORM_OK) return s;
  if ((s = check_vector_args(out_host, in_host, n)) != NORM_OK) return s;
  if (n == 0) return NORM_OK;
  const Coverage cov = coverage_of(n, o->index);
  if ((s = check_literal_grid(cov, o->index)) != NORM_OK) return s;
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  if ((s = check_out_ptrs(o, d)) != NORM_OK) return s;
  return launch_host(out_host, in_host, cov, o, d);
}

NORM_API norm_status_t norm_rows(float* out, const float* in, int64_t rows, int64_t cols,
                                 int64_t ld_out, int64_t ld_in, const norm_opts_t* o) {
  NvtxRange r("norm_rows");
  if (!o) o = &kDefaultOpts;
  norm_status_t s;
  if ((s = check_opts(o)) != NORM_OK) return s;
  if (rows < 0 || cols < 0) return fail(NORM_ERR_INVALID_VALUE, "rows < 0 or cols < 0");
  if (ld_out < cols || ld_in < cols) return fail(NORM_ERR_INVALID_VALUE, "ld < cols");
  if (rows == 0 || cols == 0) return NORM_OK;
  if (!out || !in) return fail(NORM_ERR_INVALID_VALUE, "NULL pointer with work to do");
  if (!aligned4(out) || !aligned4(in)) return fail(NORM_ERR_INVALID_VALUE, "pointer not 4-byte aligned");
  const size_t span_out = (size_t)((rows - 1) * ld_out + cols) * 4;
  const size_t span_in = (size_t)((rows - 1) * ld_in + cols) * 4;
  const bool alias = out == in && ld_out == ld_in;
  if (!alias && partial_overlap(out, span_out, in, span_in))
    return fail(NORM_ERR_OVERLAP, "out and in rows overlap");
  const Coverage rc = coverage_of(cols, o->index);
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  if ((s = check_io_ptrs(out, in, o, d)) != NORM_OK) return s;
  Workspace ws;
  if ((s = get_workspace(o, d.device, static_cast<cudaStream_t>(o->stream), &ws)) != NORM_OK) return s;
  cudaError_t e = launch_rows(out, in, rows, cols, ld_out, ld_in, rc, o->sum_out, o->sum_out_f64, d,
                              static_cast<cudaStream_t>(o->stream), ws.row_ctr);
  return e == cudaSuccess ? NORM_OK : cuda_fail(e, "rows_kernel launch");
}

NORM_API norm_status_t norm_softmax_rows(float* out, const float* in, int64_t rows, int64_t cols,
                                         int64_t ld_out, int64_t ld_in, int32_t kind,
                                         const norm_opts_t* o) {
  if (!o) o = &kDefaultOpts;
  if (kind != NORM_SOFTMAX && kind != NORM_LOG_SOFTMAX) return fail(NORM_ERR_INVALID_VALUE, "bad kind");
  {
    const norm_status_t so = check_opts(o);
    if (so != NORM_OK) return so;
  }
  if (rows < 0 || cols < 0) return fail(NORM_ERR_INVALID_VALUE, "rows < 0 or cols < 0");
  if (ld_out < cols || ld_in < cols) return fail(NORM_ERR_INVALID_VALUE, "ld < cols");
  if (rows == 0 || cols == 0) return NORM_OK;
  if (!out || !in) return fail(NORM_ERR_INVALID_VALUE, "NULL pointer with work to do");
  if (!aligned4(out) || !aligned4(in)) return fail(NORM_ERR_INVALID_VALUE, "pointer not 4-byte aligned");
  const size_t span_out = (size_t)((rows - 1) * ld_out + cols) * 4;
  const size_t span_in = (size_t)((rows - 1) * ld_in + cols) * 4;
  if (!(out == in && ld_out == ld_in) && partial_overlap(out, span_out, in, span_in))
    return fail(NORM_ERR_OVERLAP, "out and in rows overlap");
  norm_status_t s;
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  if ((s = check_device_ptr(in, "in", d, o)) != NORM_OK) return s;
  if (out != in && (s = check_device_ptr(out, "out", d, o)) != NORM_OK) return s;
  Workspace ws;
  if ((s = get_workspace(o, d.device, static_cast<cudaStream_t>(o->stream), &ws)) != NORM_OK) return s;
  cudaError_t e = launch_softmax_rows(out, in, rows, cols, ld_out, ld_in, kind == NORM_LOG_SOFTMAX, d,
                                      static_cast<cudaStream_t>(o->stream), ws.row_ctr);
  return e == cudaSuccess ? NORM_OK : cuda_fail(e, "softmax kernel launch");
}

// ---- gradients (backward.cu) ----
// gx may alias g or y exactly; any other overlap of gx with g or y is rejected.
static norm_status_t check_bwd_spans(const float* gx, const float* g, const float* y, size_t span) {
  if (gx != g && partial_overlap(gx, span, g, span)) return fail(NORM_ERR_OVERLAP, "gx and g overlap");
  if (gx != y && partial_overlap(gx, span, y, span)) return fail(NORM_ERR_OVERLAP, "gx and y overlap");
  return NORM_OK;
}

static norm_status_t check_bwd_ptrs(const float* gx, const float* g, const float* y, const float* s,
                                    const DeviceInfo& d, const norm_opts_t* o) {
  norm_status_t st;
  if ((st = check_device_ptr(gx, "gx", d, o)) != NORM_OK || (st = check_device_ptr(g, "g", d, o)) != NORM_OK ||
      (st = check_device_ptr(y, "y", d, o)) != NORM_OK)
    return st;
  if (s && (st = check_device_ptr(s, "s", d, o)) != NORM_OK) return st;
  return NORM_OK;
}

NORM_API norm_status_t norm_launch_backward(float* gx, const float* g, const float* y, const float* s,
                                            int64_t n, const norm_opts_t* o) {
  if (!o) o = &kDefaultOpts;
  norm_status_t st;
  if ((st = check_opts(o)) != NORM_OK) return st;
  if (n < 0) return fail(NORM_ERR_INVALID_VALUE, "n < 0");
  if (n == 0) return NORM_OK;
  if (!gx || !g || !y || !s) return fail(NORM_ERR_INVALID_VALUE, "NULL pointer with n > 0");
  if (!aligned4(gx) || !aligned4(g) || !aligned4(y) || !aligned4(s))
    return fail(NORM_ERR_INVALID_VALUE, "pointer not 4-byte aligned");
  if ((st = check_bwd_spans(gx, g, y, (size_t)n * 4)) != NORM_OK) return st;
  const Coverage cov = coverage_of(n, o->index);
  DeviceInfo d;
  if ((st = check_device(&d)) != NORM_OK) return st;
  if ((st = check_bwd_ptrs(gx, g, y, s, d, o)) != NORM_OK) return st;
  cudaStream_t stream = static_cast<cudaStream_t>(o->stream);
  Workspace ws;
  if ((st = get_workspace(o, d.device, stream, &ws)) != NORM_OK) return st;
  NvtxRange r("norm_launch_backward");
  const cudaError_t e = launch_normalize_backward(gx, g, y, s, cov, ws, d, stream);
  return e == cudaSuccess ? NORM_OK : cuda_fail(e, "normalize backward launch");
}

static norm_status_t rows_backward(float* gx, const float* g, const float* y, const float* s,
                                   int64_t rows, int64_t cols, int64_t ld, int kind, const norm_opts_t* o) {
  norm_status_t st;
  if ((st = check_opts(o)) != NORM_OK) return st;
  if (rows < 0 || cols < 0) return fail(NORM_ERR_INVALID_VALUE, "rows < 0 or cols < 0");
  if (ld < cols) return fail(NORM_ERR_INVALID_VALUE, "ld < cols");
  if (rows == 0 || cols == 0) return NORM_OK;
  if (!gx || !g || !y || (kind == BW_NORMALIZE && !s)) return fail(NORM_ERR_INVALID_VALUE, "NULL pointer with work to do");
  if (!aligned4(gx) || !aligned4(g) || !aligned4(y) || (s && !aligned4(s)))
    return fail(NORM_ERR_INVALID_VALUE, "pointer not 4-byte aligned");
  if ((st = check_bwd_spans(gx, g, y, (size_t)((rows - 1) * ld + cols) * 4)) != NORM_OK) return st;
  DeviceInfo d;
  if ((st = check_device(&d)) != NORM_OK) return st;
  if ((st = check_bwd_ptrs(gx, g, y, kind == BW_NORMALIZE ? s : nullptr, d, o)) != NORM_OK) return st;
  const Coverage rc = coverage_of(cols, o->index);
  Workspace ws;
  if ((st = get_workspace(o, d.device, static_cast<cudaStream_t>(o->stream), &ws)) != NORM_OK) return st;
  NvtxRange r("norm_rows_backward");
  const cudaError_t e = launch_rows_backward(gx, g, y, s, rows, cols, ld, kind, rc, d,
                                             static_cast<cudaStream_t>(o->stream), ws.row_ctr);
  return e == cudaSuccess ? NORM_OK : cuda_fail(e, "rows backward launch");
}

NORM_API norm_status_t norm_rows_backward(float* gx, const float* g, const float* y, const float* s,
                                          int64_t rows, int64_t cols, int64_t ld, const norm_opts_t* o) {
  if (!o) o = &kDefaultOpts;
  return rows_backward(gx, g, y, s, rows, cols, ld, BW_NORMALIZE, o);
}

NORM_API norm_status_t norm_softmax_rows_backward(float* gx, const float* g, const float* y, int64_t rows,
                                                  int64_t cols, int64_t ld, int32_t kind,
                                                  const norm_opts_t* o) {
  if (!o) o = &kDefaultOpts;
  if (kind != NORM_SOFTMAX && kind != NORM_LOG_SOFTMAX) return fail(NORM_ERR_INVALID_VALUE, "bad kind");
  return rows_backward(gx, g, y, nullptr, rows, cols, ld, kind == NORM_SOFTMAX ? BW_SOFTMAX : BW_LOG_SOFTMAX, o);
}

static norm_status_t check_nll(int64_t N, int64_t C, int64_t ld, int32_t reduction) {
  if (N < 0 || C < 1 || ld < C) return fail(NORM_ERR_INVALID_VALUE, "need N >= 0, C >= 1, ld >= C");
  if (reduction < NORM_REDUCTION_NONE || reduction > NORM_REDUCTION_SUM)
    return fail(NORM_ERR_INVALID_VALUE, "bad reduction");
  return NORM_OK;
}

NORM_API norm_status_t norm_nll_forward(float* loss, float* total_weight, const float* logp,
                                        const int64_t* target, const float* weight, int64_t N,
                                        int64_t C, int64_t ld, int32_t reduction,
                                        int64_t ignore_index, const norm_opts_t* o) {
  if (!o) o = &kDefaultOpts;
  norm_status_t s;
  if ((s = check_nll(N, C, ld, reduction)) != NORM_OK) return s;
  if ((s = check_opts(o)) != NORM_OK) return s;
  if (!loss || (N > 0 && (!logp || !target))) return fail(NORM_ERR_INVALID_VALUE, "NULL pointer");
  if (reduction == NORM_REDUCTION_NONE && N == 0) return NORM_OK;
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  // every pointer the kernels dereference: device memory of this device
  if ((s = check_device_ptr(loss, "loss", d, o)) != NORM_OK) return s;
  if (total_weight && (s = check_device_ptr(total_weight, "total_weight", d, o)) != NORM_OK) return s;
  if (weight && (s = check_device_ptr(weight, "weight", d, o)) != NORM_OK) return s;
  if (N > 0 && ((s = check_device_ptr(logp, "logp", d, o)) != NORM_OK ||
                (s = check_device_ptr(target, "target", d, o)) != NORM_OK))
    return s;
  cudaStream_t st = static_cast<cudaStream_t>(o->stream);
  Workspace ws;
  if ((s = get_workspace(o, d.device, st, &ws)) != NORM_OK) return s;
  cudaError_t e = launch_nll_forward(loss, total_weight, logp, target, weight, N, C, ld, reduction,
                                     ignore_index, ws, d, st);
  return e == cudaSuccess ? NORM_OK : cuda_fail(e, "nll_forward launch");
}

NORM_API norm_status_t norm_nll_backward(float* grad, const float* grad_out, const int64_t* target,
                                         const float* weight, const float* total_weight, int64_t N,
                                         int64_t C, int64_t ld, int32_t reduction,
                                         int64_t ignore_index, const norm_opts_t* o) {
  if (!o) o = &kDefaultOpts;
  norm_status_t s;
  if ((s = check_nll(N, C, ld, reduction)) != NORM_OK) return s;
  if (N == 0) return NORM_OK;
  if (!grad || !grad_out || !target) return fail(NORM_ERR_INVALID_VALUE, "NULL pointer");
  if (reduction == NORM_REDUCTION_MEAN && !total_weight)
    return fail(NORM_ERR_INVALID_VALUE, "MEAN needs total_weight");
  if ((s = check_opts(o)) != NORM_OK) return s;
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  if ((s = check_device_ptr(grad, "grad", d, o)) != NORM_OK ||
      (s = check_device_ptr(grad_out, "grad_out", d, o)) != NORM_OK ||
      (s = check_device_ptr(target, "target", d, o)) != NORM_OK)
    return s;
  if (weight && (s = check_device_ptr(weight, "weight", d, o)) != NORM_OK) return s;
  if (total_weight && (s = check_device_ptr(total_weight, "total_weight", d, o)) != NORM_OK) return s;
  cudaError_t e = launch_nll_backward(grad, grad_out, target, weight, total_weight, N, C, ld,
                                      reduction, ignore_index, d, static_cast<cudaStream_t>(o->stream));
  return e == cudaSuccess ? NORM_OK : cuda_fail(e, "nll_backward launch");
}

NORM_API norm_status_t norm_bpnn_layerforward(const float* input, float* hidden, float* output,
                                              int64_t in, int64_t hid, int32_t variant,
                                              const norm_opts_t* o) {
  if (!o) o = &kDefaultOpts;
  if (variant < NORM_BP_PRINTED || variant > NORM_BP_TMA)
    return fail(NORM_ERR_INVALID_VALUE, "bad variant");
  if (in < 0) return fail(NORM_ERR_INVALID_VALUE, "in < 0");
  if (hid != 16 || in % 16 != 0)
    return fail(NORM_ERR_UNSUPPORTED, "bpnn_layerforward needs hid == 16 and in % 16 == 0");
  if (in == 0) return NORM_OK;
  if (!input || !hidden || !output) return fail(NORM_ERR_INVALID_VALUE, "NULL pointer");
  if (in / 16 > 2147483647LL) return fail(NORM_ERR_UNSUPPORTED, "too many blocks");
  norm_status_t s;
  if ((s = check_opts(o)) != NORM_OK) return s;
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  if ((s = check_device_ptr(input, "input", d, o)) != NORM_OK ||
      (s = check_device_ptr(hidden, "hidden", d, o)) != NORM_OK ||
      (s = check_device_ptr(output, "output", d, o)) != NORM_OK)
    return s;
  Workspace ws;
  if ((s = get_workspace(o, d.device, static_cast<cudaStream_t>(o->stream), &ws)) != NORM_OK) return s;
  cudaError_t e = launch_bpnn(input, hidden, output, in, hid, variant,
                              static_cast<cudaStream_t>(o->stream), d, ws.bp_ctr);
  return e == cudaSuccess ? NORM_OK : cuda_fail(e, "bpnn kernel launch");
}

NORM_API norm_status_t norm_coverage(int64_t n, int32_t index, int64_t* count, int64_t* prefix_len) {
  if (n < 0 || !count || !prefix_len) return fail(NORM_ERR_INVALID_VALUE, "bad argument");
  if (index != NORM_INDEX_LITERAL && index != NORM_INDEX_DENSE)
    return fail(NORM_ERR_INVALID_VALUE, "bad index mode");
  const Coverage c = coverage_of(n, index);
  *count = c.kind == COV_EMPTY ? 0 : c.count;
  *prefix_len = c.kind == COV_EMPTY ? 0 : (c.kind == COV_PREFIX ? c.L : -1);
  return NORM_OK;
}

NORM_API norm_status_t norm_workspace_bytes(int64_t n, const norm_opts_t* o, size_t* bytes) {
  (void)o;
  if (n < 0 || !bytes) return fail(NORM_ERR_INVALID_VALUE, "bad argument");
  *bytes = workspace_bytes();
  return NORM_OK;
}

NORM_API norm_status_t norm_algorithmic_bytes(int64_t n, int32_t index, int64_t* bytes) {
  int64_t count, prefix;
  norm_status_t s = norm_coverage(n, index, &count, &prefix);
  if (s != NORM_OK) return s;
  if (!bytes) return fail(NORM_ERR_INVALID_VALUE, "bytes is NULL");
  *bytes = 4 * n + 8 * count;  // read all of in once + read and write C(n)
  return NORM_OK;
}

NORM_API norm_status_t norm_debug_set_events(void* begin, void* end) {
  g_ev_begin = static_cast<cudaEvent_t>(begin);
  g_ev_end = static_cast<cudaEvent_t>(end);
  return NORM_OK;
}

NORM_API norm_status_t norm_cache_release(void) {
  int cur = -1;
  cudaGetDevice(&cur);
  {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    g_ws_gen.fetch_add(1, std::memory_order_acq_rel);  // invalidates every thread's memo
    for (auto& kv : g_ws_cache) {
      cudaSetDevice(kv.first.first);
      cudaDeviceSynchronize();
      cudaFree(kv.second);
    }
    g_ws_cache.clear();
  }
  {
    std::lock_guard<std::mutex> lk(g_hs_mu);
    for (auto& kv : g_hs_cache) {
      HostStage* h = kv.second;
      cudaSetDevice(kv.first.first);
      cudaDeviceSynchronize();
      cudaFree(h->resident);
      for (auto& r : h->ring) cudaFree(r);
      cudaFree(h->chunkS);
      cudaFree(h->ws);
      for (auto& ev : h->landed) cudaEventDestroy(ev);
      for (auto& ev : h->slot_free) cudaEventDestroy(ev);
      cudaEventDestroy(h->start);
      cudaStreamDestroy(h->copy);
      delete h;
    }
    g_hs_cache.clear();
  }
  if (cur >= 0) cudaSetDevice(cur);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? NORM_OK : cuda_fail(e, "norm_cache_release");
}

NORM_API const char* norm_status_string(norm_status_t s) {
  switch (s) {
    case NORM_OK: return "NORM_OK";
    case NORM_ERR_INVALID_VALUE: return "NORM_ERR_INVALID_VALUE";
    case NORM_ERR_OVERLAP: return "NORM_ERR_OVERLAP";
    case NORM_ERR_CUDA: return "NORM_ERR_CUDA";
    case NORM_ERR_NCCL: return "NORM_ERR_NCCL";
    case NORM_ERR_WORKSPACE: return "NORM_ERR_WORKSPACE";
    case NORM_ERR_UNSUPPORTED: return "NORM_ERR_UNSUPPORTED";
  }
  return "NORM_ERR_UNKNOWN";
}

NORM_API const char* norm_last_error(void) { return g_last_error.c_str(); }
