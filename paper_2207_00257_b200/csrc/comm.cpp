// comm.cpp — multi-GPU layer of libnorm: shard planner, NCCL communicator, the
// fused peer-memory exchange, and the sharded normalize (one process per GPU,
// NVLink 5 / NVSwitch).
//
// The method's only cross-GPU exchange is the hoisted `sum`:
// each rank reduces its shard to an fp64 partial S_k (8 bytes), the W partials
// reach every rank, and the scale kernel's prologue combines them in rank order
// — an all-reduce whose order is pinned, so every rank divides by bit-identical
// s, run after run.  Three carriers: the reduce kernel's own
// peer stores into every rank's mailbox (norm_launch_sharded_peer: no collective
// launch at all), ncclAllGather / ncclAllReduce (norm_launch_sharded), or any
// caller collective between norm_shard_partial and norm_shard_finish.  The
// message is 8 bytes, pure latency; the scale cannot start before s exists.
#include <cuda_runtime.h>
#include <nccl.h>
#include <string.h>

#include <string>
#include <vector>

#include "libnorm.h"
#include "norm_internal.h"

#define NORM_API extern "C" __attribute__((visibility("default")))

using namespace lnorm;

struct norm_comm {
  ncclComm_t nccl = nullptr;
  int world = 0, rank = 0, device = -1;
  int mode = NORM_COMM_ALLGATHER;
  double* send = nullptr;  // [1] this rank's partial
  double* recv = nullptr;  // [world] all partials, rank order
  void* ws = nullptr;      // reduce workspace (zeroed)
};

static norm_status_t nccl_fail(ncclResult_t r, const char* what) {
  return fail(NORM_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

NORM_API norm_status_t norm_comm_unique_id(unsigned char id[128]) {
  if (!id) return fail(NORM_ERR_INVALID_VALUE, "id is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id, &u, 128);
  return NORM_OK;
}

NORM_API norm_status_t norm_comm_init(norm_comm_t** comm, int32_t world, int32_t rank,
                                      const unsigned char id[128]) {
  if (!comm || !id || world < 1 || rank < 0 || rank >= world)
    return fail(NORM_ERR_INVALID_VALUE, "bad comm arguments");
  *comm = nullptr;
  norm_comm* c = new norm_comm();
  c->world = world;
  c->rank = rank;
  cudaError_t e = cudaGetDevice(&c->device);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaGetDevice");
  }
  const size_t bytes = 256 + (size_t)world * sizeof(double);
  char* buf = nullptr;
  if ((e = cudaMalloc(&buf, bytes + workspace_bytes())) != cudaSuccess) {
    delete c;
    cudaGetLastError();
    return fail(NORM_ERR_WORKSPACE, "comm scratch cudaMalloc failed");
  }
  cudaMemset(buf, 0, bytes + workspace_bytes());
  c->send = reinterpret_cast<double*>(buf);
  c->recv = reinterpret_cast<double*>(buf + 256);
  c->ws = buf + ((bytes + 255) / 256) * 256;
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclResult_t r = ncclCommInitRank(&c->nccl, world, u, rank);
  if (r != ncclSuccess) {
    cudaFree(buf);
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *comm = c;
  return NORM_OK;
}

NORM_API norm_status_t norm_comm_set_mode(norm_comm_t* c, int32_t mode) {
  if (!c || (mode != NORM_COMM_ALLGATHER && mode != NORM_COMM_ALLREDUCE))
    return fail(NORM_ERR_INVALID_VALUE, "bad comm mode");
  c->mode = mode;
  return NORM_OK;
}

NORM_API norm_status_t norm_comm_destroy(norm_comm_t* c) {
  if (!c) return NORM_OK;
  norm_status_t s = NORM_OK;
  if (c->nccl) {
    ncclResult_t r = ncclCommDestroy(c->nccl);
    if (r != ncclSuccess) s = nccl_fail(r, "ncclCommDestroy");
  }
  cudaFree(c->send);
  delete c;
  return s;
}

static int64_t round8(int64_t x) { return (x / 8) * 8; }

// Slice [lo, hi) into `world` contiguous pieces whose lengths (except the last)
// are multiples of 8 elements, so each piece keeps the 32-byte phase of `lo`.
static void split(int64_t lo, int64_t hi, int world, int k, int64_t* b, int64_t* e) {
  const int64_t len = hi - lo;
  *b = k == 0 ? lo : lo + round8(len * k / world);
  *e = k == world - 1 ? hi : lo + round8(len * (k + 1) / world);
  if (*e < *b) *e = *b;
}

NORM_API norm_status_t norm_plan_shards(int64_t n, int32_t world, int32_t index,
                                        int32_t coverage_balanced, norm_shard_t* plan) {
  if (n < 0 || world < 1 || !plan) return fail(NORM_ERR_INVALID_VALUE, "bad plan arguments");
  if (index != NORM_INDEX_LITERAL && index != NORM_INDEX_DENSE)
    return fail(NORM_ERR_INVALID_VALUE, "bad index mode");
  const Coverage cov = coverage_of(n, index);
  const bool two = coverage_balanced && index == NORM_INDEX_LITERAL && cov.kind == COV_PREFIX &&
                   cov.L < n && world > 1;
  for (int k = 0; k < world; ++k) {
    norm_shard_t& p = plan[k];
    memset(&p, 0, sizeof p);
    int64_t b, e;
    if (two) {
      split(0, cov.L, world, k, &b, &e);
      if (e > b) { p.begin[p.nranges] = b; p.len[p.nranges] = e - b; p.nranges++; }
      split(cov.L, n, world, k, &b, &e);
      if (e > b) { p.begin[p.nranges] = b; p.len[p.nranges] = e - b; p.nranges++; }
    } else {
      split(0, n, world, k, &b, &e);
      if (e > b) { p.begin[0] = b; p.len[0] = e - b; p.nranges = 1; }
    }
  }
  return NORM_OK;
}

// Validate a shard; *local = number of local elements.
static norm_status_t check_shard(float* out_local, const float* in_local, const norm_shard_t* mine,
                                 int64_t n_global, const norm_opts_t* o, int64_t* local) {
  if (!mine) return fail(NORM_ERR_INVALID_VALUE, "shard is NULL");
  if (o->index != NORM_INDEX_LITERAL && o->index != NORM_INDEX_DENSE)
    return fail(NORM_ERR_INVALID_VALUE, "bad index mode");
  if (n_global < 0 || mine->nranges < 0 || mine->nranges > 2)
    return fail(NORM_ERR_INVALID_VALUE, "bad shard");
  int64_t n = 0, prev_end = 0;
  for (int k = 0; k < mine->nranges; ++k) {
    if (mine->len[k] < 0 || mine->begin[k] < prev_end || mine->begin[k] + mine->len[k] > n_global)
      return fail(NORM_ERR_INVALID_VALUE, "shard ranges must be ascending, disjoint, inside [0, n)");
    prev_end = mine->begin[k] + mine->len[k];
    n += mine->len[k];
  }
  if (n > 0) {
    if (!out_local || !in_local) return fail(NORM_ERR_INVALID_VALUE, "NULL local buffer");
    if ((reinterpret_cast<uintptr_t>(out_local) | reinterpret_cast<uintptr_t>(in_local)) & 3u)
      return fail(NORM_ERR_INVALID_VALUE, "pointer not 4-byte aligned");
    uintptr_t a = reinterpret_cast<uintptr_t>(out_local), b = reinterpret_cast<uintptr_t>(in_local);
    if (a != b && a < b + n * 4 && b < a + n * 4)
      return fail(NORM_ERR_OVERLAP, "out_local and in_local partially overlap");
  }
  const Coverage cov = coverage_of(n_global, o->index);
  if (o->index == NORM_INDEX_LITERAL && cov.G > 2147483647LL)
    return fail(NORM_ERR_UNSUPPORTED, "literal launch needs > 2^31-1 blocks");
  *local = n;
  return NORM_OK;
}

// The locally covered elements as a prefix [0, Lloc) of the local buffer (the
// layout the fused kernel handles), or -1 if they are not one.  Literal mode's
// coverage-balanced plan gives range 0 inside [0, L) and range 1 outside it, so
// Lloc = len[0]; the one-range plan gives rank 0 the prefix.
static int64_t local_covered_prefix(const norm_shard_t* mine, const Coverage& cov) {
  if (cov.kind != COV_PREFIX) return -1;
  int64_t off = 0, Lloc = 0;
  bool ended = false;
  for (int k = 0; k < mine->nranges; ++k) {
    const int64_t gb = mine->begin[k], len = mine->len[k];
    const int64_t ce = gb + len < cov.L ? gb + len : cov.L;
    const int64_t clen = ce > gb ? ce - gb : 0;
    if (clen > 0) {
      if (ended || off != Lloc) return -1;
      Lloc += clen;
    }
    if (clen < len) ended = true;
    off += len;
  }
  return Lloc;
}

// Step 3 of the sharded path: combine the W partials in rank order (scale
// prologue) and scale the locally covered elements of each owned range.
static norm_status_t shard_finish(float* out_local, const float* in_local, const norm_shard_t* mine,
                                  int64_t n_global, const double* partials, int world,
                                  const norm_opts_t* o, const DeviceInfo& d, const Workspace& ws,
                                  unsigned long long epoch = 0) {
  const Coverage cov = coverage_of(n_global, o->index);
  cudaStream_t st = static_cast<cudaStream_t>(o->stream);
  float* so = o->sum_out;
  double* so64 = o->sum_out_f64;
  int64_t off = 0;
  bool launched = false;
  // With the mailbox exchange the kernel before the first scale is this rank's
  // reduce: launch the scale as its programmatic dependent (as on one GPU), so
  // its TMA producer streams `in` while the reduce drains.  After an NCCL
  // kernel or a caller's collective there is no such edge.
  bool pdl = epoch != 0;
  cudaError_t e;
  for (int k = 0; k < mine->nranges; ++k) {
    const int64_t gb = mine->begin[k], len = mine->len[k];
    if (cov.kind == COV_PREFIX) {
      const int64_t ce = gb + len < cov.L ? gb + len : cov.L;
      const int64_t clen = ce > gb ? ce - gb : 0;
      if (clen > 0) {
        e = launch_scale(out_local + off, in_local + off, clen, partials, world, so, so64, d, pdl, st,
                         epoch, ws.scale_ctr);
        pdl = false;
        if (e != cudaSuccess) return cuda_fail(e, "scale_kernel launch");
        so = nullptr;
        so64 = nullptr;
        launched = true;
      }
    } else if (cov.kind == COV_RESIDUE && len > 0) {
      e = launch_scale_residue(out_local + off, in_local + off, len, gb, cov.G, partials, world, so,
                               so64, pdl, st, epoch);
      pdl = false;
      if (e != cudaSuccess) return cuda_fail(e, "scale_residue launch");
      so = nullptr;
      so64 = nullptr;
      launched = true;
    }
    off += len;
  }
  // Nothing covered here, but the caller wants s -- or the mailbox exchange needs
  // every rank to wait for every epoch (see publish_partial's parity argument).
  if (!launched && (so || so64 || epoch)) {
    e = launch_scale(out_local, in_local, 0, partials, world, so, so64, d, pdl, st, epoch, ws.scale_ctr);
    if (e != cudaSuccess) return cuda_fail(e, "scale_kernel launch");
  }
  return NORM_OK;
}

NORM_API norm_status_t norm_launch_sharded(norm_comm_t* c, float* out_local, const float* in_local,
                                           const norm_shard_t* mine, int64_t n_global,
                                           const norm_opts_t* o) {
  static const norm_opts_t kDef = NORM_OPTS_INIT;
  if (!o) o = &kDef;
  if (!c) return fail(NORM_ERR_INVALID_VALUE, "comm is NULL");
  int64_t local = 0;
  norm_status_t s = check_opts(o);
  if (s != NORM_OK) return s;
  if ((s = check_shard(out_local, in_local, mine, n_global, o, &local)) != NORM_OK) return s;
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  if (d.device != c->device) return fail(NORM_ERR_INVALID_VALUE, "current device != comm device");
  if (local > 0 && (s = check_io_ptrs(out_local, in_local, o, d)) != NORM_OK) return s;
  if (local == 0 && (s = check_out_ptrs(o, d)) != NORM_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(o->stream);
  Workspace ws = workspace_carve(c->ws);
  NvtxRange rr("norm_launch_sharded");
  // 1. local partial over all owned elements (the hoisted `sum`, restricted to this rank)
  {
    NvtxRange r("libnorm:reduce");
    ev_begin(st);
    cudaError_t e = launch_reduce(in_local, local, ws, c->send, d, st);
    if (e != cudaSuccess) return cuda_fail(e, "reduce_kernel launch");
    ev_end(st);
  }
  // 2. exchange: W x 8 bytes over NVLink
  if (c->mode == NORM_COMM_ALLREDUCE) {  // NCCL's own summation order; one partial back
    {
      NvtxRange r("libnorm:exchange:ncclAllReduce");
      ncclResult_t nr = ncclAllReduce(c->send, c->recv, 1, ncclFloat64, ncclSum, c->nccl, st);
      if (nr != ncclSuccess) return nccl_fail(nr, "ncclAllReduce");
    }
    NvtxRange r("libnorm:scale");
    return shard_finish(out_local, in_local, mine, n_global, c->recv, 1, o, d, ws);
  }
  {
    NvtxRange r("libnorm:exchange:ncclAllGather");
    ncclResult_t nr = ncclAllGather(c->send, c->recv, 1, ncclFloat64, c->nccl, st);
    if (nr != ncclSuccess) return nccl_fail(nr, "ncclAllGather");
  }
  // 3. rank-order combine + scale
  NvtxRange r("libnorm:scale");
  return shard_finish(out_local, in_local, mine, n_global, c->recv, c->world, o, d, ws);
}

NORM_API norm_status_t norm_shard_partial(double* partial, const float* in_local, int64_t n_local,
                                          const norm_opts_t* o) {
  static const norm_opts_t kDef = NORM_OPTS_INIT;
  if (!o) o = &kDef;
  if (!partial || n_local < 0 || (n_local > 0 && !in_local))
    return fail(NORM_ERR_INVALID_VALUE, "bad partial arguments");
  if (reinterpret_cast<uintptr_t>(in_local) & 3u)
    return fail(NORM_ERR_INVALID_VALUE, "pointer not 4-byte aligned");
  norm_status_t s = check_opts(o);
  if (s != NORM_OK) return s;
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  // the partial is written by the kernel: it must be device memory of this device
  norm_opts_t po = NORM_OPTS_INIT;
  po.flags = o->flags;
  po.sum_out_f64 = partial;
  if ((s = check_out_ptrs(&po, d)) != NORM_OK) return s;
  if (n_local > 0 && (s = check_io_ptrs(in_local, in_local, o, d)) != NORM_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(o->stream);
  Workspace ws;
  s = get_workspace(o, d.device, st, &ws);
  if (s != NORM_OK) return s;
  ev_begin(st);
  cudaError_t e = launch_reduce(in_local, n_local, ws, partial, d, st);
  if (e != cudaSuccess) return cuda_fail(e, "reduce_kernel launch");
  ev_end(st);
  return NORM_OK;
}

NORM_API norm_status_t norm_shard_finish(float* out_local, const float* in_local,
                                         const norm_shard_t* mine, int64_t n_global,
                                         const double* partials, int32_t world,
                                         const norm_opts_t* o) {
  static const norm_opts_t kDef = NORM_OPTS_INIT;
  if (!o) o = &kDef;
  if (!partials || world < 1) return fail(NORM_ERR_INVALID_VALUE, "bad partials");
  int64_t local = 0;
  norm_status_t s = check_opts(o);
  if (s != NORM_OK) return s;
  if ((s = check_shard(out_local, in_local, mine, n_global, o, &local)) != NORM_OK) return s;
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  if (local > 0 && (s = check_io_ptrs(out_local, in_local, o, d)) != NORM_OK) return s;
  if (local == 0 && (s = check_out_ptrs(o, d)) != NORM_OK) return s;
  Workspace ws;
  s = get_workspace(o, d.device, static_cast<cudaStream_t>(o->stream), &ws);
  if (s != NORM_OK) return s;
  return shard_finish(out_local, in_local, mine, n_global, partials, world, o, d, ws);
}

// ======================================================= fused peer exchange
// The B200-native replacement of the 8-byte ncclAllGather: the reduce kernel's
// last CTA stores the rank partial directly into every rank's mailbox through
// peer memory (CUDA IPC mappings; NVLink on an NVSwitch box) and the scale
// kernel's prologue waits on the local mailbox's epoch flags.  No collective
// launch sits between the two kernels.

struct norm_peer {
  int world = 0, rank = 0, device = -1;
  double* mail = nullptr;        // local mailbox: [2][world] x {partial, epoch}
  double** peer_dev = nullptr;   // device array: mailbox of rank r as mapped here
  std::vector<void*> opened;     // IPC mappings to close
  unsigned long long epoch = 0;
  bool broken = false;           // a call failed after publishing: epochs out of step
  void* ws = nullptr;            // reduce workspace
};

NORM_API norm_status_t norm_peer_create(norm_peer_t** out, int32_t world, int32_t rank,
                                        unsigned char handle[64]) {
  if (!out || !handle || world < 1 || rank < 0 || rank >= world)
    return fail(NORM_ERR_INVALID_VALUE, "bad peer arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
  *out = nullptr;
  norm_peer* p = new norm_peer();
  p->world = world;
  p->rank = rank;
  cudaError_t e = cudaGetDevice(&p->device);
  const size_t mail_bytes = ((size_t)2 * world * 2 * sizeof(double) + 4095) & ~(size_t)4095;
  if (e == cudaSuccess) e = cudaMalloc(&p->mail, mail_bytes);
  if (e == cudaSuccess) e = cudaMemset(p->mail, 0, mail_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&p->peer_dev, (size_t)world * sizeof(double*));
  if (e == cudaSuccess) e = cudaMalloc(&p->ws, workspace_bytes());
  if (e == cudaSuccess) e = cudaMemset(p->ws, 0, workspace_bytes());
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p->mail);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaFree(p->mail);
    cudaFree(p->peer_dev);
    cudaFree(p->ws);
    delete p;
    return cuda_fail(e, "norm_peer_create");
  }
  memcpy(handle, &h, 64);
  *out = p;
  return NORM_OK;
}

NORM_API norm_status_t norm_peer_connect(norm_peer_t* p, const unsigned char* handles) {
  if (!p || !handles) return fail(NORM_ERR_INVALID_VALUE, "bad peer arguments");
  std::vector<double*> ptrs(p->world);
  for (int r = 0; r < p->world; ++r) {
    if (r == p->rank) {
      ptrs[r] = p->mail;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + (size_t)r * 64, 64);
    void* q = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return cuda_fail(e, "cudaIpcOpenMemHandle (peer mailbox)");
    }
    p->opened.push_back(q);
    ptrs[r] = static_cast<double*>(q);
  }
  cudaError_t e = cudaMemcpy(p->peer_dev, ptrs.data(), (size_t)p->world * sizeof(double*),
                             cudaMemcpyHostToDevice);
  return e == cudaSuccess ? NORM_OK : cuda_fail(e, "peer table upload");
}

NORM_API norm_status_t norm_peer_destroy(norm_peer_t* p) {
  if (!p) return NORM_OK;
  cudaDeviceSynchronize();
  for (void* q : p->opened) cudaIpcCloseMemHandle(q);
  cudaFree(p->mail);
  cudaFree(p->peer_dev);
  cudaFree(p->ws);
  delete p;
  return NORM_OK;
}

NORM_API norm_status_t norm_launch_sharded_peer(norm_peer_t* p, float* out_local,
                                                const float* in_local, const norm_shard_t* mine,
                                                int64_t n_global, const norm_opts_t* o) {
  static const norm_opts_t kDef = NORM_OPTS_INIT;
  if (!o) o = &kDef;
  if (!p) return fail(NORM_ERR_INVALID_VALUE, "peer is NULL");
  if (p->broken)
    return fail(NORM_ERR_CUDA, "peer handle broken by an earlier failed call: destroy and recreate it on every rank");
  int64_t local = 0;
  norm_status_t s = check_opts(o);
  if (s != NORM_OK) return s;
  if ((s = check_shard(out_local, in_local, mine, n_global, o, &local)) != NORM_OK) return s;
  DeviceInfo d;
  if ((s = check_device(&d)) != NORM_OK) return s;
  if (d.device != p->device) return fail(NORM_ERR_INVALID_VALUE, "current device != peer device");
  if (local > 0 && (s = check_io_ptrs(out_local, in_local, o, d)) != NORM_OK) return s;
  if (local == 0 && (s = check_out_ptrs(o, d)) != NORM_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(o->stream);
  // The epoch is committed only once this rank's kernels are enqueued; a failure
  // after the publishing kernel was enqueued leaves the peers one epoch ahead of
  // us, so the handle is marked broken instead (include/libnorm.h).
  const unsigned long long epoch = p->epoch + 1;
  Workspace ws = workspace_carve(p->ws);
  const PeerPost post{p->peer_dev, p->rank, p->world, epoch};
  // One fused kernel per rank (reduce, grid barrier, publish + mailbox wait,
  // scale) when the local covered elements are a prefix of the local buffer and
  // the per-rank AUTO rule picks it (e.g. literal 2^32 at W = 8: 2 GiB + 64 MiB
  // covered per rank); otherwise reduce -> scale as below.  Both publish and
  // wait once per epoch, so ranks may take different paths.
  const Coverage gcov = coverage_of(n_global, o->index);
  const int64_t Lloc = local_covered_prefix(mine, gcov);
  int path = o->path;
  if (path == NORM_PATH_AUTO) path = auto_path(local, Lloc, Lloc >= 0, d);
  if (path == NORM_PATH_CLUSTER || path == NORM_PATH_SMALL) path = NORM_PATH_MID;  // need the mailbox step
  if ((path == NORM_PATH_FUSED || path == NORM_PATH_MID) && Lloc >= 0 && local > 0) {
    Coverage lc{};
    lc.kind = COV_PREFIX;
    lc.n = local;
    lc.L = lc.count = Lloc;
    lc.G = (local + 31) / 32;
    NvtxRange r(path == NORM_PATH_MID ? "libnorm:mid+peer-exchange" : "libnorm:fused+peer-exchange");
    ev_begin(st);
    cudaError_t e = path == NORM_PATH_MID
                        ? launch_mid(out_local, in_local, lc, ws, o->sum_out, o->sum_out_f64, d, st, post, p->mail)
                        : launch_fused(out_local, in_local, lc, ws, o->sum_out, o->sum_out_f64, d, st, post,
                                       p->mail);
    if (e != cudaSuccess) return cuda_fail(e, "fused / mid kernel cooperative launch");  // nothing enqueued
    ev_end(st);
    p->epoch = epoch;
    return NORM_OK;
  }
  {
    NvtxRange r("libnorm:reduce+peer-publish");
    ev_begin(st);
    cudaError_t e = launch_reduce(in_local, local, ws, ws.S, d, st, post);
    if (e != cudaSuccess) return cuda_fail(e, "reduce_kernel launch");  // nothing enqueued
    ev_end(st);
  }
  NvtxRange r("libnorm:peer-wait+scale");
  s = shard_finish(out_local, in_local, mine, n_global, p->mail, p->world, o, d, ws, epoch);
  if (s != NORM_OK) {
    p->broken = true;  // the reduce has published this epoch; our scale did not consume it
    return s;
  }
  p->epoch = epoch;
  return NORM_OK;
}
