// backprop.cu — SURVEY §8(f) NEXT-4: Rodinia backprop `bpnn_layerforward`, the
// kernel of Fig. backprop that the paper uses to show barrier
// elimination (§4.1) and memory-to-register promotion across
// barriers (§4.2), run on B200 in four forms with identical
// fp32 arithmetic (same products, same tree order, no contraction), so all four
// are bitwise equal to each other and to the oracle:
//   PRINTED     — as printed: 16x16 block, shared `node`/`weights`, 8 barriers.
//   ELIMINATED  — the paper's optimisations applied by hand: "Unnecessary
//                 Barrier #1/#2" removed and "Unnecessary Store #1 / Load #1"
//                 forwarded through a register (6 barriers).
//   REGISTER    — B200-first: one thread per (block, column) keeps the column's
//                 16 products in registers and runs the same tree there: no
//                 shared memory, no barriers, coalesced along the column index.
//   TMA         — REGISTER's per-column arithmetic on tiles streamed into shared
//                 memory by cp.async.bulk (contiguous runs of 15 blocks + their
//                 inputs, 4-stage ring, 2 CTAs per SM, runs from a queue).
// Index expressions and the tree condition are Rodinia's (reading R18).
#include <cuda_runtime.h>

#include "stream_common.cuh"

namespace lnorm {

constexpr int BP_H = 16;  // HEIGHT = WIDTH = hid

__device__ __forceinline__ int64_t bp_index(int64_t by, int ty, int tx, int64_t hid) {
  return (hid + 1) * BP_H * by + (hid + 1) * ty + tx + 1 + (hid + 1);
}

__global__ void __launch_bounds__(BP_H * BP_H)
    bpnn_printed_kernel(const float* __restrict__ input, float* hidden, float* output, int64_t hid) {
  __shared__ float node[BP_H];
  __shared__ float weights[BP_H][BP_H];
  const int64_t by = blockIdx.x;  // Rodinia uses blockIdx.y (<= 65535 blocks); see R18
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t index = bp_index(by, ty, tx, hid);
  const int64_t index_in = BP_H * by + ty + 1;
  if (tx == 0) node[ty] = input[index_in];
  __syncthreads();  // Unnecessary Barrier #1
  weights[ty][tx] = hidden[index];  // Unnecessary Store #1
  __syncthreads();
  weights[ty][tx] = __fmul_rn(weights[ty][tx], node[ty]);  // Unnecessary Load #1
  __syncthreads();
  for (int i = 1; i <= 4; ++i) {  // log2(HEIGHT)
    const int p = 1 << i;
    if (ty % p == 0) weights[ty][tx] = __fadd_rn(weights[ty][tx], weights[ty + p / 2][tx]);
    __syncthreads();
  }
  hidden[index] = weights[ty][tx];
  __syncthreads();  // Unnecessary Barrier #2
  if (tx == 0) output[by * hid + ty] = weights[tx][ty];
}

__global__ void __launch_bounds__(BP_H * BP_H)
    bpnn_eliminated_kernel(const float* __restrict__ input, float* hidden, float* output, int64_t hid) {
  __shared__ float node[BP_H];
  __shared__ float weights[BP_H][BP_H];
  const int64_t by = blockIdx.x;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t index = bp_index(by, ty, tx, hid);
  if (tx == 0) node[ty] = input[BP_H * by + ty + 1];
  const float h = hidden[index];  // §4.2: the store/load pair becomes this register
  __syncthreads();                // (barrier #1 gone: M_before ∩ M†_after = ∅, §4.1)
  weights[ty][tx] = __fmul_rn(h, node[ty]);
  __syncthreads();
  for (int i = 1; i <= 4; ++i) {
    const int p = 1 << i;
    if (ty % p == 0) weights[ty][tx] = __fadd_rn(weights[ty][tx], weights[ty + p / 2][tx]);
    __syncthreads();
  }
  hidden[index] = weights[ty][tx];
  if (tx == 0) output[by * hid + ty] = weights[tx][ty];  // barrier #2 gone: the tree's last
}                                                          // barrier already orders weights[0][*]

// One thread per (block by, column tx): the column's 16 products live in
// registers and the printed tree runs on them in the printed order.
__global__ void __launch_bounds__(256)
    bpnn_register_kernel(const float* __restrict__ input, float* hidden, float* output,
                         int64_t hid, int64_t blocks) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t by = t >> 4;
  const int tx = (int)(t & 15);
  if (by >= blocks) return;
  float w[BP_H];
#pragma unroll
  for (int ty = 0; ty < BP_H; ++ty)
    w[ty] = __fmul_rn(hidden[bp_index(by, ty, tx, hid)], __ldg(input + BP_H * by + ty + 1));
#pragma unroll
  for (int i = 1; i <= 4; ++i) {
    const int p = 1 << i;
#pragma unroll
    for (int ty = 0; ty < BP_H; ty += p) w[ty] = __fadd_rn(w[ty], w[ty + p / 2]);
  }
#pragma unroll
  for (int ty = 0; ty < BP_H; ++ty) hidden[bp_index(by, ty, tx, hid)] = w[ty];
  output[by * hid + tx] = w[0];  // weights[0][tx]: this column's sum
}

// TMA variant (B200-first): the 16 x 17 tiles of consecutive blocks are one
// contiguous run of hidden (block by = floats [272 by + 17, 272 by + 289)), and
// their inputs one contiguous run of input (floats [16 by + 1, 16 by + 17)), so
// a run of BPT_RUN blocks is two cp.async.bulk copies into one stage of a
// BPT_STAGES-deep ring, two CTAs per SM — up to 2 x 4 x 17 KiB in flight per SM
// instead of the register form's scattered 4-byte loads (ncu: 64 % DRAM cycles
// active, long-scoreboard bound).  Runs come from a queue (claimed one ahead,
// stage-tagged; the last producer resets it).  TMA sources must be 16-byte
// aligned: each copy starts at the aligned address at or below the run (`lead`
// extra floats, < 4) and is rounded up to 16 bytes; the last block is left to
// the global-load path (CTA 0) so no copy reads past either array.  Each consumer
// thread owns one (block, column) item per run: it copies the column's 16 values
// (17-float row stride: conflict-free) and the block's 16 inputs from shared
// memory into registers, releases the stage, then computes the same products
// and tree as every variant and stores the 16 results and the column sum.
constexpr int BPT_RUN = 15;                          // blocks per run: 240 items <= 256 consumers
constexpr int BPT_HID_BYTES = 16384;                 // 15 * 1088 B + slack
constexpr int BPT_STAGE = BPT_HID_BYTES + 1024;      // + 15 * 64 B of inputs + slack
#ifndef NORM_BPT_STAGES  // probe builds only (ring A/B): -DNORM_BPT_STAGES=6 -DNORM_BPT_CTAS=3
#define NORM_BPT_STAGES 4
#endif
#ifndef NORM_BPT_CTAS
#define NORM_BPT_CTAS 2
#endif
constexpr int BPT_STAGES = NORM_BPT_STAGES, BPT_CTAS = NORM_BPT_CTAS;
constexpr size_t BPT_SMEM = (size_t)BPT_STAGES * BPT_STAGE;
static_assert(BPT_RUN * 1088 + 16 <= BPT_HID_BYTES && BPT_RUN * 64 + 16 <= 1024, "a run fits a stage");
static_assert(BPT_RUN * BP_H <= BK_CONSUMERS, "one item per consumer thread");

__device__ __forceinline__ void bpnn_finish(float* hidden, float* output, int64_t hid, int64_t by, int tx,
                                            float* w, const float* x) {
#pragma unroll
  for (int ty = 0; ty < BP_H; ++ty) w[ty] = __fmul_rn(w[ty], x[ty]);
#pragma unroll
  for (int i = 1; i <= 4; ++i) {
    const int p = 1 << i;
#pragma unroll
    for (int ty = 0; ty < BP_H; ty += p) w[ty] = __fadd_rn(w[ty], w[ty + p / 2]);
  }
#pragma unroll
  for (int ty = 0; ty < BP_H; ++ty) hidden[bp_index(by, ty, tx, hid)] = w[ty];
  output[by * hid + tx] = w[0];
}

__device__ __forceinline__ const char* align16_down(const void* p, int* lead_floats) {
  const char* c = static_cast<const char*>(p);
  const char* a = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(c) & ~(uintptr_t)15);
  *lead_floats = (int)((c - a) >> 2);
  return a;
}

__global__ void __launch_bounds__(BK_THREADS, BPT_CTAS)
    bpnn_tma_kernel(const float* __restrict__ input, float* hidden, float* output, int64_t hid,
                    int64_t blocks, unsigned* ctr) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ __align__(8) uint64_t full[BPT_STAGES], empty[BPT_STAGES];
  __shared__ int64_t stage_run[BPT_STAGES];
  __shared__ int stage_lead[BPT_STAGES][2];
  auto r = bulk_ring_init<BPT_STAGES, BPT_STAGE>(ring, full, empty);
  const int64_t tma_blocks = blocks - 1;  // the last block: CTA 0, global loads
  const int64_t runs = (tma_blocks + BPT_RUN - 1) / BPT_RUN;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      int64_t next = (int64_t)atomicAdd(ctr, 1u);
      while (next < runs) {
        const int64_t run = next;
        next = (int64_t)atomicAdd(ctr, 1u);
        const int64_t b0 = run * BPT_RUN;
        const int64_t nb = tma_blocks - b0 < BPT_RUN ? tma_blocks - b0 : BPT_RUN;
        int lh, li;
        const char* ah = align16_down(hidden + 272 * b0 + 17, &lh);
        const char* ai = align16_down(input + BP_H * b0 + 1, &li);
        const unsigned bh = (unsigned)(((size_t)nb * 1088 + (size_t)lh * 4 + 15) & ~(size_t)15);
        const unsigned bi = (unsigned)(((size_t)nb * 64 + (size_t)li * 4 + 15) & ~(size_t)15);
        if (r.issued >= BPT_STAGES) stage_acquire(&r.empty[r.stage], r.phase ^ 1);
        stage_run[r.stage] = run;
        stage_lead[r.stage][0] = lh;
        stage_lead[r.stage][1] = li;
        mbar_arrive_expect_tx(&r.full[r.stage], bh + bi);
        unsigned char* dst = r.buf + (size_t)r.stage * BPT_STAGE;
        bulk_g2s(dst, ah, bh, &r.full[r.stage]);
        bulk_g2s(dst + BPT_HID_BYTES, ai, bi, &r.full[r.stage]);
        ++r.issued;
        r.advance();
      }
      __threadfence();  // this CTA's claims on ctr[0] precede its count on ctr[1]
      if (atomicAdd(ctr + 1, 1u) == gridDim.x - 1) {  // every producer has claimed its last run
        __threadfence();  // every other CTA's claims are visible before the reset
        ctr[0] = 0u;
        ctr[1] = 0u;
      }
      if (r.issued >= BPT_STAGES) stage_acquire(&r.empty[r.stage], r.phase ^ 1);
      stage_run[r.stage] = -1;  // end marker
      mbar_arrive(&r.full[r.stage]);
    }
    return;
  }
  const int ct = threadIdx.x - 32;
  const int bi = ct >> 4, tx = ct & 15;
  for (;;) {
    mbar_wait(&r.full[r.stage], r.phase);
    const int64_t run = *(volatile int64_t*)&stage_run[r.stage];
    if (run < 0) break;
    const int lh = *(volatile int*)&stage_lead[r.stage][0];
    const int li = *(volatile int*)&stage_lead[r.stage][1];
    const unsigned char* sb = r.buf + (size_t)r.stage * BPT_STAGE;
    const float* tile = reinterpret_cast<const float*>(sb) + lh + 272 * bi;
    const float* xin = reinterpret_cast<const float*>(sb + BPT_HID_BYTES) + li + BP_H * bi;
    const int64_t b0 = run * BPT_RUN;
    const bool mine = bi < BPT_RUN && b0 + bi < tma_blocks;
    float w[BP_H], x[BP_H];
    if (mine) {
#pragma unroll
      for (int ty = 0; ty < BP_H; ++ty) {
        w[ty] = tile[17 * ty + tx + 1];
        x[ty] = xin[ty];
      }
    }
    stage_release(&r.empty[r.stage]);  // values are in registers: the producer may refill
    r.advance();
    if (mine) bpnn_finish(hidden, output, hid, b0 + bi, tx, w, x);
  }
  if (blockIdx.x == 0 && ct < BP_H) {
    const int64_t by = blocks - 1;
    float w[BP_H], x[BP_H];
#pragma unroll
    for (int ty = 0; ty < BP_H; ++ty) {
      w[ty] = hidden[bp_index(by, ty, ct, hid)];
      x[ty] = __ldg(input + BP_H * by + ty + 1);
    }
    bpnn_finish(hidden, output, hid, by, ct, w, x);
  }
}

cudaError_t launch_bpnn(const float* input, float* hidden, float* output, int64_t in, int64_t hid,
                        int variant, cudaStream_t st, const DeviceInfo& d, unsigned* ctr) {
  const int64_t blocks = in / BP_H;
  if (blocks == 0) return cudaSuccess;
  if (variant == NORM_BP_TMA && blocks >= 2 && ctr) {
    static int configured[64] = {0};
    if (d.device < 64 && !configured[d.device]) {
      cudaError_t e = cudaFuncSetAttribute(bpnn_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)BPT_SMEM);
      if (e != cudaSuccess) return e;
      configured[d.device] = 1;
    }
    bpnn_tma_kernel<<<d.sms * BPT_CTAS, BK_THREADS, BPT_SMEM, st>>>(input, hidden, output, hid, blocks, ctr);
    return cudaGetLastError();
  }
  if (variant == NORM_BP_REGISTER || variant == NORM_BP_TMA) {
    const int64_t threads = blocks * BP_H;
    bpnn_register_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(input, hidden, output,
                                                                          hid, blocks);
  } else if (variant == NORM_BP_ELIMINATED) {
    bpnn_eliminated_kernel<<<(unsigned)blocks, dim3(BP_H, BP_H), 0, st>>>(input, hidden, output, hid);
  } else {
    bpnn_printed_kernel<<<(unsigned)blocks, dim3(BP_H, BP_H), 0, st>>>(input, hidden, output, hid);
  }
  return cudaGetLastError();
}

}  // namespace lnorm
