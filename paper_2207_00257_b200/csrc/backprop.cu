// backprop.cu — SURVEY §8(f) NEXT-4: Rodinia backprop `bpnn_layerforward`, the
// kernel of Fig. backprop that the paper uses to show barrier
// elimination (§4.1) and memory-to-register promotion across
// barriers (§4.2), run on B200 in three forms with identical
// fp32 arithmetic (same products, same tree order, no contraction), so all three
// are bitwise equal to each other and to the oracle:
//   PRINTED     — as printed: 16x16 block, shared `node`/`weights`, 8 barriers.
//   ELIMINATED  — the paper's optimisations applied by hand: "Unnecessary
//                 Barrier #1/#2" removed and "Unnecessary Store #1 / Load #1"
//                 forwarded through a register (6 barriers).
//   REGISTER    — B200-first: one thread per (block, column) keeps the column's
//                 16 products in registers and runs the same tree there: no
//                 shared memory, no barriers, coalesced along the column index.
// Index expressions and the tree condition are Rodinia's (reading R18).
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "norm_internal.h"

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

cudaError_t launch_bpnn(const float* input, float* hidden, float* output, int64_t in, int64_t hid,
                        int variant, cudaStream_t st) {
  const int64_t blocks = in / BP_H;
  if (blocks == 0) return cudaSuccess;
  if (variant == NORM_BP_REGISTER) {
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
