// scripts/microbench_l2retain.cu — design-space probe (not product code): does an
// L2::evict_last read survive a long evict_first / normal stream, does the bench's
// L2 flush evict it, and does applypriority.L2::evict_normal demote it?  Prints the
// time to re-read a window W after each scenario (HBM ~ W / 7.5 TB/s, L2 faster).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_2207_00257_b200/csrc scripts/microbench_l2retain.cu -o mb_l2
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "device_common.cuh"

using namespace lnorm;

// mode 0: ld.global.nc (no hint); 1: evict_last policy; 2: evict_first policy
__global__ void __launch_bounds__(512) rd(const float* p, int64_t nv, int mode, double* out) {
  const uint64_t pol = mode == 1 ? policy_evict_last() : policy_evict_first();
  double acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    f8 v = mode == 0 ? ld8_stream(p + i * 8) : ld8_policy(p + i * 8, pol);
    acc += sum8(v);
  }
  if (acc == 12345.678) out[0] = acc;  // keep the loads
}

__global__ void apply_normal(const float* p, int64_t bytes) {
  const char* c = reinterpret_cast<const char*>(p);
  for (int64_t o = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 128; o < bytes;
       o += (int64_t)gridDim.x * blockDim.x * 128)
    asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(c + o) : "memory");
}

int sms;
double* dout;

void read(const float* p, int64_t bytes, int mode) {
  rd<<<sms * 4, 512>>>(p, bytes / 32, mode, dout);
}

float time_read(const float* p, int64_t bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  read(p, bytes, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms * 1000.f;
}

int main() {
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  int persist_max;
  cudaDeviceGetAttribute(&persist_max, cudaDevAttrMaxPersistingL2CacheSize, 0);
  size_t persist_cur = 0;
  cudaDeviceGetLimit(&persist_cur, cudaLimitPersistingL2CacheSize);
  printf("L2 %d bytes, max persisting %d, current persisting limit %zu\n", l2, persist_max, persist_cur);
  const int64_t XB = 4ll << 30;
  float* X;
  cudaMalloc(&X, XB);
  cudaMemset(X, 0, XB);
  cudaMalloc(&dout, 64);
  char* fw;
  float* fr;
  cudaMalloc(&fw, 256 << 20);
  cudaMalloc(&fr, 256 << 20);
  cudaMemset(fr, 0, 256 << 20);
  auto flush = [&] {
    cudaMemsetAsync(fw, 1, 256 << 20);
    read(fr, 256 << 20, 0);
  };
  auto bigflush = [&] {  // 1 GiB normal stream: evicts everything normal
    read(X + (3ll << 28), 1ll << 30, 0);
  };
  const float* S = X + (1ll << 26);  // stream region: [256 MiB, 4 GiB)
  const int64_t SB = XB - (256ll << 20);
  for (int64_t wmib : {32, 64, 96}) {
    const int64_t W = wmib << 20;
    struct Sc {
      const char* name;
      int id;
    } sc[] = {{"cold (after 1 GiB stream + flush)", 0},
              {"hot (W just read, normal)", 1},
              {"W evict_last; stream 3.75 GiB normal", 2},
              {"W evict_last; stream 3.75 GiB evict_first", 3},
              {"W normal; stream 3.75 GiB evict_first", 4},
              {"W evict_last; applypriority normal; stream evict_first", 5},
              {"W evict_last; bench flush (256 MiB memset + 256 MiB read)", 6},
              {"W evict_last; then re-read W evict_first; stream evict_first", 7},
              {"W evict_last; then re-read W no-hint; stream evict_first", 8}};
    for (auto& s : sc) {
      std::vector<float> t;
      for (int rep = 0; rep < 9; ++rep) {
        bigflush();
        flush();
        // demote anything a previous scenario left at evict_last
        apply_normal<<<sms * 4, 256>>>(X, XB);
        bigflush();
        flush();
        switch (s.id) {
          case 0: break;
          case 1: read(X, W, 0); break;
          case 2: read(X, W, 1); read(S, SB, 0); break;
          case 3: read(X, W, 1); read(S, SB, 2); break;
          case 4: read(X, W, 0); read(S, SB, 2); break;
          case 5: read(X, W, 1); apply_normal<<<sms * 4, 256>>>(X, W); read(S, SB, 2); break;
          case 6: read(X, W, 1); flush(); break;
          case 7: read(X, W, 1); read(X, W, 2); read(S, SB, 2); break;
          case 8: read(X, W, 1); read(X, W, 0); read(S, SB, 2); break;
        }
        cudaDeviceSynchronize();
        t.push_back(time_read(X, W));
      }
      std::sort(t.begin(), t.end());
      printf("W=%3lld MiB  %-60s re-read %8.2f us (min %7.2f)  -> %7.0f GB/s\n", (long long)wmib, s.name,
             t[4], t[0], W / (t[4] * 1e3));
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
