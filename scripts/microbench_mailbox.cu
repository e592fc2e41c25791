// scripts/microbench_mailbox.cu — design probe (not product code): cost of the
// mailbox exchange's publish + combine for W ranks, serial (one thread, as in
// round 1) vs warp-cooperative (publish_partial_warp / combine_parts_warp from
// stream_common.cuh, one lane per rank).  W CTAs in one launch stand in for the
// W ranks: CTA k publishes its partial into all W mailboxes and then waits for /
// combines its own mailbox.  All mailboxes live on this GPU, so the remote
// stores are local here (an NVLink store costs more, which makes the serial
// chain worse, not better).  Prints µs per launch (CUDA events over back-to-back
// launches; launch overhead is the same for both forms) and checks both forms
// give the same combined sum.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -Ipaper_2207_00257_b200/csrc -o /tmp/mb_mailbox scripts/microbench_mailbox.cu && /tmp/mb_mailbox
#include <cstdio>
#include <vector>

#include "stream_common.cuh"

using namespace lnorm;

__device__ void publish_serial(const PeerPost& post, double S) {
  const size_t slot = ((size_t)(post.epoch & 1) * post.world + post.rank) * 2;
  for (int r = 0; r < post.world; ++r) st_relaxed_sys_f64(post.mail[r] + slot, S);
  __threadfence_system();
  for (int r = 0; r < post.world; ++r)
    st_release_sys_u64(reinterpret_cast<unsigned long long*>(post.mail[r] + slot + 1), post.epoch);
}

__device__ double combine_serial(const double* mail, int world, unsigned long long epoch) {
  const double* box = mail + (size_t)(epoch & 1) * world * 2;
  for (int r = 0; r < world; ++r) {
    const unsigned long long* flag = reinterpret_cast<const unsigned long long*>(box + 2 * r + 1);
    while (ld_acquire_sys_u64(flag) != epoch) __nanosleep(64);
  }
  double S = ld_relaxed_sys_f64(box);
  for (int r = 1; r < world; ++r) S += ld_relaxed_sys_f64(box + 2 * r);
  return S;
}

template <bool WARP>
__global__ void exchange(double* const* mails, int world, unsigned long long epoch, double* out) {
  const int rank = blockIdx.x;
  const PeerPost post{mails, rank, world, epoch};
  const double part = 1.0 / 3.0 + rank * 0.1;  // non-trivial roundings in the sum
  double S;
  if (WARP) {
    publish_partial_warp(post, part);
    combine_parts_warp(mails[rank], world, &S, epoch);
  } else if (threadIdx.x == 0) {
    publish_serial(post, part);
    S = combine_serial(mails[rank], world, epoch);
  }
  if (threadIdx.x == 0) out[rank] = S;
}

int main() {
  const int reps = 2000;
  for (int world : {2, 4, 8}) {
    std::vector<double*> h(world);
    for (int r = 0; r < world; ++r) {
      cudaMalloc(&h[r], 2 * world * 2 * sizeof(double));
      cudaMemset(h[r], 0, 2 * world * 2 * sizeof(double));
    }
    double** d;
    cudaMalloc(&d, world * sizeof(double*));
    cudaMemcpy(d, h.data(), world * sizeof(double*), cudaMemcpyHostToDevice);
    double* out;
    cudaMalloc(&out, world * sizeof(double));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    unsigned long long epoch = 1;
    double res[2][8];
    float us[2];
    for (int form = 0; form < 2; ++form) {
      for (int i = 0; i < 50; ++i, ++epoch)
        form ? exchange<true><<<world, 32>>>(d, world, epoch, out) : exchange<false><<<world, 32>>>(d, world, epoch, out);
      cudaEventRecord(a);
      for (int i = 0; i < reps; ++i, ++epoch)
        form ? exchange<true><<<world, 32>>>(d, world, epoch, out) : exchange<false><<<world, 32>>>(d, world, epoch, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      us[form] = ms * 1e3f / reps;
      // one more launch at a fixed epoch parity to compare the sums
      const unsigned long long e = epoch + (epoch & 1);  // even epoch
      form ? exchange<true><<<world, 32>>>(d, world, e, out) : exchange<false><<<world, 32>>>(d, world, e, out);
      epoch = e + 1;
      cudaMemcpy(res[form], out, world * sizeof(double), cudaMemcpyDeviceToHost);
    }
    cudaError_t err = cudaGetLastError();
    bool same = true;
    for (int r = 0; r < world; ++r) same &= res[0][r] == res[1][r] && res[0][r] == res[0][0];
    printf("W=%d: serial %.2f us per launch, warp-cooperative %.2f us per launch; sums %s (%s)\n", world, us[0],
           us[1], same ? "bit-identical" : "DIFFER", err == cudaSuccess ? "ok" : cudaGetErrorString(err));
    for (auto p : h) cudaFree(p);
    cudaFree(d);
    cudaFree(out);
  }
  return 0;
}
