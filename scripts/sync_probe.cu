// Microbenchmark: cost of mbarrier try_wait / test_wait / arrive on this part.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/sync_probe scripts/sync_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_1804_04806_b200/csrc/kernels/sm100.cuh"
using namespace ucudnn::sm100;

__global__ void probe(long long* out, int iters) {
  __shared__ __align__(8) std::uint64_t bar[4];
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // complete phase 0 of bar[0]
    mbar_arrive(&bar[0]);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) mbar_wait(&bar[0], 0);  // already complete
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) {  // arrive + wait ping (own barrier, 1 thread)
      mbar_arrive(&bar[1]);
      mbar_wait(&bar[1], i & 1);
    }
    long long t2 = clock64();
    out[0] = (t1 - t0) / iters;
    out[1] = (t2 - t1) / iters;
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  probe<<<1, 32>>>(d, 1000);
  probe<<<1, 32>>>(d, 1000);
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  std::printf("try_wait on completed phase: %lld cyc/iter; arrive+wait round trip: %lld cyc/iter (%s)\n", h[0], h[1],
              cudaGetErrorString(cudaGetLastError()));
  return 0;
}
