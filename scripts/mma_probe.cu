// Microbenchmark: tcgen05.mma kind::tf32 throughput for M=128, N in {64,128,256},
// SWIZZLE_128B K-major smem operands, one accumulator, `per_commit` MMAs per
// tcgen05.commit (+ wait on it when `wait` is set).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma_probe scripts/mma_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_1804_04806_b200/csrc/kernels/sm100.cuh"
using namespace ucudnn::sm100;

__global__ void __launch_bounds__(128, 1) probe(long long* out, int iters, int N, int per_commit, int wait) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  __shared__ __align__(8) std::uint64_t bar;
  __shared__ std::uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (128 + 256) * 32; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = slot;
  if (warp == 0) {
    const std::uint32_t sa = smem_u32(smem), sb = sa + 128 * 128;
    const std::uint32_t idesc = idesc_tf32(128, N);
    long long t0 = clock64();
    int ph = 0;
    for (int i = 0; i < iters; ++i) {
      if (wait == 2) {  // 4 MMAs per lane-0 block, one commit per per_commit MMAs
        for (int q0 = 0; q0 < per_commit; q0 += 4) {
          if (lane == 0) {
            for (int q = 0; q < 4; ++q)
              mma_tf32(tmem, umma_desc_sw128(sa + (q & 3) * 32), umma_desc_sw128(sb + (q & 3) * 32), idesc, 1);
            if (q0 + 4 >= per_commit) mma_commit(&bar);
          }
          __syncwarp();
        }
      } else {
      if (lane == 0) {
        for (int q = 0; q < per_commit; ++q)
          mma_tf32(tmem, umma_desc_sw128(sa + (q & 3) * 32), umma_desc_sw128(sb + (q & 3) * 32), idesc, 1);
        mma_commit(&bar);
      }
      __syncwarp();
      }
      if (wait == 1) {
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    if (wait != 1) {
      // drain: the last commit's phase
      mbar_wait(&bar, (iters - 1) & 1);
    }
    long long t1 = clock64();
    if (lane == 0) out[0] = (t1 - t0) / ((long long)iters * per_commit);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int N : {64, 192})
    for (int pc : {4, 8, 16})
      for (int w : {0, 2}) {
        probe<<<148, 128, 64 * 1024>>>(d, 64, N, pc, w);
        probe<<<148, 128, 64 * 1024>>>(d, 512, N, pc, w);
        long long h;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        const double macs = 128.0 * N * 8;
        std::printf("N=%3d mma/commit=%2d wait=%d: %lld cyc/MMA  (%.0f MAC/cyc/SM, %.0f TFLOP/s @1.9GHz x148) %s\n", N,
                    pc, w, h, macs / h, 2 * macs / h * 1.9e9 * 148 / 1e12, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
