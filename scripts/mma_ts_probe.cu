// Probe: issue rate of tcgen05.mma kind::tf32 (M = 128, N, K = 8) with A from
// shared memory (SS) vs A from tensor memory (TS), `per` MMAs per commit,
// with or without waiting for each commit (a ring's round trip).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma_ts_probe scripts/mma_ts_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_1804_04806_b200/csrc/kernels/sm100.cuh"
using namespace ucudnn::sm100;

__device__ __forceinline__ void mma_ts(std::uint32_t d, std::uint32_t a, std::uint64_t b, std::uint32_t idesc,
                                       std::uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) probe(int N, int iters, int per, int ts, int nacc, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  __shared__ __align__(8) std::uint64_t bar;
  __shared__ std::uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < (16384 + 256 * 128) / 4; i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = float((i * 2654435761u) % 1000) * 1e-3f - 0.5f;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  fence_async_smem();
  if (warp == 1) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = slot;
  if (warp == 1) {
    const std::uint32_t idesc = idesc_tf32(128, N);
    const std::uint32_t sa = smem_u32(smem), sb = sa + 16384;
    std::uint32_t ph = 0;
    long long t0 = 0;
    for (int it = -2; it < iters; ++it) {
      if (it == 0) t0 = clock64();
      if (lane == 0) {
        for (int j = 0; j < per; ++j) {
          const int k = j & 3;
          const std::uint32_t dcol = std::uint32_t((j % nacc) * N);
          if (ts)
            mma_ts(tmem + dcol, tmem + 384 + 8 * k, umma_desc_sw128(sb + 32 * k), idesc, 1u);
          else
            mma_tf32(tmem + dcol, umma_desc_sw128(sa + 32 * k), umma_desc_sw128(sb + 32 * k), idesc, 1u);
        }
        mma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    const long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

template <int PER, int NACC, int TS>
__global__ void __launch_bounds__(128, 1) probe_u(int N, int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  __shared__ __align__(8) std::uint64_t bar;
  __shared__ std::uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < (16384 + 256 * 128) / 4; i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = float((i * 2654435761u) % 1000) * 1e-3f - 0.5f;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  fence_async_smem();
  if (warp == 1) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = slot;
  if (warp == 1) {
    const std::uint32_t idesc = idesc_tf32(128, N);
    const std::uint32_t sa = smem_u32(smem), sb = sa + 16384;
    const std::uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sb);
    std::uint32_t ph = 0;
    long long t0 = 0;
    for (int it = -2; it < iters; ++it) {
      if (it == 0) t0 = clock64();
      if (lane == 0) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int k = j & 3;
          const std::uint32_t dcol = std::uint32_t((j % NACC) * 128);
          if (TS)
            mma_ts(tmem + dcol, tmem + 384 + 8 * k, db + 2 * k, idesc, 1u);
          else
            mma_tf32(tmem + dcol, da + 2 * k, db + 2 * k, idesc, 1u);
        }
        mma_commit(&bar);
      }
      __syncwarp();
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    const long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

template <int PER, int NACC, int TS>
void run_u(long long* d, int N) {
  cudaFuncSetAttribute(probe_u<PER, NACC, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  const int iters = 2000;
  probe_u<PER, NACC, TS><<<148, 128, 60 * 1024>>>(N, iters, d);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("unrolled N=%3d %s nacc=%d per=%2d: %7.1f cyc/MMA (floor %d)  err=%s\n", N, TS ? "TS" : "SS", NACC, PER,
         double(h) / iters / PER, 128 * N / 256, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  for (int N : {64, 128}) {
    run_u<8, 1, 0>(d, N); run_u<32, 1, 0>(d, N); run_u<32, 2, 0>(d, N); run_u<32, 3, 0>(d, N);
    run_u<8, 1, 1>(d, N); run_u<32, 1, 1>(d, N); run_u<32, 2, 1>(d, N); run_u<32, 3, 1>(d, N);
  }
  run_u<32, 1, 0>(d, 256); run_u<32, 1, 1>(d, 256); run_u<32, 1, 0>(d, 32); run_u<32, 4, 0>(d, 32);
  for (int N : {64})
    for (int ts : {0, 1})
      for (int nacc : {1, 2})
        for (int per : {8, 32}) {
          if (nacc * N > 384) continue;
          const int iters = 2000;
          probe<<<148, 128, 60 * 1024>>>(N, iters, per, ts, nacc, d);
          long long h = 0;
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
          printf("N=%3d %s nacc=%d per=%2d: %7.1f cyc/MMA (floor %d)  err=%s\n", N, ts ? "TS" : "SS", nacc, per,
                 double(h) / iters / per, 128 * N / 256, cudaGetErrorString(cudaGetLastError()));
        }
  return 0;
}
