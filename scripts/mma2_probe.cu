// Probe: 2-SM UMMA (tcgen05.mma.cta_group::2, kind::tf32) on a CTA pair.
// Each CTA holds 128 rows of A and N/2 rows of B (K = 8, SW128 K-major);
// CTA 0 issues D[256 x N] = A B^T, the commit multicasts to both CTAs, and
// each checks its 128 x N slice against the host. Then times `iters`
// commit groups of `per` MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma2_probe scripts/mma2_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_1804_04806_b200/csrc/kernels/sm100.cuh"
using namespace ucudnn::sm100;

constexpr int K = 8;

__device__ __forceinline__ std::uint32_t cta_rank() {
  std::uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(const float* A, const float* B, float* D, int N, int iters, int per, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  float* sa = reinterpret_cast<float*>(smem);
  float* sb = reinterpret_cast<float*>(smem + 128 * 128);
  __shared__ std::uint32_t slot;
  __shared__ __align__(8) std::uint64_t bar;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const std::uint32_t rank = cta_rank();
  const int nh = N / 2;
  for (int i = tid; i < (128 + nh) * 32; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  __syncthreads();
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const std::uint32_t byte = (m / 8) * 1024 + (m % 8) * 128 + (((k / 4) ^ (m % 8)) * 16) + (k % 4) * 4;
    sa[byte / 4] = A[(rank * 128 + m) * K + k];
  }
  for (int i = tid; i < nh * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const std::uint32_t byte = (n / 8) * 1024 + (n % 8) * 128 + (((k / 4) ^ (n % 8)) * 16) + (k % 4) * 4;
    sb[byte / 4] = B[(rank * nh + n) * K + k];
  }
  fence_async_smem();
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  csync();
  tc_fence_after();
  const std::uint32_t tm = slot;
  const std::uint32_t idesc = idesc_tf32(256, N);
  long long t0 = clock64();
  int ph = 0;
  for (int it = 0; it < iters; ++it) {
    if (rank == 0 && warp == 0) {
      if (lane == 0) {
        for (int q = 0; q < per; ++q) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
              "l"(umma_desc_sw128(smem_u32(sa))), "l"(umma_desc_sw128(smem_u32(sb))), "r"(idesc),
              "r"((it | q) != 0 ? 1 : 0)
              : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((unsigned short)3)
            : "memory");
      }
      __syncwarp();
    }
    mbar_wait(&bar, ph);
    ph ^= 1;
  }
  long long t1 = clock64();
  tc_fence_after();
  if (rank == 0 && tid == 0) cyc[0] = (t1 - t0) / ((long long)iters * per);
  // accumulated iters*per times the same product: divide on the host
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tmem_ld32(tm + (std::uint32_t(warp * 32) << 16) + c0, v);
    for (int j = 0; j < 32; ++j) D[(rank * 128 + warp * 32 + lane) * N + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  csync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256) : "memory");
  }
}

int main() {
  for (int N : {64, 128, 256}) {
    std::vector<float> A(256 * K), B(N * K), D(256 * N);
    for (int i = 0; i < 256 * K; ++i) A[i] = float((i * 7 + i / 13) % 7 - 3);
    for (int i = 0; i < N * K; ++i) B[i] = float((i * 5 + 1) % 7 - 3);
    float *dA, *dB, *dD;
    long long* dc;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int per : {1, 4, 8, 16}) {
      const int iters = 64;
      cudaMemset(dD, 0, D.size() * 4);
      probe<<<2, 128, 64 * 1024>>>(dA, dB, dD, N, iters, per, dc);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      long long cyc = 0;
      cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 256; ++m)
        for (int n = 0; n < N; ++n) {
          double r = 0;
          for (int k = 0; k < K; ++k) r += A[m * K + k] * B[n * K + k];
          maxerr = std::max(maxerr, std::abs(r * iters * per - D[m * N + n]));
        }
      const double macs = 256.0 * N * 8;
      std::printf("N=%3d per=%2d: max err %g, %lld cyc/MMA -> %.0f MAC/cyc per SM pair (%s)\n", N, per, maxerr, cyc,
                  macs / cyc, cudaGetErrorString(e));
    }
  }
  return 0;
}
