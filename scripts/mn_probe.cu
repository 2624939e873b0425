// Probe: tcgen05.mma kind::tf32 with MN-major operands in the SWIZZLE_128B
// layout a TMA box {32 MN elements (128 B), 32 K rows} produces: per 32-wide
// MN chunk, K row k at k*128 B (chunks 4096 B apart), 16 B granules XORed
// with (k mod 8). D[m][n] = sum_k A[m][k] B[n][k], M = 128, N = 64, K = 32
// (4 MMAs of K = 8), integer data; prints max error per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mn_probe scripts/mn_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>
#include <algorithm>
#include "../paper_1804_04806_b200/csrc/kernels/sm100.cuh"
using namespace ucudnn::sm100;

constexpr int M = 128, N = 64, K = 32;

__host__ __device__ inline std::uint64_t mkdesc(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo, int layout) {
  std::uint64_t d = 0;
  d |= std::uint64_t((saddr >> 4) & 0x3FFF);
  d |= std::uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= std::uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= std::uint64_t(1) << 46;
  d |= std::uint64_t(layout) << 61;
  return d;
}

__device__ inline std::uint32_t kmajor_byte(int mn, int k) {
  return (mn / 8) * 1024 + (mn % 8) * 128 + (((k / 4) ^ (mn % 8)) * 16) + (k % 4) * 4;
}
__device__ inline std::uint32_t mnmajor_byte(int mn, int k) {
  return (mn / 32) * 4096 + k * 128 + ((((mn % 32) / 4) ^ (k % 8)) * 16) + (mn % 4) * 4;
}
// 128B swizzle with 32 B atomicity (CUTLASS Layout_MN_SW128_32B_Atom: Swizzle<2,5,2> on byte
// addresses, 4 K rows of 128 B per atom): 32 B granule index ^= (k mod 4)
__device__ inline std::uint32_t mn32_byte(int mn, int k) {
  return (mn / 32) * 4096 + k * 128 + ((((mn % 32) / 8) ^ (k % 4)) * 32) + (mn % 8) * 4;
}

// variant bits: 1 = A MN-major, 2 = B MN-major, 4 = swap LBO/SBO of MN-major descriptors,
// 8 = MN-major operands in the 128B/32B-atom layout (descriptor layout type 1, SBO = 512)
__global__ void probe(const float* A, const float* B, float* D, int variant) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  float* sa = reinterpret_cast<float*>(smem);          // 16 KB
  float* sb = reinterpret_cast<float*>(smem + 16384);  // 8 KB
  __shared__ std::uint32_t slot;
  __shared__ __align__(8) std::uint64_t bar;
  const int tid = threadIdx.x;
  const bool amn = variant & 1, bmn = variant & 2, swap = variant & 4, b32 = variant & 8;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    sa[(amn ? (b32 ? mn32_byte(m, k) : mnmajor_byte(m, k)) : kmajor_byte(m, k)) / 4] = A[m * K + k];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    sb[(bmn ? (b32 ? mn32_byte(n, k) : mnmajor_byte(n, k)) : kmajor_byte(n, k)) / 4] = B[n * K + k];
  }
  fence_async_smem();
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (tid < 32) tmem_alloc<64>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tm = slot;
  if (tid == 0) {
    const std::uint32_t a = smem_u32(sa), b = smem_u32(sb);
    std::uint32_t idesc = idesc_tf32(M, N);
    if (amn) idesc |= 1u << 15;
    if (bmn) idesc |= 1u << 16;
    for (int j = 0; j < K / 8; ++j) {
      // K-major: advance 32 B within the 128 B row; MN-major: advance one 8-row group (1024 B)
      const std::uint64_t ad = (amn && b32) ? (swap ? mkdesc(a + j * 1024, 512, 4096, 1) : mkdesc(a + j * 1024, 4096, 512, 1))
                             : amn ? (swap ? mkdesc(a + j * 1024, 1024, 4096, 2) : mkdesc(a + j * 1024, 4096, 1024, 2))
                                   : mkdesc(a + j * 32, 16, 1024, 2);
      const std::uint64_t bd = (bmn && b32) ? (swap ? mkdesc(b + j * 1024, 512, 4096, 1) : mkdesc(b + j * 1024, 4096, 512, 1))
                             : bmn ? (swap ? mkdesc(b + j * 1024, 1024, 4096, 2) : mkdesc(b + j * 1024, 4096, 1024, 2))
                                   : mkdesc(b + j * 32, 16, 1024, 2);
      mma_tf32(tm, ad, bd, idesc, j > 0);
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int warp = tid / 32, lane = tid % 32;
  for (int c0 = 0; c0 < N; c0 += 32) {
    float v[32];
    tmem_ld32(tm + (std::uint32_t(warp * 32) << 16) + c0, v);
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * N + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) {
    tc_fence_after();
    tmem_free<64>(tm);
  }
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  for (int i = 0; i < M * K; ++i) A[i] = float((i * 7 + i / 5) % 7 - 3);
  for (int i = 0; i < N * K; ++i) B[i] = float((i * 5 + 1 + i / 3) % 7 - 3);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int variants[] = {0, 1, 2, 3, 9, 10, 11, 13, 14, 15};
  for (int v : variants) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, 40 * 1024>>>(dA, dB, dD, v);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0, maxgot = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += A[m * K + k] * B[n * K + k];
        maxerr = std::max(maxerr, std::abs(r - D[m * N + n]));
        maxref = std::max(maxref, std::abs(r));
        maxgot = std::max(maxgot, (double)std::abs(D[m * N + n]));
      }
    std::printf("variant %d (A %s, B %s%s): max err %.3g (max |ref| %.3g, max |got| %.3g) %s\n", v,
                (v & 1) ? "MN" : "K", (v & 2) ? "MN" : "K", (v & 4) ? ", lbo/sbo swapped" : (v & 8) ? ", 128B/32B atoms" : "", maxerr, maxref,
                maxgot, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
