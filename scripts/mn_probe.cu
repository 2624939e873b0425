// Probe: tcgen05.mma kind::tf32 with an MN-major A operand (SWIZZLE_128B or
// no-swizzle canonical layouts), K-major B. D[m][n] = sum_k A[m][k] B[n][k],
// M = 128, N = 64, K = 8, integer data; prints max error per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mn_probe scripts/mn_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_1804_04806_b200/csrc/kernels/sm100.cuh"
using namespace ucudnn::sm100;

constexpr int M = 128, N = 64, K = 8;

__host__ __device__ inline std::uint64_t mkdesc(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo, int layout) {
  std::uint64_t d = 0;
  d |= std::uint64_t((saddr >> 4) & 0x3FFF);
  d |= std::uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= std::uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= std::uint64_t(1) << 46;
  d |= std::uint64_t(layout) << 61;
  return d;
}

// variant: 0 = A MN-major SW128 (LBO = MN-block stride 1024, SBO = 8192)
//          1 = same with LBO/SBO swapped
//          2 = A MN-major no-swizzle (core 8 K-rows x 4 MN, LBO = K-block, SBO = MN-block)
//          3 = same with LBO/SBO swapped
//          4 = A K-major SW128 (control)
__global__ void probe(const float* A, const float* B, float* D, int variant) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  float* sa = reinterpret_cast<float*>(smem);             // 16 KB region
  float* sb = reinterpret_cast<float*>(smem + 16384);     // B: N rows x 32 floats, K-major SW128 (only k < 8 used)
  __shared__ std::uint32_t slot;
  __shared__ __align__(8) std::uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < 4096 + N * 32; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  __syncthreads();
  // A element (m, k) placement
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    std::uint32_t byte;
    if (variant == 0 || variant == 1) {
      // atom: 8 K-rows x 128 B (32 MN elems); MN blocks 1024 B apart; swizzle chunk ^= row
      const int mb = m / 32, mi = m % 32;
      const std::uint32_t row = k, chunk = mi / 4, e = mi % 4;
      byte = mb * 1024 + row * 128 + ((chunk ^ row) * 16) + e * 4;
    } else if (variant == 2 || variant == 3) {
      // core matrix: 8 K-rows x 16 B (4 MN); MN blocks of 4 at 128 B stride
      const int mb = m / 4, e = m % 4;
      byte = mb * 128 + k * 16 + e * 4;
    } else {
      // K-major SW128: row m (128 B, 32 K elems), 8-row groups 1024 B
      const std::uint32_t chunk = k / 4, e = k % 4;
      byte = (m / 8) * 1024 + (m % 8) * 128 + ((chunk ^ (m % 8)) * 16) + e * 4;
    }
    sa[byte / 4] = A[m * K + k];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const std::uint32_t chunk = k / 4, e = k % 4;
    const std::uint32_t byte = (n / 8) * 1024 + (n % 8) * 128 + ((chunk ^ (n % 8)) * 16) + e * 4;
    sb[byte / 4] = B[n * K + k];
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
    std::uint64_t ad;
    std::uint32_t idesc = idesc_tf32(M, N);
    if (variant == 0) ad = mkdesc(a, 1024, 8192, 2), idesc |= 1u << 15;
    else if (variant == 1) ad = mkdesc(a, 8192, 1024, 2), idesc |= 1u << 15;
    else if (variant == 2) ad = mkdesc(a, 4096, 128, 0), idesc |= 1u << 15;
    else if (variant == 3) ad = mkdesc(a, 128, 4096, 0), idesc |= 1u << 15;
    else ad = mkdesc(a, 16, 1024, 2);
    const std::uint64_t bd = mkdesc(b, 16, 1024, 2);
    mma_tf32(tm, ad, bd, idesc, 0);
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  // 4 warps x 32 lanes = 128 rows; columns 0..63
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
  for (int i = 0; i < M * K; ++i) A[i] = float((i * 7) % 7 - 3);
  for (int i = 0; i < N * K; ++i) B[i] = float((i * 5 + 1) % 7 - 3);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int v = 0; v < 5; ++v) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, 48 * 1024>>>(dA, dB, dD, v);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += A[m * K + k] * B[n * K + k];
        maxerr = std::max(maxerr, std::abs(r - D[m * N + n]));
        maxref = std::max(maxref, std::abs(r));
      }
    std::printf("variant %d: max err %.3g (max |ref| %.3g) %s\n", v, maxerr, maxref, cudaGetErrorString(e));
  }
  return 0;
}
