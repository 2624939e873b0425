// Probe: can a K-major SWIZZLE_128B UMMA operand start at an arbitrary ROW
// (multiple of 128 B, not of the 1024 B swizzle atom) by setting the
// descriptor's base-offset field? A strip of 256 rows x 8 tf32 is written in
// the SW128 pattern; D = A[off : off+128] * B^T for off in {0, 1, 3, 8, 13}.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/offset_probe scripts/offset_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../paper_1804_04806_b200/csrc/kernels/sm100.cuh"
using namespace ucudnn::sm100;

constexpr int ROWS = 256, N = 64, K = 8;

__global__ void probe(const float* A, const float* B, float* D, int off, int mode) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  float* sa = reinterpret_cast<float*>(smem);
  float* sb = reinterpret_cast<float*>(smem + ROWS * 128);
  __shared__ std::uint32_t slot;
  __shared__ __align__(8) std::uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < (ROWS + N) * 32; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  __syncthreads();
  for (int i = tid; i < ROWS * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const std::uint32_t byte = m * 128 + (((k / 4) ^ (m % 8)) * 16) + (k % 4) * 4;
    sa[byte / 4] = A[m * K + k];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const std::uint32_t byte = n * 128 + (((k / 4) ^ (n % 8)) * 16) + (k % 4) * 4;
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
    const std::uint32_t a = smem_u32(sa) + off * 128, b = smem_u32(sb);
    std::uint64_t ad = umma_desc_sw128(a);
    if (mode == 1) ad |= std::uint64_t((off & 7)) << 49;           // base offset = row phase
    if (mode == 2) ad |= std::uint64_t(((a >> 7) & 7)) << 49;      // same, from the address
    mma_tf32(tm, ad, umma_desc_sw128(b), idesc_tf32(128, N), 0);
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
  std::vector<float> A(ROWS * K), B(N * K), D(128 * N);
  for (int i = 0; i < ROWS * K; ++i) A[i] = float((i * 7 + i / 11) % 7 - 3);
  for (int i = 0; i < N * K; ++i) B[i] = float((i * 5 + 1) % 7 - 3);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode = 0; mode < 3; ++mode)
    for (int off : {0, 1, 3, 8, 13}) {
      cudaMemset(dD, 0, D.size() * 4);
      probe<<<1, 128, 60 * 1024>>>(dA, dB, dD, off, mode);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          double r = 0;
          for (int k = 0; k < K; ++k) r += A[(m + off) * K + k] * B[n * K + k];
          maxerr = std::max(maxerr, std::abs(r - D[m * N + n]));
        }
      std::printf("mode %d off %2d: max err %g %s\n", mode, off, maxerr, cudaGetErrorString(e));
    }
  return 0;
}
