// Microbenchmark: rate at which warps can gather 128-byte rows (32
// consecutive floats at an arbitrary 4-byte offset) from an L2-resident
// buffer into shared memory, by mechanism:
//   0: cp.async 4 B per lane (LDGSTS), one wait per batch of rows
//   1: LDG.32 into registers (batch of 8 rows), then STS.32
//   2: cp.async 4 B with .cg-style bypass impossible -> same as 0 but rows
//      spread over 4 MiB (L1 miss heavy) -- compares L1 reuse
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/gather_probe scripts/gather_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void probe(const float* __restrict__ buf, int n_floats, int rows_per_warp, int mode, int span) {
  extern __shared__ float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* wsm = sm + warp * 32 * 8;
  std::uint32_t seed = blockIdx.x * 7919u + warp * 104729u;
  float acc = 0.f;
  for (int r = 0; r < rows_per_warp; r += 8) {
    std::uint32_t off[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      seed = seed * 1664525u + 1013904223u;
      off[j] = (seed >> 8) % std::uint32_t(span);
    }
    if (mode == 0 || mode == 2) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float* src = buf + off[j] + lane;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(wsm + j * 32 + lane)), "l"(src)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 3;" ::: "memory");
    } else {
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldg(buf + off[j] + lane);
#pragma unroll
      for (int j = 0; j < 8; ++j) wsm[j * 32 + lane] = v[j];
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
  acc += wsm[lane];
  if (acc == 12345.f) printf("x");
}

int main() {
  const int n = 64 << 20;  // 256 MiB buffer
  float* buf;
  cudaMalloc(&buf, std::size_t(n) * 4 + 4096);
  cudaMemset(buf, 0, std::size_t(n) * 4 + 4096);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode : {0, 1}) {
    for (int span_mb : {1, 16, 64}) {
      for (int warps : {8, 16, 32}) {
        const int span = span_mb << 18;  // floats
        const int rows = 4096;
        const int smem = warps * 32 * 8 * 4;
        probe<<<148, warps * 32, smem>>>(buf, n, 64, mode, span);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<<<148, warps * 32, smem>>>(buf, n, rows, mode, span);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = 148.0 * warps * rows * 128;
        std::printf("mode %d span %3d MiB warps %2d: %8.1f GB/s  %6.1f B/clk/SM @1.9GHz  %s\n", mode, span_mb, warps,
                    bytes / ms / 1e6, bytes / (ms * 1e-3) / 1.9e9 / 148, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
