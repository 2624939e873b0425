// Microbenchmark: TMA tiled-load throughput per SM on this part, as a
// function of box rows (x 128 B), pipeline depth and working-set size.
// One persistent CTA per SM; lane 0 of warp 0 streams boxes through an
// S-stage mbarrier ring; warp 1 lane 0 consumes (wait full -> arrive empty).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe scripts/tma_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#include "../paper_1804_04806_b200/csrc/kernels/sm100.cuh"
using namespace ucudnn::sm100;

__device__ __forceinline__ void expect_tx_relaxed(std::uint64_t* bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void wait_relaxed(std::uint64_t* bar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void wait_poll(std::uint64_t* bar, std::uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap map, int rows, int stages,
                                                int iters, int ntiles, int mc, int variant) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const std::uint32_t box_bytes = rows * 128;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + stages * box_bytes * mc);
  std::uint64_t* empty = full + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int nprod = variant == 5 ? 2 : variant == 6 ? 3 : 1;
  const int pq = warp == 0 ? 0 : warp - 1;
  if ((warp == 0 || (variant >= 5 && warp == 2) || (variant == 6 && warp == 3)) && lane == 0) {
    for (int it = pq; it < iters; it += nprod) {
      const int s = it % stages;
      if (variant == 2) wait_relaxed(&empty[s], ((it / stages) & 1) ^ 1);
      else if (variant == 4) wait_poll(&empty[s], ((it / stages) & 1) ^ 1);
      else mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      const int t = (blockIdx.x * 7919 + it * 13) % ntiles;
      if (variant == 0 || variant >= 4) mbar_expect_tx(&full[s], box_bytes * mc);
      if (variant == 1 || variant == 2) expect_tx_relaxed(&full[s], box_bytes * mc);
      for (int m = 0; m < mc; ++m)
        tma_2d(smem + (s * mc + m) * box_bytes, &map, &full[s], 0, ((t + m * 17) % ntiles) * rows);
      if (variant == 3) mbar_expect_tx(&full[s], box_bytes * mc);
    }
  } else if (warp == 1 && lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      if (variant == 2) wait_relaxed(&full[s], (it / stages) & 1);
      else if (variant == 4) wait_poll(&full[s], (it / stages) & 1);
      else mbar_wait(&full[s], (it / stages) & 1);
      mbar_arrive(&empty[s]);
    }
  }
}

int main() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const std::size_t big = std::size_t(1) << 30;  // 1 GiB
  float* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 0, big);
  const int sms = 148;
  for (std::size_t ws : {std::size_t(16) << 20}) {
    const std::size_t rows_total = ws / 128;
    for (int rows : {64, 128}) {
      CUtensorMap map;
      cuuint64_t dims[2] = {32, rows_total};
      cuuint64_t strides[1] = {128};
      cuuint32_t box[2] = {32, cuuint32_t(rows)};
      cuuint32_t es[2] = {1, 1};
      enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int ntiles = int(rows_total / rows);
      for (int mc : {1, 2}) {
       for (int variant : {0, 5, 6}) {
        for (int stages : {3, 6}) {
        for (int cps : {1}) {
          const int smem = stages * rows * 128 * mc + 2048;
          if (smem * cps > 220 * 1024) continue;
          const int iters = int((std::size_t(512) << 20) / (std::size_t(sms) * rows * 128 * mc)) + 8;
          probe<<<sms * cps, 128, smem>>>(map, rows, stages, 8, ntiles, mc, variant);
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          cudaEventRecord(e0);
          probe<<<sms * cps, 128, smem>>>(map, rows, stages, iters, ntiles, mc, variant);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          const double bytes = double(sms) * cps * iters * rows * 128 * mc;
          std::printf("v%d cps=%d ws=%5zu MiB box=%3d rows x%d stages=%d: %7.1f GB/s  %5.1f B/clk/SM @1.9GHz  err=%s\n",
                      variant, cps, ws >> 20, rows, mc, stages, bytes / ms / 1e6, bytes / (ms * 1e-3) / 1.9e9 / sms,
                      cudaGetErrorString(cudaGetLastError()));
        }
        }
       }
      }
    }
  }
  return 0;
}
