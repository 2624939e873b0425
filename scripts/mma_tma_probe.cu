// Probe: does concurrent TMA traffic into shared memory slow tcgen05.mma?
// Warp 1 issues `per` MMAs (128 x N x 8, tf32) per commit; warp 0 optionally
// streams 16 KB TMA boxes into a separate smem ring (3 producer warps).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma_tma_probe scripts/mma_tma_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "../paper_1804_04806_b200/csrc/kernels/sm100.cuh"
using namespace ucudnn::sm100;

__global__ void __launch_bounds__(256, 1) probe(const __grid_constant__ CUtensorMap map, int N, int iters, int per,
                                                int tma_on, long long* out, int ntiles, int nbuf) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  unsigned char* ops = smem;                  // MMA operands: nbuf x (A 16 KB + B N*128)
  const std::uint32_t bufb = 16384 + N * 128;
  unsigned char* ring = smem + (tma_on ? 0 : 0) + nbuf * bufb;  // TMA ring: 6 x 16 KB (when on)
  __shared__ __align__(8) std::uint64_t bar, full[6], empty[6];
  __shared__ std::uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < int(nbuf * bufb / 4); i += blockDim.x)
    reinterpret_cast<float*>(ops)[i] = float((i * 2654435761u) % 1000) * 1e-3f - 0.5f;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int s = 0; s < 6; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_fence_init();
    done = 0;
  }
  fence_async_smem();
  if (warp == 1) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tm = slot;
  if (warp == 1) {
    const std::uint32_t a0 = smem_u32(ops), idesc = idesc_tf32(128, N);
    const std::uint64_t da0 = umma_desc_sw128(a0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (lane == 0) {
        // buffer = (it % nbuf): descriptors are precomputed base + (byte offset >> 4)
        const std::uint64_t da = da0 + (((it % nbuf) * bufb) >> 4), db = da + (16384 >> 4);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q >= per) break;
          mma_tf32(tm, da + 2 * (q & 3), db + 2 * (q & 3), idesc, 1);
        }
        mma_commit(&bar);
      }
      __syncwarp();
    }
    mbar_wait(&bar, (iters - 1) & 1);
    long long t1 = clock64();
    if (lane == 0) {
      out[blockIdx.x] = (t1 - t0) / ((long long)iters * per);
      done = 1;
    }
  } else if (tma_on && (warp == 0 || warp == 2 || warp == 3) && lane == 0) {
    const int pq = warp == 0 ? 0 : warp - 1;
    for (int it = pq; !done; it += 3) {
      const int s = it % 6;
      mbar_wait(&empty[s], ((it / 6) & 1) ^ 1);
      mbar_expect_tx(&full[s], 16384);
      tma_2d(ring + s * 16384, &map, &full[s], 0, ((blockIdx.x * 977 + it * 13) % ntiles) * 128);
      mbar_wait(&full[s], (it / 6) & 1);  // consume immediately
      mbar_arrive(&empty[s]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<256>(tm);
  }
}

int main() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  const std::size_t bytes = std::size_t(64) << 20;
  float* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  CUtensorMap map;
  cuuint64_t dims[2] = {32, bytes / 128};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int N : {64, 192, 256})
    for (int nbuf : {2, 4})
      for (int per : {8}) {
        const int tma = nbuf == 4 ? 1 : 0;  // nbuf 4: with 3 producers streaming TMA into a ring
        const int smem = nbuf * (16384 + N * 128) + 1024 + 6 * 16384;
        if (smem > 200 * 1024) continue;
        probe<<<148, 256, smem>>>(map, N, 200, per, tma, d, int(bytes / 128 / 128), nbuf);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        std::printf("N=%3d nbuf=%d per=%d: %.0f cyc/MMA (%.0f MAC/cyc/SM) %s\n", N, nbuf, per, avg, 128.0 * N * 8 / avg,
                    cudaGetErrorString(e));
      }
  return 0;
}
