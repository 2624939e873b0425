// UCUDNN_ALGO_IMPLICIT_GEMM (0 workspace) for 1x1 stride-1 unpadded layers
// (ResNet bottleneck and projection convolutions): the convolution is a
// batched GEMM over each image's H*W plane, and both operands can be read by
// TMA straight from the caller's NCHW / KC tensors -- no gather, no copy.
//
//   Forward        y[n][k][p]  = alpha * sum_c  x[n][c][p]  * w[k][c] + beta * y   (reference_conv.hpp:70-100)
//   BackwardData   dx[n][c][p] = alpha * sum_k dy[n][k][p]  * w[k][c] + beta * dx  (reference_conv.hpp:105-135)
//
// GEMM: M = positions p of one image (128 per tile; the last tile of a plane
// is cut by TMA out-of-bounds zero fill and the epilogue's bounds), N =
// output channels, reduction = input channels. A = a {32 positions, 32
// channels} box per 32-position block of the (p, c, n) view of x / dy, which
// lands as 32 K-rows of 128 B: the *MN-major* operand in the 128B/32B-atom
// swizzle (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, DESIGN finding 5). B: Forward
// reads w as (c, k): a {32 c, BN k} box is the K-major SW128 operand;
// BackwardData needs B[c][k] = w[k][c], whose rows (c) are contiguous along
// N: {32 c, 32 k} boxes are MN-major blocks (instruction-descriptor bit 16).
// Needs H*W % 4 == 0 (16 B plane stride) and C % 4 == 0 / K % 4 == 0.
// Stride-2 BackwardData (ResNet projection shortcuts) is the stride-1 GEMM
// on dy's plane with each result written to the top-left of its 2x2 dx block
// and beta * dx (or 0) to the three tapless phases. (A stride-2 Forward would
// need a traversal stride along w, which TMA does not offer for the
// innermost dimension.)
//
// Persistent, one CTA per SM: three producer threads (warps 0, 2, 3) owning
// ring stages s % 3 (one thread's TMA stream keeps about one stage in flight,
// finding 2), warp 1 TMEM owner + MMA issuer with two accumulator sets,
// warps 4-11 the NCHW epilogue (32 lanes = 32 consecutive positions: coalesced).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "conv_common.h"
#include "launch.h"
#include "sm100.cuh"
#include "z1x1.h"

namespace ucudnn {
using namespace sm100;

namespace {

constexpr int kBM = 128;
constexpr int kMaxBN = 256;
constexpr int kMaxStages = 8;
constexpr int kThreads = 384;  // 3 producer warps (+1 idle), MMA warp, 8 epilogue warps
constexpr std::uint32_t kABytes = kBM * 128;

struct OParams {
  float* out;
  float alpha, beta;
  int HW, Cs, Co;       // source plane size, reduction channels, output channels
  // stride 2 (BackwardData only): 2 = dy plane -> 2x2 dx blocks
  int s2, OW, H, W;
  int BN, n_tiles, tpi;  // column tile, column tiles, position tiles per image
  int units, chunks, stages, bd;
  long long oimg;        // Co * HW
};

__device__ __forceinline__ void tma_3d(void* dst, const void* tmap, std::uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ std::uint64_t desc_mn32(std::uint32_t saddr) {
  std::uint64_t d = 0;
  d |= std::uint64_t((saddr >> 4) & 0x3FFF);
  d |= std::uint64_t(4096 >> 4) << 16;
  d |= std::uint64_t(512 >> 4) << 32;
  d |= std::uint64_t(1) << 46;
  d |= std::uint64_t(1) << 61;
  return d;
}
__device__ __forceinline__ void mbar_wait_sleep(std::uint64_t* bar, std::uint32_t parity) {
  std::uint32_t ok = 0, ns = 64;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(ns);
    if (ns < 2048) ns <<= 1;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    z1x1_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, const OParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t b_bytes = (std::uint32_t(p.BN) * 128 + 1023) & ~1023u;
  const std::uint32_t stage_bytes = kABytes + b_bytes;
  const int kStages = p.stages;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kStages * stage_bytes);
  std::uint64_t* empty = full + kMaxStages;
  std::uint64_t* tfull = empty + kMaxStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);

  if (threadIdx.x == 0) {
    prefetch_tmap(&amap);
    prefetch_tmap(&bmap);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 256);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = tmem_base_uniform(tmem_slot);

  if (warp == 0 || warp == 2 || warp == 3) {
    // ------------------------------------------------ TMA producers (stage s owned by thread s % 3)
    const int pq = warp == 0 ? 0 : warp - 1;
    const int nprod = kStages < 3 ? kStages : 3;
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const int mt = u % (p.units / p.n_tiles), nt = u / (p.units / p.n_tiles);
        const int n = mt / p.tpi, t = mt - n * p.tpi, p0 = t * kBM;
        for (int ch = 0; ch < p.chunks; ++ch, ++it) {
          if ((it % kStages) % nprod != pq) continue;
          const int s = it % kStages;
          mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          unsigned char* sa = smem + s * stage_bytes;
          mbar_expect_tx(&full[s], kABytes + std::uint32_t(p.BN) * 128);
#pragma unroll
          for (int b = 0; b < 4; ++b) tma_3d(sa + b * 4096, &amap, &full[s], p0 + b * 32, ch * 32, n);
          if (p.bd) {
            for (int b = 0; b < p.BN / 32; ++b)
              tma_2d(sa + kABytes + b * 4096, &bmap, &full[s], nt * p.BN + b * 32, ch * 32);
          } else {
            tma_2d(sa + kABytes, &bmap, &full[s], ch * 32, nt * p.BN);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN) | (1u << 15) | (p.bd ? (1u << 16) : 0u);
    const std::uint32_t sbase = smem_u32(smem);
    int it = 0, tl = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++tl) {
      const int acc = tl & 1;
      mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
      tc_fence_after();
      const std::uint32_t dtm = tmem + std::uint32_t(acc * kMaxBN);
      for (int ch = 0; ch < p.chunks; ++ch, ++it) {
        const int s = it % kStages;
        mbar_wait(&full[s], (it / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          const std::uint32_t sa = sbase + s * stage_bytes, sb = sa + kABytes;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            mma_tf32(dtm, desc_mn32(sa + j * 1024), p.bd ? desc_mn32(sb + j * 1024) : umma_desc_sw128(sb + j * 32),
                     idesc, (ch | j) ? 1u : 0u);
          mma_commit(&empty[s]);
          if (ch + 1 == p.chunks) mma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 4-11)
    // two warp groups share every tile: warp w reads TMEM lanes 32 (w % 4)
    // (its 32 positions) and group (w - 4) / 4 takes alternate 32-column
    // chunks -- at 256 output channels one group's stores could not keep up
    // with the MMAs (ncu: 64 -> 256 Forward at 0.41 of HBM, 4 warps)
    const int ew = warp & 3, eg = (warp - 4) >> 2;
    int tl = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++tl) {
      const int mt = u % (p.units / p.n_tiles), nt = u / (p.units / p.n_tiles);
      const int n = mt / p.tpi, t = mt - n * p.tpi;
      int pos = t * kBM + ew * 32 + lane;  // source-plane position (s1, BD s2)
      bool live = pos < p.HW;
      long long ostride = p.HW;            // output plane size
      if (p.s2 == 2) {
        const int i = pos / p.OW, j = pos - i * p.OW;
        pos = 2 * i * p.W + 2 * j;  // top-left of the 2x2 dx block
        ostride = (long long)p.H * p.W;
      }
      const int acc = tl & 1;
      mbar_wait_sleep(&tfull[acc], (tl >> 1) & 1);
      tc_fence_after();
      float* ob = p.out + (long long)n * p.oimg + (long long)nt * p.BN * ostride + pos;
      const int ncol = min(p.BN, p.Co - nt * p.BN);
      for (int c0 = eg * 32; c0 < ncol; c0 += 64) {
        float v[32];
        tmem_ld32(tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t(acc * kMaxBN + c0), v);
        if (!live) continue;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (c0 + j >= ncol) break;
          float* dst = ob + (long long)(c0 + j) * ostride;
          const float val = p.alpha * v[j];
          if (p.s2 == 2) {
            // the 2x2 dx block of dy position (i, j): only its top-left
            // element has a tap (1x1 filter, stride 2); the rest get beta * dx
            const int i2 = pos / p.W, j2 = pos - i2 * p.W;
            const bool r1 = i2 + 1 < p.H, c1 = j2 + 1 < p.W;
            if (p.beta == 0.f) {
              dst[0] = val;
              if (c1) dst[1] = 0.f;
              if (r1) {
                dst[p.W] = 0.f;
                if (c1) dst[p.W + 1] = 0.f;
              }
            } else {
              dst[0] = val + p.beta * dst[0];
              if (c1) dst[1] = p.beta * dst[1];
              if (r1) {
                dst[p.W] = p.beta * dst[p.W];
                if (c1) dst[p.W + 1] = p.beta * dst[p.W + 1];
              }
            }
          } else {
            *dst = p.beta == 0.f ? val : val + p.beta * *dst;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

int sm_count() {
  static int v = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return v;
}

int pick_bn(int n, int quantum) {
  const int tiles = (n + kMaxBN - 1) / kMaxBN;
  return ((n + tiles - 1) / tiles + quantum - 1) / quantum * quantum;
}

}  // namespace

bool z1x1_supports(int op, const ConvShape& s) {
  if (op != kFwd && op != kBwdData) return false;
  if (s.R != 1 || s.S != 1 || s.ph != 0 || s.pw != 0 || s.sh != s.sw || (s.sh != 1 && s.sh != 2) ||
      !tune("z1x1", 1))
    return false;
  if (s.C % 4 || s.K % 4 || s.N >= 65536 || std::int64_t(s.C) * s.H * s.W >= (1ll << 31)) return false;
  if (s.sh == 1) return std::int64_t(s.H) * s.W % 4 == 0;
  // stride 2: BackwardData only -- a Forward would need a traversal stride
  // on the innermost (w) dimension, which TMA does not support (cuda.h:
  // elementStrides[0] is ignored without interleave)
  return op == kBwdData && std::int64_t(s.OH()) * s.OW() % 4 == 0 && tune("z1x1_s2", 1);
}

cudaError_t z1x1_run(int op, const ConvShape& s, const float* a, const float* w, float* out, float alpha, float beta,
                     cudaStream_t st) {
  const bool bd = op == kBwdData;
  const int OH = s.OH(), OW = s.OW();
  OParams p{};
  p.out = out; p.alpha = alpha; p.beta = beta;
  p.s2 = s.sh == 1 ? 0 : 2;
  p.OW = OW; p.H = s.H; p.W = s.W;
  // source plane: x (Forward), dy (BackwardData)
  const int HW = bd ? OH * OW : s.H * s.W;
  p.HW = HW;
  p.Cs = bd ? s.K : s.C;
  p.Co = bd ? s.C : s.K;
  p.bd = bd ? 1 : 0;
  p.BN = pick_bn(p.Co, bd ? 32 : 16);  // MN-major B comes in whole 32-column blocks
  p.n_tiles = (p.Co + p.BN - 1) / p.BN;
  p.tpi = (HW + kBM - 1) / kBM;
  p.units = s.N * p.tpi * p.n_tiles;
  p.chunks = (p.Cs + 31) / 32;
  p.oimg = std::int64_t(p.Co) * (bd ? std::int64_t(s.H) * s.W : std::int64_t(OH) * OW);
  if ((reinterpret_cast<std::uintptr_t>(a) | reinterpret_cast<std::uintptr_t>(w)) & 15) return cudaErrorMisalignedAddress;
  CUtensorMap amap{}, bmap{};
  {
    // source as (p, c, n): {32, 32, 1} boxes -> MN-major 32-position blocks
    const cuuint64_t dims[3] = {cuuint64_t(HW), cuuint64_t(p.Cs), cuuint64_t(s.N)};
    const cuuint64_t strides[2] = {cuuint64_t(HW) * 4, cuuint64_t(p.Cs) * HW * 4};
    const cuuint32_t box[3] = {32, 32, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (encode_tiled()(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(a), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    // w as (c, k): Forward {32 c, BN k} K-major boxes; BackwardData {32 c, 32 k} MN-major blocks
    const cuuint64_t dims[2] = {cuuint64_t(s.C), cuuint64_t(s.K)};
    const cuuint64_t strides[1] = {cuuint64_t(s.C) * 4};
    const cuuint32_t box[2] = {32, cuuint32_t(bd ? 32 : p.BN)};
    const cuuint32_t es[2] = {1, 1};
    if (encode_tiled()(&bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(w), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE,
                       bd ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int stage_bytes = int(kABytes) + ((p.BN * 128 + 1023) & ~1023);
  p.stages = std::max(2, std::min({kMaxStages, tune("z1_stages", 8), (200 * 1024) / stage_bytes}));
  const int smem = p.stages * stage_bytes + 1024 + 256;
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(z1x1_kernel), smem);
  if (e != cudaSuccess) return e;
  const int grid = std::min(p.units, sm_count());
  trace_variant("z1x1 bd=%d s2=%d tiles=%d n_tiles=%d BN=%d chunks=%d stages=%d grid=%d", p.bd, p.s2,
                p.units / p.n_tiles, p.n_tiles, p.BN, p.chunks, p.stages, grid);
  return launch_pdl(z1x1_kernel, dim3(grid), dim3(kThreads), std::size_t(smem), st, amap, bmap, p);
}

}  // namespace ucudnn
