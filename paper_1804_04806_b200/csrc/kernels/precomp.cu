// UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM: implicit GEMM fed entirely by TMA.
//
// NCHW fp32 rows of odd width (27, 13, 55 ... floats) violate TMA's 16-byte
// stride rule, so this algorithm first re-lays the micro-batch's activation
// into a channels-last copy in the workspace (HBM-bound, ~2x the activation
// bytes) and pre-tiles the filter into the UMMA canonical layout. The main
// loop then issues, per 32-deep reduction step, one TMA *im2col* load for
// the 128-pixel A tile (zero-fill supplies the padding, the traversal stride
// supplies the conv stride) and one bulk copy for the B tile -- no SIMT work
// at all on the operand path. Workspace grows with the micro-batch
// (b * H * W * C_pad * 4 + |W|), which is exactly the trade micro-batching
// exploits.
//
// Persistent kernel, one CTA per SM, 256 threads:
//   warp 0 lane 0  TMA / bulk-copy producer over a 4-deep smem ring
//   warp 1         TMEM owner + tcgen05.mma issuer (double-buffered
//                  accumulators: 2 x 256 TMEM columns)
//   warps 4-7      epilogue: TMEM -> registers -> NCHW with alpha/beta,
//                  overlapping the next tile's main loop.
// Forward and stride-1 BackwardData share it (BackwardData = forward conv of
// dy with the flipped, transposed filter and padding R-1-p).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>

#include "bfilter.h"
#include "conv_common.h"
#include "precomp.h"
#include "sm100.cuh"

namespace ucudnn {
using namespace sm100;

namespace {

constexpr int kBM = 128;
constexpr int kStages = 4;
constexpr int kThreads = 256;
constexpr int kMaxBN = 256;

struct PrecompParams {
  const float* btiles;  // [n_tile][kstep][8 kgroups][BN rows][4]
  float* out;
  float alpha, beta;
  int M;         // output pixels (rows)
  int Nout;      // output channels (cols)
  int P;         // output pixels per image
  int BN, n_tiles, m_tiles, ksteps;
  int small_c;   // 1: 4-channel taps, 8 taps per step; 0: 32 channels of one tap per step
  int taps, S, c_chunks;
  int OW, OHW, sh, sw, ph, pw;  // output geometry in the *input* frame of the TMA map
  FastDiv fd_P, fd_OW, fd_mt;
};

__device__ __forceinline__ void tile_coords(const PrecompParams& p, int t, int& mt, int& nt) {
  std::uint32_t q, r;
  p.fd_mt.divmod(std::uint32_t(t), q, r);
  nt = int(q);
  mt = int(r);
}

__global__ void __launch_bounds__(kThreads, 1)
    precomp_kernel(const __grid_constant__ CUtensorMap amap, const PrecompParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t a_bytes = kBM * 128;
  const std::uint32_t b_bytes = std::uint32_t(p.BN) * 128;
  const std::uint32_t stage_bytes = a_bytes + ((b_bytes + 1023) & ~1023u);
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kStages * stage_bytes);
  std::uint64_t* empty = full + kStages;
  std::uint64_t* tfull = empty + kStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);

  if (threadIdx.x == 0) {
    prefetch_tmap(&amap);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;
  const int total_tiles = p.m_tiles * p.n_tiles;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ producer
      int it = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        int mt, nt;
        tile_coords(p, t, mt, nt);
        // TMA start coordinate of the tile's first output pixel (raster order)
        std::uint32_t n, pix, oh, ow;
        p.fd_P.divmod(std::uint32_t(mt * kBM), n, pix);
        p.fd_OW.divmod(pix, oh, ow);
        const int cw = int(ow) * p.sw - p.pw, ch = int(oh) * p.sh - p.ph;
        const float* bsrc = p.btiles + std::size_t(nt) * p.ksteps * (b_bytes / 4);
        for (int k = 0; k < p.ksteps; ++k, ++it) {
          const int s = it % kStages;
          mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          unsigned char* sa = smem + s * stage_bytes;
          mbar_expect_tx(&full[s], a_bytes + b_bytes);
          if (p.small_c) {
#pragma unroll 1
            for (int g = 0; g < 8; ++g) {
              int tap = k * 8 + g;
              if (tap >= p.taps) tap = p.taps - 1;  // its B rows are zero
              const int r = tap / p.S, q = tap - r * p.S;
              tma_im2col_4d(sa + g * (kBM * 16), &amap, &full[s], 0, cw, ch, int(n), (unsigned short)q,
                            (unsigned short)r);
            }
          } else {
            const int tap = k / p.c_chunks, cc = k - tap * p.c_chunks;
            const int r = tap / p.S, q = tap - r * p.S;
            tma_im2col_4d(sa, &amap, &full[s], cc * 32, cw, ch, int(n), (unsigned short)q, (unsigned short)r);
          }
          bulk_g2s(sa + a_bytes, bsrc + std::size_t(k) * (b_bytes / 4), b_bytes, &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN);
    const std::uint32_t sbase = smem_u32(smem);
    const std::uint32_t lbo_b = std::uint32_t(p.BN) * 16;
    int it = 0, tl = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++tl) {
      const int acc = tl & 1;
      mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
      tc_fence_after();
      const std::uint32_t dtm = tmem + std::uint32_t(acc * kMaxBN);
      for (int k = 0; k < p.ksteps; ++k, ++it) {
        const int s = it % kStages;
        mbar_wait(&full[s], (it / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          const std::uint32_t sa = sbase + s * stage_bytes, sb = sa + a_bytes;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            std::uint64_t ad = p.small_c ? umma_desc(sa + 2 * q * (kBM * 16), kBM * 16, 128)
                                         : umma_desc_sw128(sa + q * 32);
            std::uint64_t bd = umma_desc(sb + 2 * q * lbo_b, lbo_b, 128);
            mma_tf32(dtm, ad, bd, idesc, (k | q) != 0);
          }
          mma_commit(&empty[s]);
          if (k == p.ksteps - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue
    const int ew = warp - 4;
    int tl = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++tl) {
      int mt, nt;
      tile_coords(p, t, mt, nt);
      const int acc = tl & 1;
      mbar_wait(&tfull[acc], (tl >> 1) & 1);
      tc_fence_after();
      const int row = mt * kBM + ew * 32 + lane;
      const bool ok = row < p.M;
      std::int64_t obase = 0;
      if (ok) {
        std::uint32_t n, pix;
        p.fd_P.divmod(std::uint32_t(row), n, pix);
        obase = std::int64_t(n) * p.Nout * p.P + pix;
      }
      const std::uint32_t tbase = tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t(acc * kMaxBN);
      for (int c0 = 0; c0 < p.BN; c0 += 32) {
        float v[32];
        tmem_ld32(tbase + std::uint32_t(c0), v);
        if (!ok) continue;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = nt * p.BN + c0 + j;
          if (c0 + j >= p.BN || col >= p.Nout) break;
          float* dst = p.out + obase + std::int64_t(col) * p.P;
          const float val = p.alpha * v[j];
          *dst = p.beta == 0.f ? val : val + p.beta * *dst;
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

// NCHW -> N(HW)Cp, zero-filling channels C..Cp-1 (32 x 32 smem transpose).
__global__ void to_nhwc_kernel(const float* __restrict__ src, float* __restrict__ dst, int C, int HW, int Cp) {
  __shared__ float tile[32][33];
  const int n = blockIdx.z;
  const int p0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const float* s = src + std::int64_t(n) * C * HW;
  float* d = dst + std::int64_t(n) * HW * Cp;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, pp = p0 + threadIdx.x;
    tile[i][threadIdx.x] = (c < C && pp < HW) ? s[std::int64_t(c) * HW + pp] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int pp = p0 + i, c = c0 + threadIdx.x;
    if (pp < HW && c < Cp) d[std::int64_t(pp) * Cp + c] = tile[threadIdx.x][i];
  }
}

// Filter -> B tiles [n_tile][kstep][kgroup 8][BN][4]. Output channel o,
// reduction (tap, ch). Forward: W[o][ch][tap]; flip_transpose (stride-1
// BackwardData): W[ch][o][taps-1-tap] with rows o over C and ch over K.
__global__ void pack_filter_kernel(const float* __restrict__ w, float* __restrict__ out, int O, int I, int taps,
                                   int BN, int n_tiles, int ksteps, int small_c, int c_chunks, int flip) {
  const std::int64_t total = std::int64_t(n_tiles) * ksteps * 8 * BN;  // 16-byte units
  for (std::int64_t u = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; u < total;
       u += std::int64_t(gridDim.x) * blockDim.x) {
    const int row = int(u % BN);
    std::int64_t rest = u / BN;
    const int g = int(rest % 8);
    rest /= 8;
    const int k = int(rest % ksteps);
    const int nt = int(rest / ksteps);
    const int o = nt * BN + row;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int tap, ch;
      if (small_c) {
        tap = k * 8 + g;
        ch = e;
      } else {
        tap = k / c_chunks;
        ch = (k - tap * c_chunks) * 32 + g * 4 + e;
      }
      float x = 0.f;
      if (o < O && ch < I && tap < taps)
        x = flip ? w[(std::int64_t(ch) * O + o) * taps + (taps - 1 - tap)] : w[(std::int64_t(o) * I + ch) * taps + tap];
      v[e] = x;
    }
    reinterpret_cast<float4*>(out)[u] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

PFN_cuTensorMapEncodeIm2col_v12000 encode_im2col() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(f);
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

int cpad(int c) { return c <= 4 ? 4 : (c + 31) / 32 * 32; }
int pick_bn(int n) {
  int tiles = (n + 255) / 256;
  return ((n + tiles - 1) / tiles + 15) / 16 * 16;
}
std::size_t align256(std::size_t b) { return (b + 255) / 256 * 256; }

// Geometry of one launch: input (Cin x Hin x Win, NHWC copy with Cp
// channels) convolved to (Nout x Hout x Wout) by an R x S filter.
struct Geo {
  int N, Cin, Hin, Win, Nout, Hout, Wout, R, S, ph, pw, sh, sw;
};

std::size_t geo_ws(const Geo& g, int* ksteps_out = nullptr, int* bn_out = nullptr) {
  const int Cp = cpad(g.Cin), taps = g.R * g.S;
  const bool small = Cp == 4;
  const int ksteps = small ? (taps + 7) / 8 : taps * (Cp / 32);
  const int BN = pick_bn(g.Nout), n_tiles = (g.Nout + BN - 1) / BN;
  if (ksteps_out) *ksteps_out = ksteps;
  if (bn_out) *bn_out = BN;
  return align256(std::size_t(n_tiles) * ksteps * BN * 128) + align256(std::size_t(g.N) * g.Hin * g.Win * Cp * 4);
}

cudaError_t run_geo(const Geo& g, const float* act, const float* w, int flip, float* out, void* ws, float alpha,
                    float beta, cudaStream_t st, int flags) {
  const int Cp = cpad(g.Cin), taps = g.R * g.S;
  int ksteps = 0, BN = 0;
  geo_ws(g, &ksteps, &BN);
  const int n_tiles = (g.Nout + BN - 1) / BN;
  // packed filter first: its size does not depend on the micro-batch, so
  // later micro-batches of the same call reuse it (kFilterReady)
  float* btiles = static_cast<float*>(ws);
  float* act_nhwc = reinterpret_cast<float*>(static_cast<char*>(ws) +
                                             align256(std::size_t(n_tiles) * ksteps * BN * 128));
  const int HW = g.Hin * g.Win;
  count_launch();
  to_nhwc_kernel<<<dim3((HW + 31) / 32, (Cp + 31) / 32, g.N), dim3(32, 8), 0, st>>>(act, act_nhwc, g.Cin, HW, Cp);
  if (!(flags & kFilterReady)) {
    const std::int64_t units = std::int64_t(n_tiles) * ksteps * 8 * BN;
    const int blocks = int(std::min<std::int64_t>((units + 255) / 256, 8 * sm_count()));
    count_launch();
    pack_filter_kernel<<<blocks, 256, 0, st>>>(w, btiles, g.Nout, g.Cin, taps, BN, n_tiles, ksteps, Cp == 4 ? 1 : 0,
                                               Cp / 32, flip);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  CUtensorMap amap;
  const cuuint64_t dims[4] = {cuuint64_t(Cp), cuuint64_t(g.Win), cuuint64_t(g.Hin), cuuint64_t(g.N)};
  const cuuint64_t strides[3] = {cuuint64_t(Cp) * 4, cuuint64_t(Cp) * 4 * g.Win, cuuint64_t(Cp) * 4 * g.Win * g.Hin};
  const int lower[2] = {-g.pw, -g.ph};
  const int upper[2] = {g.pw - (g.S - 1), g.ph - (g.R - 1)};
  const cuuint32_t estr[4] = {1, cuuint32_t(g.sw), cuuint32_t(g.sh), 1};
  const bool small = Cp == 4;
  CUresult r = encode_im2col()(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, act_nhwc, dims, strides, lower, upper,
                               small ? 4 : 32, kBM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               small ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  int drv = 0;
  cudaDriverGetVersion(&drv);
  if (drv <= 13010 && std::size_t(g.N) * HW * Cp * 4 < 131072)  // encoder quirk (see CUTLASS im2col traits)
    reinterpret_cast<std::uint64_t*>(&amap)[1] &= ~(1ull << 21);

  PrecompParams p{};
  p.btiles = btiles;
  p.out = out;
  p.alpha = alpha;
  p.beta = beta;
  p.P = g.Hout * g.Wout;
  p.M = g.N * p.P;
  p.Nout = g.Nout;
  p.BN = BN;
  p.n_tiles = n_tiles;
  p.m_tiles = (p.M + kBM - 1) / kBM;
  p.ksteps = ksteps;
  p.small_c = small ? 1 : 0;
  p.taps = taps;
  p.S = g.S;
  p.c_chunks = Cp / 32;
  p.OW = g.Wout;
  p.OHW = p.P;
  p.sh = g.sh;
  p.sw = g.sw;
  p.ph = g.ph;
  p.pw = g.pw;
  p.fd_P = FastDiv(std::uint32_t(p.P));
  p.fd_OW = FastDiv(std::uint32_t(g.Wout));
  p.fd_mt = FastDiv(std::uint32_t(p.m_tiles));
  const int stage_bytes = kBM * 128 + ((BN * 128 + 1023) & ~1023);
  // >= 116 KB so the persistent grid lands one CTA per SM (each owns all
  // 512 TMEM columns)
  const int smem = std::max(kStages * stage_bytes + 1024 + 256, 116 * 1024);
  static int smem_set = 0;
  if (smem > smem_set) {
    e = cudaFuncSetAttribute(precomp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    smem_set = 227 * 1024;
  }
  const int grid = std::min(sm_count(), p.m_tiles * p.n_tiles);
  count_launch();
  precomp_kernel<<<grid, kThreads, smem, st>>>(amap, p);
  return cudaGetLastError();
}

Geo fwd_geo(const ConvShape& s) {
  return Geo{s.N, s.C, s.H, s.W, s.K, s.OH(), s.OW(), s.R, s.S, s.ph, s.pw, s.sh, s.sw};
}
// stride-1 BackwardData as a forward conv of dy with the flipped filter
Geo bwd_data_geo(const ConvShape& s) {
  return Geo{s.N, s.K, s.OH(), s.OW(), s.C, s.H, s.W, s.R, s.S, s.R - 1 - s.ph, s.S - 1 - s.pw, 1, 1};
}

}  // namespace

bool precomp_supports(int op, const ConvShape& s) {
  if (op == kFwd) return s.sh <= 8 && s.sw <= 8 && s.ph <= 127 && s.pw <= 127 && s.R <= 64 && s.S <= 64;
  if (op == kBwdData) return s.sh == 1 && s.sw == 1 && s.ph <= s.R - 1 && s.pw <= s.S - 1;
  // BackwardFilter: TMA-tiled phase-split operands (bfilter.cu)
  return bf_supports(s);
}

std::int64_t precomp_workspace(int op, const ConvShape& s) {
  if (op == kFwd) return std::int64_t(geo_ws(fwd_geo(s)));
  if (op == kBwdData) return std::int64_t(geo_ws(bwd_data_geo(s)));
  return bf_workspace(s);
}

cudaError_t precomp_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                        float beta, cudaStream_t st, int flags) {
  if (op == kFwd) return run_geo(fwd_geo(s), a, b, 0, out, ws, alpha, beta, st, flags);
  if (op == kBwdData) return run_geo(bwd_data_geo(s), a, b, 1, out, ws, alpha, beta, st, flags);
  return bf_run(s, a, b, out, ws, alpha, beta, st);
}

}  // namespace ucudnn
