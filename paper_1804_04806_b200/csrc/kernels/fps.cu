// Forward of few-channel strided layers (AlexNet conv1: 3 channels, 11x11,
// stride 4; ResNet conv1: 3 channels, 7x7, stride 2) from a space-to-depth
// patch in shared memory -- UCUDNN_ALGO_IMPLICIT_GEMM's path for these shapes
// (no workspace at all).
//
//   y[n][k][oh][ow] = alpha * sum_{c,r,s} x[n][c][oh*sh-ph+r][ow*sw-pw+s] * w[k][c][r][s] + beta * y
//   (reference_conv.hpp:70-100)
//
// GEMM: M = output positions (a tile = 4 blocks of 32: rpt output rows of
// bpr = ceil(OW / 32) blocks each), N = K output channels, reduction = the
// C*R*S filter taps in w's own (c, r, s) order. The zero-workspace gather
// (igemm_tc.cu) reads these operands at stride sw along a warp (16 sectors per
// instruction at stride 4); here a CTA copies, once per tile, the input rows
// its output rows need into shared memory split by column phase
//   P[c][rr][b][j] = x[n][c][oh0*sh - ph + rr][j*sw + b - pw]   (0 off the image)
// (the patch of bfs.cu, rows of rpt output rows together), and every A
// K-row (c, r, s) of a 32-position block is then one contiguous 32-float run
// of P: one conflict-free LDS + one STS into the MN-major 128B/32B-atom
// operand (DESIGN finding 5). B (filter rows, (c, r, s)-contiguous) arrives
// by cp.async. P is double-buffered: the next tile's fill overlaps this
// tile's last MMAs. Two TMEM accumulator sets: the NCHW epilogue of a tile
// overlaps the next tile's MMAs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "conv_common.h"
#include "fps.h"
#include "launch.h"
#include "sm100.cuh"

namespace ucudnn {
using namespace sm100;

namespace {

constexpr int kBM = 128;
constexpr int kProd = 16;
constexpr int kThreads = (5 + kProd) * 32;
constexpr int kMaxStages = 6;
constexpr int kMaxCRS = 512;
constexpr int kBRows = 4;  // filter rows per producer thread: K <= 16 * 4
constexpr std::uint32_t kABytes = kBM * 128;

struct FGeo {
  int N, C, H, W, K, R, S, ph, pw, sh, OH, OW;
  int crs, chunks, Kp;  // reduction rows, 32-row chunks, K padded to 16
  int bpr, rpt;         // 32-position blocks per output row, output rows per tile
  int RR, JP;           // patch rows, patch row pitch (floats)
  int tiles_per_img, units, grid, stages;
  std::size_t p_bytes, b_bytes, stage_bytes, smem;
};

struct FParams {
  const float* x;
  const float* w;
  float* y;
  float alpha, beta;
  int C, H, W, K, R, S, ph, pw, sh, shl, OH, OW;
  int crs, chunks, Kp, bpr, rpt, RR, JP, tiles_per_img, units, stages;
  int p_floats;
  long long CHW, KOHW;
};

__device__ __forceinline__ void cp_async4(std::uint32_t dst, const float* src, std::uint32_t src_size) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_size) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(std::uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
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
// MN-major 128B / 32 B-atom descriptor: LBO 4096 B between 32-position
// blocks, SBO 512 B (4 K-rows per atom)
__device__ __forceinline__ std::uint64_t desc_mn32(std::uint32_t saddr) {
  std::uint64_t d = 0;
  d |= std::uint64_t((saddr >> 4) & 0x3FFF);
  d |= std::uint64_t(4096 >> 4) << 16;
  d |= std::uint64_t(512 >> 4) << 32;
  d |= std::uint64_t(1) << 46;
  d |= std::uint64_t(1) << 61;
  return d;
}

__device__ __forceinline__ void unit_origin(const FParams& p, int u, int& n, int& oh0) {
  n = u / p.tiles_per_img;
  oh0 = (u - n * p.tiles_per_img) * p.rpt;
}

// patch of tile u into buffer pb: C*RR input rows x JP*sh columns (sh == sw)
__device__ __forceinline__ void fill_patch(const FParams& p, int u, std::uint32_t pb, int pw, int lane) {
  int n, oh0;
  unit_origin(p, u, n, oh0);
  const int cols = p.JP * p.sh;
  const float* xn = p.x + (long long)n * p.CHW;
  for (int cr = pw; cr < p.C * p.RR; cr += kProd) {
    const int c = cr / p.RR, rr = cr - c * p.RR;
    const int ih = oh0 * p.sh - p.ph + rr;
    const bool rok = unsigned(ih) < unsigned(p.H);
    const float* row = xn + ((long long)c * p.H + (rok ? ih : 0)) * p.W;
    const std::uint32_t dst0 =
        pb + std::uint32_t(cr * p.sh * p.JP + (lane & (p.sh - 1)) * p.JP + (lane >> p.shl)) * 4;
    const std::uint32_t jstep = std::uint32_t(32 >> p.shl) * 4;
    const float* src0 = row + lane - p.pw;
    const int iw0 = lane - p.pw;
    for (int it = 0; it * 32 < cols; ++it) {
      const bool ok = rok && unsigned(iw0 + 32 * it) < unsigned(p.W);
      cp_async4(dst0 + std::uint32_t(it) * jstep, ok ? src0 + 32 * it : row, ok ? 4u : 0u);
    }
  }
  cp_async_commit();
}

__global__ void __launch_bounds__(kThreads, 1) fps_kernel(const FParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t b_bytes = (std::uint32_t(p.Kp) * 128 + 1023) & ~1023u;
  const std::uint32_t stage_bytes = kABytes + b_bytes;
  const int kStages = p.stages;
  float* P = reinterpret_cast<float*>(smem + kStages * stage_bytes);
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(P + 2 * p.p_floats);
  std::uint64_t* empty = full + kMaxStages;
  std::uint64_t* tfull = empty + kMaxStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  __shared__ int pofs[kMaxCRS];  // reduction row (c, r, s) -> its run in a P buffer (tile row 0)

  for (int j = threadIdx.x; j < p.chunks * 32; j += blockDim.x) {
    int o = -1;
    if (j < p.crs) {
      const int RS = p.R * p.S;
      const int c = j / RS, rs = j - c * RS, r = rs / p.S, s = rs - r * p.S;
      o = ((c * p.RR + r) * p.sh + s % p.sh) * p.JP + s / p.sh;
    }
    pofs[j] = o;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 2 * kProd * 32);  // per producer thread: STS arrive + cp.async arrive
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    mbar_fence_init();
  }
  if (warp == 4) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = tmem_base_uniform(tmem_slot);
  const int my_units = blockIdx.x < p.units ? (p.units - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;

  if (warp >= 5) {
    // ------------------------------------------------ producers
    const int pw = warp - 5;
    const int blk = pw & 3;  // A block this warp builds: output row t, columns ow0 .. ow0 + 31
    const int jq = pw >> 2;  // its K-rows j = jq + 4 i (j & 3 == jq: a fixed swizzle phase)
    const int t = blk / p.bpr, ow0 = (blk - t * p.bpr) * 32;
    const bool blk_live = t < p.rpt;
    const std::uint32_t sbase = smem_u32(smem);
    const std::uint32_t p0 = smem_u32(P);
    // A: K-row j of block blk at blk*4096 + j*128, 32 B granule (lane/8) ^ (j & 3)
    const std::uint32_t adst = std::uint32_t(blk) * 4096 + std::uint32_t(jq) * 128 +
                               ((std::uint32_t(lane >> 3) ^ std::uint32_t(jq)) << 5) + std::uint32_t(lane & 7) * 4;
    const std::uint32_t bsw = std::uint32_t(lane >> 2), bl = std::uint32_t(lane & 3) * 4;
    // this thread's filter rows: source pointer (advanced by 32 per chunk)
    // and B-tile destination, computed once
    const float* bsrc[kBRows];
    std::uint32_t bdst[kBRows];
    bool brow[kBRows];
#pragma unroll
    for (int q = 0; q < kBRows; ++q) {
      const int k = pw + kProd * q;
      brow[q] = k < p.K;
      bsrc[q] = p.w + (brow[q] ? (long long)k * p.crs + lane : 0);
      bdst[q] = std::uint32_t(k) * 128 + ((bsw ^ std::uint32_t(k & 7)) << 4) + bl;
    }
    int st = 0;
    std::uint32_t ph = 0, buf = 0;
    if (my_units > 0) {
      fill_patch(p, blockIdx.x, p0, pw, lane);
      cp_async_wait_all();
      named_sync(1, kProd * 32);
    }
    for (int i = 0; i < my_units; ++i) {
      const int u = blockIdx.x + i * gridDim.x;
      int n, oh0;
      unit_origin(p, u, n, oh0);
      const bool live = blk_live && oh0 + t < p.OH;
      // this block's runs start at row t of the tile, column ow0
      const std::uint32_t pbase =
          p0 + buf * std::uint32_t(p.p_floats) * 4 + std::uint32_t(t * p.sh * p.sh * p.JP + ow0 + lane) * 4;
      for (int ch = 0; ch < p.chunks; ++ch) {
        mbar_wait(&empty[st], ph ^ 1);
        const std::uint32_t sa = sbase + st * stage_bytes, sb = sa + kABytes;
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int o = pofs[ch * 32 + jq + 4 * q];
          v[q] = 0.f;
          if (live && o >= 0) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[q]) : "r"(pbase + std::uint32_t(o) * 4));
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(sa + adst + std::uint32_t(q) * 512), "f"(v[q]) : "memory");
        // B: filter rows k = pw + 16 i, 32 reduction entries each
        const bool kok = ch * 32 + lane < p.crs;
#pragma unroll
        for (int q = 0; q < kBRows; ++q)
          if (pw + kProd * q < p.Kp)
            cp_async4(sb + bdst[q], bsrc[q] + ch * 32, (kok && brow[q]) ? 4u : 0u);
        mbar_arrive(&full[st]);
        cp_async_arrive(&full[st]);
        if (++st == kStages) {
          st = 0;
          ph ^= 1;
        }
      }
      if (i + 1 < my_units) {
        fill_patch(p, u + gridDim.x, p0 + (buf ^ 1) * std::uint32_t(p.p_floats) * 4, pw, lane);
        cp_async_wait_all();
        named_sync(1, kProd * 32);
        buf ^= 1;
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------------ MMA issuer
    const std::uint32_t idesc = idesc_tf32(kBM, p.Kp) | (1u << 15);  // A MN-major, B K-major
    const std::uint32_t sbase = smem_u32(smem);
    int it = 0;
    for (int i = 0; i < my_units; ++i) {
      const int acc = i & 1;
      mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const std::uint32_t dtm = tmem + std::uint32_t(acc * 256);
      for (int ch = 0; ch < p.chunks; ++ch, ++it) {
        const int st = it % kStages;
        mbar_wait(&full[st], (it / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          fence_async_smem();
          const std::uint32_t sa = sbase + st * stage_bytes, sb = sa + kABytes;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            mma_tf32(dtm, desc_mn32(sa + j * 1024), umma_desc_sw128(sb + j * 32), idesc, (ch | j) ? 1u : 0u);
          mma_commit(&empty[st]);
          if (ch + 1 == p.chunks) mma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ epilogue: TMEM lane = position of block `warp`
    const int t = warp / p.bpr, ow = (warp - t * p.bpr) * 32 + lane;
    for (int i = 0; i < my_units; ++i) {
      const int u = blockIdx.x + i * gridDim.x;
      int n, oh0;
      unit_origin(p, u, n, oh0);
      const int acc = i & 1;
      mbar_wait_sleep(&tfull[acc], (i >> 1) & 1);
      tc_fence_after();
      const bool live = t < p.rpt && oh0 + t < p.OH && ow < p.OW;
      float* yb = p.y + (long long)n * p.KOHW + (long long)(oh0 + t) * p.OW + ow;
      const long long ks = (long long)p.OH * p.OW;
      for (int c0 = 0; c0 < p.K; c0 += 32) {
        float v[32];
        tmem_ld32(tmem + (std::uint32_t(warp * 32) << 16) + std::uint32_t(acc * 256 + c0), v);
        if (!live) continue;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (c0 + j >= p.K) break;
          float* dst = yb + (long long)(c0 + j) * ks;
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
  if (warp == 4) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
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

FGeo make_fgeo(const ConvShape& s) {
  FGeo g{};
  g.N = s.N; g.C = s.C; g.H = s.H; g.W = s.W; g.K = s.K; g.R = s.R; g.S = s.S;
  g.ph = s.ph; g.pw = s.pw; g.sh = s.sh; g.OH = s.OH(); g.OW = s.OW();
  g.crs = s.C * s.R * s.S;
  g.chunks = (g.crs + 31) / 32;
  g.Kp = (s.K + 15) / 16 * 16;
  g.bpr = (g.OW + 31) / 32;
  g.rpt = g.bpr <= 4 && 4 % g.bpr == 0 ? 4 / g.bpr : 1;
  g.RR = (g.rpt - 1) * s.sh + s.R;
  const int need = g.bpr * 32 + (s.S - 1) / s.sw;
  const int m = 32 / std::max(1, s.sw);
  g.JP = need;
  while (g.JP % 32 != m % 32) ++g.JP;
  g.tiles_per_img = (g.OH + g.rpt - 1) / g.rpt;
  g.units = s.N * g.tiles_per_img;
  g.grid = std::min(sm_count(), g.units);
  g.p_bytes = std::size_t(s.C) * g.RR * s.sw * g.JP * 4;
  g.b_bytes = (std::size_t(g.Kp) * 128 + 1023) & ~std::size_t(1023);
  g.stage_bytes = kABytes + g.b_bytes;
  g.stages = 2;
  while (g.stages < kMaxStages && (g.stages + 1) * g.stage_bytes + 2 * g.p_bytes + 1024 + 256 <= 220 * 1024)
    ++g.stages;
  g.stages = std::max(2, std::min(g.stages, tune("fps_stages", kMaxStages)));
  g.smem = g.stages * g.stage_bytes + 2 * g.p_bytes + 1024 + 256;
  return g;
}

}  // namespace

bool fps_supports(const ConvShape& s) {
  if (s.sh != s.sw || (s.sh != 2 && s.sh != 4) || s.C > 4 || s.K > kProd * kBRows || !tune("fps", 1)) return false;
  const FGeo g = make_fgeo(s);
  return g.bpr <= 4 && g.chunks * 32 <= kMaxCRS && g.smem <= 220 * 1024 &&
         std::int64_t(s.N) * s.K * g.OH * g.OW < (1ll << 40);
}

cudaError_t fps_run(const ConvShape& s, const float* x, const float* w, float* y, float alpha, float beta,
                    cudaStream_t st) {
  const FGeo g = make_fgeo(s);
  FParams p{};
  p.x = x; p.w = w; p.y = y; p.alpha = alpha; p.beta = beta;
  p.C = g.C; p.H = g.H; p.W = g.W; p.K = g.K; p.R = g.R; p.S = g.S; p.ph = g.ph; p.pw = g.pw; p.sh = g.sh;
  p.shl = g.sh == 4 ? 2 : 1;
  p.OH = g.OH; p.OW = g.OW;
  p.crs = g.crs; p.chunks = g.chunks; p.Kp = g.Kp; p.bpr = g.bpr; p.rpt = g.rpt; p.RR = g.RR; p.JP = g.JP;
  p.tiles_per_img = g.tiles_per_img; p.units = g.units; p.stages = g.stages;
  p.p_floats = int(g.p_bytes / 4);
  p.CHW = std::int64_t(g.C) * g.H * g.W;
  p.KOHW = std::int64_t(g.K) * g.OH * g.OW;
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(fps_kernel), int(g.smem));
  if (e != cudaSuccess) return e;
  trace_variant("fps units=%d grid=%d crs=%d Kp=%d bpr=%d rpt=%d JP=%d stages=%d", g.units, g.grid, g.crs, g.Kp, g.bpr,
                g.rpt, g.JP, g.stages);
  return launch_pdl(fps_kernel, dim3(g.grid), dim3(kThreads), g.smem, st, p);
}

}  // namespace ucudnn
