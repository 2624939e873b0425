// BackwardFilter of few-channel strided layers (AlexNet conv1: 3 channels,
// 11x11, stride 4; ResNet conv1: 3 channels, 7x7, stride 2) through a
// space-to-depth patch in shared memory -- part of UCUDNN_ALGO_IMPLICIT_GATHER_GEMM (6).
//
//   dW[k][c][r][s] = beta * dW + alpha * sum_{n,oh,ow} dy[n][k][oh][ow] * x[n][c][oh*sh-ph+r][ow*sw-pw+s]
//   (reference_conv.hpp:141-180)
//
// GEMM (roles swapped as in bflsu.cu): M = k (<= 128), N = x rows q = (c, r, s)
// in dW's own order, reduction = output pixels. The gather kernel reads each
// x row of a 32-pixel step at stride sw from L2 (AlexNet conv1: 32 lanes span
// 512 B, 16 sectors per instruction, ~363 such instructions per step: L1
// bound, 0.55 ms at 256 images). Here a CTA owns whole output rows (n, oh):
// per row it copies the x patch the row needs once -- C x R input rows,
// coalesced -- into shared memory split by column phase,
//   P[c][r][b][j] = x[n][c][oh*sh - ph + r][j*sw + b - pw]   (0 off the image),
// and then every x row q = (c, r, s) of a step is a *contiguous* 32-float run
// of P (j = ow + s / sw, phase b = s % sw): one conflict-free LDS + one STS
// into the SW128 K-major B tile. dy rows (32 pixels of k) arrive by cp.async.
// The P row pitch JP is chosen = 32 / sw (mod 32) so the phase-splitting
// writes of the fill are conflict-free too; P is double-buffered, the next
// row's fill (cp.async) overlapping the current row's last MMAs.
//
// Each CTA accumulates its rows in TMEM (<= 512 columns: N <= 512 x rows,
// split into two MMAs of <= 256) and at the end stores its partial sums to
// its own workspace slice; a finalize kernel adds the slices in a fixed order
// -- so this BackwardFilter is deterministic (no atomics anywhere).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "bfs.h"
#include "conv_common.h"
#include "launch.h"
#include "sm100.cuh"

namespace ucudnn {
using namespace sm100;

namespace {

constexpr int kBM = 128;
constexpr int kProd = 16;
constexpr int kRowsPer = 24;  // x rows per producer thread (rows_pad <= 16 * 24 = 384)
constexpr int kThreads = (5 + kProd) * 32;
constexpr int kMaxStages = 4;
constexpr int kMaxRows = kProd * kRowsPer;

struct SGeo {
  int N, C, H, W, K, R, S, ph, pw, sh, sw, OH, OW;
  int rows, rows_pad, n1, n2;  // x rows C*R*S, padded to 16, MMA halves
  int steps;                   // 32-pixel steps per output row
  int JP;                      // P row pitch (floats)
  int units;                   // output rows N*OH
  int grid;
  std::size_t p_bytes, b_bytes, stage_bytes, smem;
  int stages;
};

struct SParams {
  const float* x;
  const float* dy;
  float* slices;
  int C, H, W, K, R, S, ph, pw, sh, shl, OH, OW;  // shl = log2(sh)
  int rows, rows_pad, n1, n2, steps, JP, units;
  int p_floats;  // one P buffer
  int stages;
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
  std::uint32_t ok = 0, ns = 256;
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
    if (ns < 8192) ns <<= 1;
  }
}

// P fill of output row u (n, oh) into buffer pb: C*R input rows x JP*sw columns
__device__ __forceinline__ void fill_patch(const SParams& p, int u, std::uint32_t pb, int pw, int lane) {
  const int n = u / p.OH, oh = u - n * p.OH;
  const int cols = p.JP * p.sh;  // sh == sw
  const float* xn = p.x + (long long)n * p.CHW;
  for (int cr = pw; cr < p.C * p.R; cr += kProd) {
    const int c = cr / p.R, r = cr - c * p.R;
    const int ih = oh * p.sh - p.ph + r;
    const bool rok = unsigned(ih) < unsigned(p.H);
    const float* row = xn + ((long long)c * p.H + (rok ? ih : 0)) * p.W;
    // column col = lane + 32 * it: its phase b = lane % sh is fixed per lane
    // (sh divides 32) and j advances by 32 / sh per iteration
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

__global__ void __launch_bounds__(kThreads, 1) bfs_kernel(const SParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t a_bytes = kBM * 128;
  const std::uint32_t b_bytes = (std::uint32_t(p.rows_pad) * 128 + 1023) & ~1023u;
  const std::uint32_t stage_bytes = a_bytes + b_bytes;
  const int kStages = p.stages;
  float* P = reinterpret_cast<float*>(smem + kStages * stage_bytes);  // two buffers of p_floats
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(P + 2 * p.p_floats);
  std::uint64_t* empty = full + kMaxStages;
  std::uint64_t* tfull = empty + kMaxStages;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tfull + 1);
  __shared__ int pofs[kMaxRows];  // x row q -> offset of its run in a P buffer (-1: padding row)

  // the A rows k >= K stay zero for the whole kernel
  for (int i = threadIdx.x; i < kStages * int(stage_bytes / 4); i += blockDim.x)
    reinterpret_cast<float*>(smem)[i] = 0.f;
  for (int q = threadIdx.x; q < p.rows_pad; q += blockDim.x) {
    int o = -1;
    if (q < p.rows) {
      const int RS = p.R * p.S;
      const int c = q / RS, rs = q - c * RS, r = rs / p.S, s = rs - r * p.S;
      o = ((c * p.R + r) * p.sh + s % p.sh) * p.JP + s / p.sh;
    }
    pofs[q] = o;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 2 * kProd * 32);  // per producer thread: STS arrive + cp.async arrive
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_fence_init();
  }
  if (warp == 4) tmem_alloc<512>(tmem_slot);
  fence_async_smem();  // the zeroed A rows are read by the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = tmem_base_uniform(tmem_slot);
  const int my_units = blockIdx.x < p.units ? (p.units - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  const int total_steps = my_units * p.steps;

  if (warp >= 5) {
    // ------------------------------------------------ producers
    const int pw = warp - 5;
    const std::uint32_t sbase = smem_u32(smem);
    const std::uint32_t p0 = smem_u32(P);
    int st = 0;
    std::uint32_t ph = 0, buf = 0;
    if (my_units > 0) {
      fill_patch(p, blockIdx.x, p0, pw, lane);
      cp_async_wait_all();
      named_sync(1, kProd * 32);
    }
    const std::uint32_t bsw = std::uint32_t(lane >> 2), bl = std::uint32_t(lane & 3) * 4;
    // this thread's x rows q = pw + kProd * i: patch offset and B-tile
    // destination, in registers (the build loop is then kRowsPer independent
    // LDS -> STS pairs instead of a dependent table walk)
    int po[kRowsPer];
    std::uint32_t bd[kRowsPer];
#pragma unroll
    for (int i = 0; i < kRowsPer; ++i) {
      const int q = pw + kProd * i;
      po[i] = q < p.rows_pad ? pofs[q] : -2;
      bd[i] = std::uint32_t(q) * 128 + ((bsw ^ std::uint32_t(q & 7)) << 4) + bl;
    }
    for (int i = 0; i < my_units; ++i) {
      const int u = blockIdx.x + i * gridDim.x;
      const int n = u / p.OH, oh = u - n * p.OH;
      const std::uint32_t Pb = p0 + buf * std::uint32_t(p.p_floats) * 4 + std::uint32_t(lane) * 4;
      const float* dyrow = p.dy + (long long)n * p.KOHW + (long long)oh * p.OW;
      for (int t = 0; t < p.steps; ++t) {
        const int ow0 = t * 32;
        mbar_wait(&empty[st], ph ^ 1);
        const std::uint32_t sa = sbase + st * stage_bytes, sb = sa + a_bytes;
        // B: x rows of this step from the patch
        float v[kRowsPer];
        const std::uint32_t pst = Pb + std::uint32_t(ow0) * 4;
#pragma unroll
        for (int r = 0; r < kRowsPer; ++r) {
          v[r] = 0.f;
          if (po[r] >= 0) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[r]) : "r"(pst + std::uint32_t(po[r]) * 4));
        }
#pragma unroll
        for (int r = 0; r < kRowsPer; ++r)
          if (po[r] != -2) asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + bd[r]), "f"(v[r]) : "memory");
        // A: dy rows k of the step's 32 pixels (zero past the row's end)
        const bool pok = ow0 + lane < p.OW;
        for (int k = pw; k < p.K; k += kProd)
          cp_async4(sa + std::uint32_t(k) * 128 + ((bsw ^ std::uint32_t(k & 7)) << 4) + bl,
                    dyrow + (long long)k * p.OH * p.OW + ow0 + (pok ? lane : 0), pok ? 4u : 0u);
        mbar_arrive(&full[st]);      // release: this thread's B stores
        cp_async_arrive(&full[st]);  // fires when this thread's dy copies land
        if (++st == kStages) {
          st = 0;
          ph ^= 1;
        }
      }
      if (i + 1 < my_units) {
        // the next row's patch into the other buffer (its copies overlap the
        // MMAs of this row's last stages), then everyone waits for it
        fill_patch(p, u + gridDim.x, p0 + (buf ^ 1) * std::uint32_t(p.p_floats) * 4, pw, lane);
        cp_async_wait_all();
        named_sync(1, kProd * 32);
        buf ^= 1;
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------------ MMA issuer
    const std::uint32_t id1 = idesc_tf32(kBM, p.n1), id2 = idesc_tf32(kBM, p.n2 > 0 ? p.n2 : 16);
    const std::uint32_t sbase = smem_u32(smem);
    for (int g = 0; g < total_steps; ++g) {
      const int st = g % kStages;
      mbar_wait(&full[st], (g / kStages) & 1);
      tc_fence_after();
      if (lane == 0) {
        fence_async_smem();  // generic-proxy writes (STS, cp.async) -> tensor core
        const std::uint32_t sa = sbase + st * stage_bytes, sb = sa + a_bytes;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          mma_tf32(tmem, umma_desc_sw128(sa + j * 32), umma_desc_sw128(sb + j * 32), id1, (g | j) ? 1u : 0u);
          if (p.n2 > 0)
            mma_tf32(tmem + std::uint32_t(p.n1), umma_desc_sw128(sa + j * 32),
                     umma_desc_sw128(sb + std::uint32_t(p.n1) * 128 + j * 32), id2, (g | j) ? 1u : 0u);
        }
        mma_commit(&empty[st]);
        if (g + 1 == total_steps) mma_commit(tfull);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------ epilogue: this CTA's slice
    const int k = warp * 32 + lane;
    float* slice = p.slices + (long long)blockIdx.x * p.rows * p.K;
    if (total_steps > 0) {
      mbar_wait_sleep(tfull, 0);
      tc_fence_after();
    }
    for (int q0 = 0; q0 < p.rows_pad; q0 += 32) {
      float v[32];
      if (total_steps > 0) {
        tmem_ld32(tmem + (std::uint32_t(warp * 32) << 16) + std::uint32_t(q0), v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
      if (k >= p.K) continue;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (q0 + j < p.rows) slice[(long long)(q0 + j) * p.K + k] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// dW[k][q] = beta * dW + alpha * sum_g slice_g[q][k], slices added in order
struct SFinal {
  const float* slices;
  float* dw;
  float alpha, beta;
  int rows, K, nslices;
};
__global__ void __launch_bounds__(256) bfs_finalize_kernel(const SFinal f) {
  pdl_wait();
  const long long n = (long long)f.rows * f.K;
  const long long stride = n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int q = int(i / f.K), k = int(i - (long long)q * f.K);
    float acc = 0.f;
    for (int g = 0; g < f.nslices; ++g) acc += f.slices[g * stride + i];
    float* d = f.dw + (long long)k * f.rows + q;
    *d = f.beta == 0.f ? f.alpha * acc : f.alpha * acc + f.beta * *d;
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

SGeo make_sgeo(const ConvShape& s) {
  SGeo g{};
  g.N = s.N; g.C = s.C; g.H = s.H; g.W = s.W; g.K = s.K; g.R = s.R; g.S = s.S;
  g.ph = s.ph; g.pw = s.pw; g.sh = s.sh; g.sw = s.sw; g.OH = s.OH(); g.OW = s.OW();
  g.rows = s.C * s.R * s.S;
  g.rows_pad = (g.rows + 15) / 16 * 16;
  if (g.rows_pad <= 256) {
    g.n1 = g.rows_pad;
    g.n2 = 0;
  } else {
    g.n1 = (g.rows_pad / 2 + 15) / 16 * 16;
    g.n2 = g.rows_pad - g.n1;
  }
  g.steps = (g.OW + 31) / 32;
  const int need = g.steps * 32 + (s.S - 1) / s.sw;  // largest j read + 1
  const int m = 32 / std::max(1, s.sw);               // JP = 32 / sw (mod 32): conflict-free fill
  g.JP = need;
  while (g.JP % 32 != m % 32) ++g.JP;
  g.units = s.N * g.OH;
  g.grid = std::min(sm_count(), g.units);
  g.p_bytes = std::size_t(s.C) * s.R * s.sw * g.JP * 4;
  g.b_bytes = (std::size_t(g.rows_pad) * 128 + 1023) & ~std::size_t(1023);
  g.stage_bytes = kBM * 128 + g.b_bytes;
  // as many ring stages as fit next to the two patch buffers (2..4)
  g.stages = 2;
  while (g.stages < kMaxStages && (g.stages + 1) * g.stage_bytes + 2 * g.p_bytes + 1024 + 128 <= 220 * 1024)
    ++g.stages;
  g.stages = std::min(g.stages, tune("bfs_stages", kMaxStages));
  g.stages = std::max(g.stages, 2);
  g.smem = g.stages * g.stage_bytes + 2 * g.p_bytes + 1024 + 128;
  return g;
}

}  // namespace

bool bfs_supports(const ConvShape& s) {
  if (s.sh != s.sw || (s.sh != 2 && s.sh != 4) || s.C > 4 || s.K > kBM || !tune("bfs", 1)) return false;
  const SGeo g = make_sgeo(s);
  return g.rows_pad <= kMaxRows && g.smem <= 220 * 1024 && std::int64_t(s.N) * s.C * s.H * s.W < (1ll << 40);
}

std::int64_t bfs_workspace(const ConvShape& s) {
  const SGeo g = make_sgeo(s);
  return (std::int64_t(g.grid) * g.rows * g.K * 4 + 255) / 256 * 256;
}

cudaError_t bfs_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha, float beta,
                    cudaStream_t st) {
  const SGeo g = make_sgeo(s);
  SParams p{};
  p.x = x; p.dy = dy; p.slices = static_cast<float*>(ws);
  p.C = g.C; p.H = g.H; p.W = g.W; p.K = g.K; p.R = g.R; p.S = g.S; p.ph = g.ph; p.pw = g.pw; p.sh = g.sh;
  p.shl = g.sh == 4 ? 2 : 1;
  p.OH = g.OH; p.OW = g.OW;
  p.rows = g.rows; p.rows_pad = g.rows_pad; p.n1 = g.n1; p.n2 = g.n2; p.steps = g.steps; p.JP = g.JP;
  p.units = g.units;
  p.p_floats = int(g.p_bytes / 4);
  p.stages = g.stages;
  p.CHW = std::int64_t(g.C) * g.H * g.W;
  p.KOHW = std::int64_t(g.K) * g.OH * g.OW;
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(bfs_kernel), int(g.smem));
  if (e != cudaSuccess) return e;
  trace_variant("bfs units=%d grid=%d rows=%d n1=%d n2=%d steps=%d JP=%d stages=%d", g.units, g.grid, g.rows, g.n1,
                g.n2, g.steps, g.JP, g.stages);
  e = launch_pdl(bfs_kernel, dim3(g.grid), dim3(kThreads), g.smem, st, p);
  if (e != cudaSuccess) return e;
  SFinal f{p.slices, dw, alpha, beta, g.rows, g.K, g.grid};
  const long long n = (long long)g.rows * g.K;
  return launch_pdl(bfs_finalize_kernel, dim3(int(std::min<long long>((n + 255) / 256, 4 * sm_count()))), dim3(256), 0,
                    st, f);
}

}  // namespace ucudnn
