// UCUDNN_ALGO_IMPLICIT_GEMM: zero-workspace implicit-GEMM convolution on
// tcgen05 tensor cores (kind::tf32, fp32 accumulators in TMEM).
//
// One CTA computes a 128 x BN tile of the conv-as-GEMM (see IgemmParams for
// the per-op GEMM view). Warp roles (288 threads):
//   warps 0-3  gather the A operand (128 rows x 32 reduction elements per
//              chunk) straight from the NCHW tensor -- padding, stride and
//              tails become zeros -- into the no-swizzle K-major UMMA layout,
//              then run the epilogue (TMEM -> registers -> NCHW / atomics);
//   warps 4-7  gather the B operand (BN rows x 32) the same way;
//   warp 8     owns TMEM and issues tcgen05.mma from one elected lane.
// Producers and the MMA issuer meet on a `stages`-deep ring of mbarriers
// (full: 256 producer arrivals; empty: one tcgen05.commit). Nothing is staged
// in global memory, so the algorithm needs no workspace.
//
// Semantics follow the reference convolution loops
// (/root/reference/proj/include/ubatch/reference_conv.hpp:70-171): forward
// gather, BackwardData as the exact adjoint, BackwardFilter accumulating into
// dw (output scale 1, no 1/N).
#include <cuda_runtime.h>

#include "conv_common.h"
#include "igemm.h"
#include "bflsu.h"
#include "fct.h"
#include "fps.h"
#include "z1x1.h"
#include "sm100.cuh"

namespace ucudnn {
using namespace sm100;

namespace {

constexpr int kBM = 128;
constexpr int kChunk = 32;     // reduction elements per pipeline stage
constexpr int kThreads = 288;
constexpr int kTmemCols = 256;

struct ColInfo {
  int off;
  int hw;  // (h << 16) | (w & 0xffff), both signed 16-bit
};
__device__ __forceinline__ int col_h(int hw) { return hw >> 16; }
__device__ __forceinline__ int col_w(int hw) { return int(short(hw & 0xffff)); }
constexpr int kInvalidHW = 0x40000000;  // h = 16384: fails every bounds test

__device__ __forceinline__ void sts128(std::uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// Column table for the row-lane gathers (Fwd / BwdData A operand): one entry
// per reduction index, padded to whole chunks with an always-invalid entry.
template <int OP>
__device__ void build_table(const IgemmParams& p, ColInfo* tab, int n_entries) {
  for (int kg = threadIdx.x; kg < n_entries; kg += blockDim.x) {
    ColInfo ci{0, kInvalidHW};
    if (kg < p.Kg) {
      if (OP == kFwd) {  // kg = (c, r, s): x offset c*H*W + r*W + s
        std::uint32_t c, rs, r, s;
        p.fd_RS.divmod(kg, c, rs);
        p.fd_S.divmod(rs, r, s);
        ci.off = int(c) * p.H * p.W + int(r) * p.W + int(s);
        ci.hw = (int(r) << 16) | int(s);
      } else {  // kg = (k, rr, ss): dy offset k*P - rr*OW - ss
        std::uint32_t k, t, rr, ss;
        p.fd_RaSb.divmod(kg, k, t);
        p.fd_Sb.divmod(t, rr, ss);
        ci.off = int(k) * p.OH * p.OW - int(rr) * p.OW - int(ss);
        ci.hw = (int(-int(rr)) << 16) | (int(-int(ss)) & 0xffff);
      }
    }
    tab[kg] = ci;
  }
}

template <int OP>
__global__ void __launch_bounds__(kThreads, 1) igemm_kernel(const IgemmParams p) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * kBM, n0 = blockIdx.y * p.BN;

  // reduction range of this CTA (split-K along grid.z for BwdFilter)
  const int total_chunks = (p.Kg + kChunk - 1) / kChunk;
  const int c_begin = blockIdx.z * p.chunks_per_split;
  const int c_end = min(total_chunks, c_begin + p.chunks_per_split);
  const int nchunks = max(0, c_end - c_begin);
  const int kg_end = min(p.Kg, c_end * kChunk);

  unsigned char* stage_base = smem;
  ColInfo* table = reinterpret_cast<ColInfo*>(smem + p.stages * p.stage_bytes);
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + p.stages * p.stage_bytes + p.table_bytes);
  std::uint64_t* full = bars;
  std::uint64_t* empty = bars + p.stages;
  std::uint64_t* done = bars + 2 * p.stages;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(done + 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 256);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_fence_init();
  }
  if (OP != kBwdFilter) build_table<OP>(p, table, total_chunks * kChunk);
  if (warp == 8) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = tmem_base_uniform(tmem_slot);

  const std::uint32_t smem0 = smem_u32(stage_base);
  const std::uint32_t a_bytes = 8 * p.lbo_a;

  if (warp == 8) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      const std::uint32_t idesc = idesc_tf32(kBM, p.BN);
      for (int i = 0; i < nchunks; ++i) {
        const int s = i % p.stages;
        mbar_wait(&full[s], (i / p.stages) & 1);
        tc_fence_after();
        const std::uint32_t sa = smem0 + s * p.stage_bytes, sb = sa + a_bytes;
#pragma unroll
        for (int q = 0; q < kChunk / 8; ++q) {
          std::uint64_t ad = umma_desc(sa + 2 * q * p.lbo_a, p.lbo_a, 128);
          std::uint64_t bd = umma_desc(sb + 2 * q * p.lbo_b, p.lbo_b, 128);
          mma_tf32(tmem, ad, bd, idesc, (i | q) != 0);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(done);
    }
    __syncwarp();
  } else if (warp < 4) {
    // ------------------------------------------------ A producers
    const int t = threadIdx.x;  // 0..127
    if (OP != kBwdFilter) {
      // row lanes: thread t owns GEMM row m0 + t for every chunk
      const int m = m0 + t;
      bool row_ok = m < p.M;
      int row_base = 0, row_h = 0, row_w = 0;
      const int lim_h = OP == kFwd ? p.H : p.OH, lim_w = OP == kFwd ? p.W : p.OW;
      if (row_ok) {
        if (OP == kFwd) {
          std::uint32_t n, pix, oh, ow;
          p.fd_P.divmod(m, n, pix);
          p.fd_OW.divmod(pix, oh, ow);
          row_h = int(oh) * p.sh - p.ph;
          row_w = int(ow) * p.sw - p.pw;
          row_base = int(n) * p.C * p.H * p.W + row_h * p.W + row_w;
        } else {
          std::uint32_t n, t2, ih, iw;
          p.fd_HWp.divmod(m, n, t2);
          p.fd_Wp.divmod(t2, ih, iw);
          row_h = p.jh0 + int(ih);
          row_w = p.jw0 + int(iw);
          row_base = int(n) * p.K * p.OH * p.OW + row_h * p.OW + row_w;
        }
      }
      if (!row_ok) row_h = kInvalidHW >> 16;
      const float* src = p.a + row_base;
      for (int i = 0; i < nchunks; ++i) {
        const int s = i % p.stages;
        mbar_wait(&empty[s], ((i / p.stages) & 1) ^ 1);
        const ColInfo* ct = table + (c_begin + i) * kChunk;
        float v[kChunk];
#pragma unroll
        for (int e = 0; e < kChunk; ++e) {
          const ColInfo ci = ct[e];
          const int hh = row_h + col_h(ci.hw), ww = row_w + col_w(ci.hw);
          v[e] = (unsigned(hh) < unsigned(lim_h) && unsigned(ww) < unsigned(lim_w)) ? __ldg(src + ci.off) : 0.f;
        }
        const std::uint32_t sa = smem0 + s * p.stage_bytes + t * 16;
#pragma unroll
        for (int g = 0; g < 8; ++g) sts128(sa + g * p.lbo_a, v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
        fence_async_smem();
        mbar_arrive(&full[s]);
      }
    } else {
      // BwdFilter A = im2col(x): rows (c,r,s), reduction over pixels.
      // k lanes: thread t serves k-group g = t % 8 of rows t/8 + 16j.
      const int g = t & 7;
      int rb[8], rh[8], rw[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int row = m0 + (t >> 3) + 16 * j;
        if (row < p.M) {
          std::uint32_t c, rs, r, s;
          p.fd_RS.divmod(row, c, rs);
          p.fd_S.divmod(rs, r, s);
          rb[j] = int(c) * p.H * p.W + int(r) * p.W + int(s);
          rh[j] = int(r);
          rw[j] = int(s);
        } else {
          rb[j] = 0;
          rh[j] = 1 << 20;
          rw[j] = 0;
        }
      }
      for (int i = 0; i < nchunks; ++i) {
        const int s = i % p.stages;
        mbar_wait(&empty[s], ((i / p.stages) & 1) ^ 1);
        int co[4], ch[4], cw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = (c_begin + i) * kChunk + 4 * g + e;
          if (j < kg_end) {
            std::uint32_t n, pix, oh, ow;
            p.fd_P.divmod(j, n, pix);
            p.fd_OW.divmod(pix, oh, ow);
            ch[e] = int(oh) * p.sh - p.ph;
            cw[e] = int(ow) * p.sw - p.pw;
            co[e] = int(n) * p.C * p.H * p.W + ch[e] * p.W + cw[e];
          } else {
            co[e] = 0;
            ch[e] = 1 << 20;
            cw[e] = 0;
          }
        }
        float v[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int hh = rh[j] + ch[e], ww = rw[j] + cw[e];
            v[j][e] = (unsigned(hh) < unsigned(p.H) && unsigned(ww) < unsigned(p.W)) ? __ldg(p.a + rb[j] + co[e])
                                                                                      : 0.f;
          }
        const std::uint32_t sa = smem0 + s * p.stage_bytes + g * p.lbo_a + (t >> 3) * 16;
#pragma unroll
        for (int j = 0; j < 8; ++j) sts128(sa + j * 256, v[j][0], v[j][1], v[j][2], v[j][3]);
        fence_async_smem();
        mbar_arrive(&full[s]);
      }
    }
  } else {
    // ------------------------------------------------ B producers (k lanes)
    const int t = threadIdx.x - 128;
    const int g = t & 7;
    const int rows_per_thread = p.BN / 16;
    for (int i = 0; i < nchunks; ++i) {
      const int s = i % p.stages;
      mbar_wait(&empty[s], ((i / p.stages) & 1) ^ 1);
      const int kg0 = (c_begin + i) * kChunk + 4 * g;
      const std::uint32_t sb = smem0 + s * p.stage_bytes + a_bytes + g * p.lbo_b + (t >> 3) * 16;
      // per-chunk column offsets of this thread's 4 reduction indices
      int co[4];
      bool cok[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kg = kg0 + e;
        cok[e] = kg < kg_end;
        co[e] = 0;
        if (cok[e]) {
          if (OP == kFwd) {
            co[e] = kg;
          } else if (OP == kBwdData) {
            std::uint32_t k, tt, rr, ss;
            p.fd_RaSb.divmod(kg, k, tt);
            p.fd_Sb.divmod(tt, rr, ss);
            co[e] = int(k) * p.C * p.R * p.S + (p.pa + p.sh * int(rr)) * p.S + p.pb + p.sw * int(ss);
          } else {
            std::uint32_t n, pix;
            p.fd_P.divmod(kg, n, pix);
            co[e] = int(n) * p.K * p.OH * p.OW + int(pix);
          }
        }
      }
      for (int j = 0; j < rows_per_thread; ++j) {
        const int row = n0 + (t >> 3) + 16 * j;
        float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
        if (row < p.Ng) {
          int rbase;
          if (OP == kFwd) rbase = row * p.C * p.R * p.S;
          else if (OP == kBwdData) rbase = row * p.R * p.S;
          else rbase = row * p.OH * p.OW;
          const float* src = p.b + rbase;
          if (cok[0]) v0 = __ldg(src + co[0]);
          if (cok[1]) v1 = __ldg(src + co[1]);
          if (cok[2]) v2 = __ldg(src + co[2]);
          if (cok[3]) v3 = __ldg(src + co[3]);
        }
        sts128(sb + j * 256, v0, v1, v2, v3);
      }
      fence_async_smem();
      mbar_arrive(&full[s]);
    }
  }

  // ------------------------------------------------ epilogue (warps 0-3)
  if (warp < 4) {
    if (nchunks > 0) {
      mbar_wait(done, 0);
      tc_fence_after();
    }
    const int row = m0 + warp * 32 + lane;
    bool row_ok = row < p.M;
    std::int64_t obase = 0;
    std::int64_t cstride = 0;
    if (row_ok) {
      if (OP == kFwd) {
        std::uint32_t n, pix;
        p.fd_P.divmod(row, n, pix);
        cstride = std::int64_t(p.OH) * p.OW;
        obase = std::int64_t(n) * p.K * cstride + pix;
      } else if (OP == kBwdData) {
        std::uint32_t n, t2, ih, iw;
        p.fd_HWp.divmod(row, n, t2);
        p.fd_Wp.divmod(t2, ih, iw);
        const int h = p.pa + p.sh * (p.jh0 + int(ih)) - p.ph;
        const int w = p.pb + p.sw * (p.jw0 + int(iw)) - p.pw;
        cstride = std::int64_t(p.H) * p.W;
        obase = std::int64_t(n) * p.C * cstride + std::int64_t(h) * p.W + w;
      } else {
        cstride = std::int64_t(p.C) * p.R * p.S;  // dw[k, crs]
        obase = row;
      }
    }
    if (OP == kBwdFilter && nchunks == 0) row_ok = false;
    for (int c0 = 0; c0 < p.BN; c0 += 32) {
      float acc[32];
      if (nchunks > 0) {
        tmem_ld32(tmem + (std::uint32_t(warp * 32) << 16) + std::uint32_t(c0), acc);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
      }
      if (!row_ok) continue;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int col = n0 + c0 + j;
        if (c0 + j >= p.BN || col >= p.Ng) break;
        float* dst = p.out + obase + std::int64_t(col) * cstride;
        const float val = p.alpha * acc[j];
        if (OP == kBwdFilter) {
          red_add(dst, val);
        } else {
          *dst = p.beta == 0.f ? val : val + p.beta * *dst;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_free<kTmemCols>(tmem);
  }
}

__global__ void scale_kernel(float* p, std::int64_t n, float beta) {
  std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x;
  for (; i < n; i += std::int64_t(gridDim.x) * blockDim.x) p[i] = beta == 0.f ? 0.f : p[i] * beta;
}

int num_sms() {
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
}

int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Column tile: <= 256, multiple of 16, balanced over the needed tiles.
int pick_bn(int ng) {
  int tiles = (ng + 255) / 256;
  return round_up((ng + tiles - 1) / tiles, 16);
}

cudaError_t launch(int op, IgemmParams p, int grid_x, int grid_y, int grid_z, cudaStream_t stream) {
  p.lbo_a = kBM * 16 + 16;
  p.lbo_b = p.BN * 16 + 16;
  p.stage_bytes = round_up(8 * (p.lbo_a + p.lbo_b), 128);
  const int total_chunks = (p.Kg + kChunk - 1) / kChunk;
  p.table_bytes = op == kBwdFilter ? 0 : round_up(total_chunks * kChunk * int(sizeof(ColInfo)), 128);
  const int fixed = int(p.table_bytes) + 64 * 8 + 64;
  const int budget = 227 * 1024;
  int stages = (budget - fixed) / int(p.stage_bytes);
  stages = stages > 4 ? 4 : stages;
  if (stages < 2) return cudaErrorInvalidConfiguration;
  p.stages = stages;
  const int smem = int(p.stage_bytes) * stages + fixed;
  void (*kern)(IgemmParams) = op == kFwd ? igemm_kernel<kFwd> : op == kBwdData ? igemm_kernel<kBwdData>
                                                                                : igemm_kernel<kBwdFilter>;
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), 227 * 1024);
  if (e != cudaSuccess) return e;
  count_launch();
  kern<<<dim3(grid_x, grid_y, grid_z), kThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

void fill_common(IgemmParams& p, const ConvShape& s) {
  p.N = s.N; p.C = s.C; p.H = s.H; p.W = s.W; p.K = s.K; p.R = s.R; p.S = s.S;
  p.ph = s.ph; p.pw = s.pw; p.sh = s.sh; p.sw = s.sw; p.OH = s.OH(); p.OW = s.OW();
  p.fd_P = FastDiv(std::uint32_t(p.OH * p.OW));
  p.fd_OW = FastDiv(std::uint32_t(p.OW));
  p.fd_RS = FastDiv(std::uint32_t(s.R * s.S));
  p.fd_S = FastDiv(std::uint32_t(s.S));
}

}  // namespace

cudaError_t igemm_forward(const ConvShape& s, const float* x, const float* w, float* y, float alpha, float beta,
                          cudaStream_t stream) {
  // 1x1 stride-1 layers: TMA straight from the NCHW planes
  if (tune("z", 1) && z1x1_supports(kFwd, s)) return z1x1_run(kFwd, s, x, w, y, alpha, beta, stream);
  // few-channel strided layers (AlexNet / ResNet conv1): the shared-memory patch kernel
  if (tune("z", 1) && fct_fwd_supports(s)) return fct_fwd_run(s, x, w, y, alpha, beta, stream);
  if (tune("z", 1) && fct1_supports(kFwd, s)) return fct1_run(kFwd, s, x, w, y, nullptr, alpha, beta, stream, 0);
  if (tune("z", 1) && fps_supports(s)) return fps_run(s, x, w, y, alpha, beta, stream);
  if (tune("z", 1) && zgemm_supports(kFwd, s)) return zgemm_forward(s, x, w, y, alpha, beta, stream);
  IgemmParams p{};
  fill_common(p, s);
  p.a = x; p.b = w; p.out = y; p.alpha = alpha; p.beta = beta;
  p.M = s.N * p.OH * p.OW;
  p.Ng = s.K;
  p.Kg = s.C * s.R * s.S;
  p.BN = pick_bn(p.Ng);
  p.chunks_per_split = (p.Kg + kChunk - 1) / kChunk;
  return launch(kFwd, p, (p.M + kBM - 1) / kBM, (p.Ng + p.BN - 1) / p.BN, 1, stream);
}

// Stride phases: for input row h, t = h + ph, phase pa = t mod sh, and only
// taps r = pa + sh*rr reach it, from output row t/sh - rr. Each phase is an
// independent dense GEMM (no multiplications by structural zeros).
cudaError_t igemm_backward_data(const ConvShape& s, const float* dy, const float* w, float* dx, float alpha,
                                float beta, cudaStream_t stream) {
  if (tune("z", 1) && z1x1_supports(kBwdData, s)) return z1x1_run(kBwdData, s, dy, w, dx, alpha, beta, stream);
  if (tune("z", 1) && fct_bwdd_supports(s)) return fct_bwdd_run(s, dy, w, dx, alpha, beta, stream);
  if (tune("z", 1) && zgemm_supports(kBwdData, s)) return zgemm_backward_data(s, dy, w, dx, alpha, beta, stream);
  for (int pa = 0; pa < s.sh; ++pa)
    for (int pb = 0; pb < s.sw; ++pb) {
      IgemmParams p{};
      fill_common(p, s);
      p.a = dy; p.b = w; p.out = dx; p.alpha = alpha; p.beta = beta;
      p.pa = pa; p.pb = pb;
      p.Ra = pa < s.R ? (s.R - pa + s.sh - 1) / s.sh : 0;
      p.Sb = pb < s.S ? (s.S - pb + s.sw - 1) / s.sw : 0;
      // input rows of this phase: h = pa + sh*j - ph in [0, H)
      p.jh0 = (s.ph - pa + s.sh - 1) >= 0 ? (s.ph - pa + s.sh - 1) / s.sh : 0;
      int jh1 = (s.H - 1 + s.ph - pa) >= 0 ? (s.H - 1 + s.ph - pa) / s.sh + 1 : 0;
      p.jw0 = (s.pw - pb + s.sw - 1) >= 0 ? (s.pw - pb + s.sw - 1) / s.sw : 0;
      int jw1 = (s.W - 1 + s.pw - pb) >= 0 ? (s.W - 1 + s.pw - pb) / s.sw + 1 : 0;
      p.Hp = jh1 - p.jh0;
      p.Wp = jw1 - p.jw0;
      if (p.Hp <= 0 || p.Wp <= 0) continue;
      p.fd_HWp = FastDiv(std::uint32_t(p.Hp * p.Wp));
      p.fd_Wp = FastDiv(std::uint32_t(p.Wp));
      p.fd_RaSb = FastDiv(std::uint32_t(p.Ra > 0 && p.Sb > 0 ? p.Ra * p.Sb : 1));
      p.fd_Sb = FastDiv(std::uint32_t(p.Sb > 0 ? p.Sb : 1));
      p.M = s.N * p.Hp * p.Wp;
      p.Ng = s.C;
      p.Kg = s.K * p.Ra * p.Sb;
      p.BN = pick_bn(p.Ng);
      p.chunks_per_split = (p.Kg + kChunk - 1) / kChunk;
      if (p.chunks_per_split == 0) p.chunks_per_split = 1;
      cudaError_t e = launch(kBwdData, p, (p.M + kBM - 1) / kBM, (p.Ng + p.BN - 1) / p.BN, 1, stream);
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}

cudaError_t scale_tensor(float* p, std::int64_t n, float beta, cudaStream_t stream) {
  if (beta == 1.f || n == 0) return cudaSuccess;
  int blocks = int(std::min<std::int64_t>((n + 255) / 256, 4 * num_sms()));
  count_launch();
  scale_kernel<<<blocks, 256, 0, stream>>>(p, n, beta);
  return cudaGetLastError();
}

cudaError_t igemm_backward_filter(const ConvShape& s, const float* x, const float* dy, float* dw, float alpha,
                                  float beta, cudaStream_t stream) {
  // the gather BackwardFilter (bflsu.cu) with its REDs aimed straight at dW:
  // no scratch, so still zero workspace
  if (tune("z", 1) && bfl_supports(s)) return bfl_run(s, x, dy, dw, nullptr, alpha, beta, stream, true);
  cudaError_t e = scale_tensor(dw, s.w_elems(), beta, stream);
  if (e != cudaSuccess) return e;
  IgemmParams p{};
  fill_common(p, s);
  p.a = x; p.b = dy; p.out = dw; p.alpha = alpha; p.beta = 1.f;
  p.M = s.C * s.R * s.S;
  p.Ng = s.K;
  p.Kg = s.N * p.OH * p.OW;
  p.BN = pick_bn(p.Ng);
  const int tiles = ((p.M + kBM - 1) / kBM) * ((p.Ng + p.BN - 1) / p.BN);
  const int chunks = (p.Kg + kChunk - 1) / kChunk;
  // split the pixel reduction so the grid covers ~2 waves, >= 8 chunks each
  int splits = deterministic() ? 1 : std::max(1, std::min(chunks / 8, (2 * num_sms() + tiles - 1) / tiles));
  p.chunks_per_split = (chunks + splits - 1) / splits;
  splits = (chunks + p.chunks_per_split - 1) / p.chunks_per_split;
  return launch(kBwdFilter, p, (p.M + kBM - 1) / kBM, (p.Ng + p.BN - 1) / p.BN, splits, stream);
}

}  // namespace ucudnn
