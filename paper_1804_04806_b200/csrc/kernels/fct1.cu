// Stride-1 implicit GEMM with the im2col operand built in tensor memory, for
// the narrow-output layers the TMA im2col kernels are L2-bound on (AlexNet
// conv2 BackwardData: N = 64 output channels, a 16 KB im2col box re-read from
// L2 per four 128 x 64 x 8 MMAs, DESIGN finding 23). Opt-in: it trades the L2
// traffic for tensor-memory traffic and loses (finding 24).
//
//   out[n][o][oh][ow] = alpha * sum_{c,r,s} in[n][c][oh+r-ph][ow+s-pw] * B[o][(c, r, s)] + beta * out
//
// Forward: in = x, B = w viewed [K][C*R*S] (no workspace). BackwardData:
// in = dy, o = input channel, ph' = R-1-ph, B[c][(k, r, s)] = w[k][c][R-1-r]
// [S-1-s] packed once into the workspace (reference_conv.hpp:70-138).
//
// A tile is msub sub-tiles of TRo whole output rows (<= 128 pixels each, one
// per TMEM lane). The reduction runs over channel chunks of CC = 32: loader
// warps copy the chunk's PH = msub*TRo + R - 1 input rows into a double-
// buffered shared-memory ring (coalesced loads, zero off the image), and each
// producer thread -- one pixel = one TMEM lane -- reads its taps for 32
// reduction columns at a time (lanes are consecutive pixels: conflict-free;
// the (c, r, s) -> ring-offset map is a table) and stores them with one
// tcgen05.st; the filter streams through a TMA ring of 32-column K-major
// SWIZZLE_128B chunks, each feeding the MMAs of all msub sub-tiles. Every
// input element is read from L2 once per tile (PH / (msub*TRo) ~1.5x), not
// once per filter tap.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "conv_common.h"
#include "fct.h"
#include "launch.h"
#include "sm100.cuh"

namespace ucudnn {
using namespace sm100;

namespace {

constexpr int kBM = 128;
constexpr int kMaxSlots = 8;
constexpr int kMaxB = 8;
constexpr int kCC = 32;  // input channels per ring fill
constexpr int kMaxTab = kCC * 64;
// warps: 0-7 A producers (sub-tile m = warp / 4, lane quarter warp % 4),
// 8 MMA issuer, 9 filter TMA, 10-13 row loaders, 14-17 epilogue
constexpr int kThreads1 = 18 * 32;

struct P1 {
  const float* in;
  float* out;
  float alpha, beta;
  int Cin, Hi, Wi, Nout, R, S, ph, pw, Ho, Wo;
  int TRo, np, msub, tiles_per_img, units;
  int nchunks, PH, XW, spc;  // channel chunks, ring rows, ring cols, 32-column slots per chunk
  int BN, nslots, nbst, nacc;
  long long in_img, out_img;
};

__device__ __forceinline__ void mbar_wait_sleep1(std::uint64_t* bar, std::uint32_t parity) {
  std::uint32_t ok = 0, ns = 32;
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
    if (ns < 256) ns <<= 1;
  }
}
__device__ __forceinline__ void tmem_st32b(std::uint32_t taddr, const float (&v)[32]) {
  const std::uint32_t* r = reinterpret_cast<const std::uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_ts_w(std::uint32_t d_tmem, std::uint32_t a_tmem, std::uint64_t bdesc,
                                         std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tma_2d_u32(std::uint32_t dst, const void* tmap, std::uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

__global__ void __launch_bounds__(kThreads1, 1) fct1_kernel(const __grid_constant__ CUtensorMap bmap, const P1 p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t bst_bytes = std::uint32_t(p.BN) * 128;
  unsigned char* bring = smem;                                          // [nbst][BN x 128 B]
  float* ring = reinterpret_cast<float*>(bring + p.nbst * bst_bytes);  // [2][kCC][PH][XW]
  const int ring_floats = kCC * p.PH * p.XW;
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(ring + 2 * ring_floats);
  std::uint64_t* afull = bars;
  std::uint64_t* aempty = afull + kMaxSlots;
  std::uint64_t* bfull = aempty + kMaxSlots;
  std::uint64_t* bempty = bfull + kMaxB;
  std::uint64_t* rfull = bempty + kMaxB;
  std::uint64_t* rempty = rfull + 2;
  std::uint64_t* tfull = rempty + 2;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  __shared__ __align__(16) int tab[kMaxTab];  // chunk-local reduction column (c, r, s) -> ring offset
  const int red = kCC * p.R * p.S;
  for (int q = threadIdx.x; q < red; q += blockDim.x) {
    const int RS = p.R * p.S, c = q / RS, rs = q - c * RS, r = rs / p.S, s = rs - r * p.S;
    tab[q] = (c * p.PH + r) * p.XW + s;
  }
  if (threadIdx.x == 0) {
    prefetch_tmap(&bmap);
    for (int s = 0; s < kMaxSlots; ++s) {
      mbar_init(&afull[s], p.msub * 128);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < kMaxB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&rfull[b], 4 * 32);
      mbar_init(&rempty[b], p.msub * 128);
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    mbar_fence_init();
  }
  if (warp == 8) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  const std::uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const int t0 = int((long long)blockIdx.x * p.units / gridDim.x);
  const int my_units = int((long long)(blockIdx.x + 1) * p.units / gridDim.x) - t0;
  const std::uint32_t a_col0 = std::uint32_t(p.nacc * p.msub * p.BN);
  const int tile_rows = p.msub * p.TRo;

  if (warp < 4 * p.msub) {
    // ------------------------------------------------ A producers: one output pixel per thread
    const int m = warp >> 2, quarter = warp & 3;
    const int px = quarter * 32 + lane;
    const int pe = px < p.np ? px : 0;
    const int rl = pe / p.Wo, ow = pe - rl * p.Wo;
    const std::uint32_t lane_off = std::uint32_t(((m * p.TRo + rl) * p.XW + ow) * 4);
    const std::uint32_t tlane = tmem + (std::uint32_t(quarter * 32) << 16) + a_col0 + std::uint32_t(m * 32);
    int g = 0, f = 0;
    RingPos rs;
    for (int i = 0; i < my_units; ++i) {
      for (int cc = 0; cc < p.nchunks; ++cc, ++f) {
        const int rb = f & 1;
        mbar_wait(&rfull[rb], (f >> 1) & 1);
        const std::uint32_t base = smem_u32(ring) + std::uint32_t(rb * ring_floats * 4) + lane_off;
        for (int sl = 0; sl < p.spc; ++sl, ++g, rs.step(p.nslots)) {
          const int slot = rs.slot;
          mbar_wait(&aempty[slot], rs.ph ^ 1);
          tc_fence_after();
          float v[32];
          const int4* tq = reinterpret_cast<const int4*>(tab + sl * 32);
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const int4 o = tq[j4];
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[4 * j4 + 0]) : "r"(base + std::uint32_t(o.x) * 4));
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[4 * j4 + 1]) : "r"(base + std::uint32_t(o.y) * 4));
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[4 * j4 + 2]) : "r"(base + std::uint32_t(o.z) * 4));
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[4 * j4 + 3]) : "r"(base + std::uint32_t(o.w) * 4));
          }
          tmem_st32b(tlane + std::uint32_t(slot * p.msub * 32), v);
          tc_fence_before();
          mbar_arrive(&afull[slot]);
        }
        mbar_arrive(&rempty[rb]);
      }
    }
  } else if (warp == 8) {
    // ------------------------------------------------ MMA issuer (whole warp, one elected lane)
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN);
    const std::uint64_t bd0 = umma_desc_sw128(smem_u32(bring));
    const std::uint32_t bst_desc = bst_bytes >> 4;
    int g = 0;
    RingPos rs, rb;
    for (int i = 0; i < my_units; ++i) {
      const int acc = p.nacc == 2 ? (i & 1) : 0;
      const int use = p.nacc == 2 ? (i >> 1) : i;
      mbar_wait(&tempty[acc], (use & 1) ^ 1);
      tc_fence_after();
      const std::uint32_t d = tmem + std::uint32_t(acc * p.msub * p.BN);
      const int nsl = p.nchunks * p.spc;
      for (int k0 = 0; k0 < nsl; ++k0, ++g, rs.step(p.nslots), rb.step(p.nbst)) {
        const int slot = rs.slot, bs = rb.slot;
        mbar_wait(&afull[slot], rs.ph);
        mbar_wait(&bfull[bs], rb.ph);
        tc_fence_after();
        const std::uint32_t ta = tmem + a_col0 + std::uint32_t(slot * p.msub * 32);
        const std::uint64_t bd = bd0 + std::uint64_t(bs) * bst_desc;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          for (int m = 0; m < p.msub; ++m)
            mma_ts_w(d + std::uint32_t(m * p.BN), ta + std::uint32_t(m * 32 + 8 * k), bd + 2 * k, idesc,
                     (k0 | k) ? 1u : 0u);
        mma_commit_w(&aempty[slot]);
        mma_commit_w(&bempty[bs]);
        if (k0 + 1 == nsl) mma_commit_w(&tfull[acc]);
        __syncwarp();
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------ filter chunks by TMA (32 reduction columns x BN rows)
    if (lane == 0) {
      int g = 0;
      for (int i = 0; i < my_units; ++i)
        for (int cc = 0; cc < p.nchunks; ++cc)
          for (int sl = 0; sl < p.spc; ++sl, ++g) {
            const int bs = g % p.nbst;
            mbar_wait_sleep1(&bempty[bs], ((g / p.nbst) & 1) ^ 1);
            mbar_expect_tx(&bfull[bs], bst_bytes);
            tma_2d_u32(smem_u32(bring) + std::uint32_t(bs) * bst_bytes, &bmap, &bfull[bs],
                       cc * kCC * p.R * p.S + sl * 32, 0);
          }
    }
    __syncwarp();
  } else if (warp >= 10 && warp < 14) {
    // ------------------------------------------------ row loaders: a chunk's PH input rows of kCC channels
    const int lw = warp - 10;
    int f = 0;
    for (int i = 0; i < my_units; ++i) {
      const int u = t0 + i;
      const int n = u / p.tiles_per_img, oh0 = (u - n * p.tiles_per_img) * tile_rows;
      const float* inn = p.in + (long long)n * p.in_img;
      for (int cc = 0; cc < p.nchunks; ++cc, ++f) {
        const int rb = f & 1;
        mbar_wait_sleep1(&rempty[rb], ((f >> 1) & 1) ^ 1);
        float* dst0 = ring + rb * ring_floats;
        const int nrows = kCC * p.PH;
        constexpr int kB = 8;  // rows per batch
        for (int r0 = lw; r0 < nrows; r0 += 4 * kB) {
          float v[kB][2];
#pragma unroll
          for (int b = 0; b < kB; ++b) {
            const int row = r0 + 4 * b;
            const int cl = row / p.PH, t = row - cl * p.PH;
            const int c = cc * kCC + cl, ih = oh0 + t - p.ph;
            const bool rok = row < nrows && c < p.Cin && unsigned(ih) < unsigned(p.Hi);
            const float* src = inn + ((long long)(rok ? c : 0) * p.Hi + (rok ? ih : 0)) * p.Wi;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int col = lane + 32 * h, iw = col - p.pw;
              v[b][h] = rok && col < p.XW && unsigned(iw) < unsigned(p.Wi) ? __ldg(src + iw) : 0.f;
            }
          }
#pragma unroll
          for (int b = 0; b < kB; ++b) {
            const int row = r0 + 4 * b;
            if (row >= nrows) break;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int col = lane + 32 * h;
              if (col < p.XW) dst0[row * p.XW + col] = v[b][h];
            }
          }
        }
        mbar_arrive(&rfull[rb]);  // release: this thread's ring stores
      }
    }
  } else if (warp >= 14) {
    // ------------------------------------------------ epilogue (NCHW stores, lane = pixel)
    const int quarter = warp & 3;
    const int px = quarter * 32 + lane;
    const int rl = px / p.Wo, ow = px - rl * p.Wo;
    const long long HoWo = (long long)p.Ho * p.Wo;
    for (int i = 0; i < my_units; ++i) {
      const int u = t0 + i;
      const int n = u / p.tiles_per_img, oh0 = (u - n * p.tiles_per_img) * tile_rows;
      const int acc = p.nacc == 2 ? (i & 1) : 0;
      const int use = p.nacc == 2 ? (i >> 1) : i;
      mbar_wait_sleep1(&tfull[acc], use & 1);
      tc_fence_after();
      for (int m = 0; m < p.msub; ++m) {
        const int oh = oh0 + m * p.TRo + rl;
        const bool live = px < p.np && oh < p.Ho;
        float* ob = p.out + (long long)n * p.out_img + (long long)oh * p.Wo + ow;
        for (int c0 = 0; c0 < p.BN; c0 += 32) {
          float v[32];
          tmem_ld32(tmem + (std::uint32_t(quarter * 32) << 16) + std::uint32_t((acc * p.msub + m) * p.BN + c0), v);
          if (!live) continue;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (c0 + j >= p.Nout) break;
            float* dst = ob + (long long)(c0 + j) * HoWo;
            const float val = p.alpha * v[j];
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
  if (warp == 8) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// BackwardData's filter: B[c][(k, r, s)] = w[k][c][R-1-r][S-1-s]
__global__ void fct1_pack_bd_kernel(const float* __restrict__ w, float* __restrict__ b, int K, int C, int R, int S) {
  const long long n = (long long)K * C * R * S;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int RS = R * S;
    const long long c = i / ((long long)K * RS);
    const long long rem = i - c * K * RS;
    const int k = int(rem / RS), rs = int(rem - (long long)k * RS), r = rs / S, s = rs - r * S;
    b[i] = w[(((long long)k * C + c) * R + (R - 1 - r)) * S + (S - 1 - s)];
  }
}

int sm_count1() {
  static int v = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return v;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled1() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// the stride-1 problem of op 0 / 1 in input -> output terms
struct G1 {
  bool ok = false;
  int Cin, Hi, Wi, Nout, ph, pw, Ho, Wo, kred;
  int TRo, np, msub, tiles_per_img, units, grid;
  int nchunks, PH, XW, spc, BN, nslots, nbst, nacc;
  std::size_t smem;
};

G1 make_g1(int op, const ConvShape& s) {
  G1 g;
  if (s.sh != 1 || s.sw != 1) return g;
  if (op == 0) {
    g.Cin = s.C; g.Hi = s.H; g.Wi = s.W; g.Nout = s.K; g.ph = s.ph; g.pw = s.pw; g.Ho = s.OH(); g.Wo = s.OW();
  } else {
    g.Cin = s.K; g.Hi = s.OH(); g.Wi = s.OW(); g.Nout = s.C; g.ph = s.R - 1 - s.ph; g.pw = s.S - 1 - s.pw;
    g.Ho = s.H; g.Wo = s.W;
    if (g.ph < 0 || g.pw < 0 || g.Hi + 2 * g.ph - s.R + 1 != g.Ho || g.Wi + 2 * g.pw - s.S + 1 != g.Wo) return g;
  }
  g.kred = g.Cin * s.R * s.S;
  if (g.Wo > kBM || g.Cin % kCC != 0 || (g.kred % 4) != 0 || kCC * s.R * s.S > kMaxTab) return g;
  g.BN = (g.Nout + 15) / 16 * 16;
  if (g.BN > 256) return g;
  g.TRo = kBM / g.Wo;
  g.np = g.TRo * g.Wo;
  g.msub = std::max(1, std::min(2, tune("fct1_msub", 2)));
  g.tiles_per_img = (g.Ho + g.msub * g.TRo - 1) / (g.msub * g.TRo);
  g.units = s.N * g.tiles_per_img;
  g.grid = std::min(sm_count1(), g.units);
  g.nchunks = g.Cin / kCC;
  g.PH = g.msub * g.TRo + s.R - 1;
  g.XW = std::max(32, (g.Wo + s.S - 1 + 31) / 32 * 32);
  if (g.XW > 64) return g;
  g.spc = kCC * s.R * s.S / 32;
  g.nacc = 2 * g.msub * g.BN + 2 * g.msub * 32 <= 512 ? 2 : 1;
  g.nslots = std::min(kMaxSlots, (512 - g.nacc * g.msub * g.BN) / (g.msub * 32));
  const std::size_t ring = std::size_t(2) * kCC * g.PH * g.XW * 4;
  const std::size_t fixed = ring + 1024 + 512;
  const std::size_t bst = std::size_t(g.BN) * 128;
  // (the tap table takes 8 KB of static shared memory next to this)
  g.nbst = int(std::min<std::size_t>(kMaxB, (212 * 1024 - std::min<std::size_t>(fixed, 212 * 1024)) / bst));
  g.smem = fixed + g.nbst * bst;
  // opt-in (UCUDNN_TUNE=fct1=1): exact, but measured 1.8-2.4x slower than the
  // TMA im2col kernel on AlexNet conv2 / ResNet 3x3 -- MMAs reading a 128 x 8
  // A slice from TMEM next to the producers' tcgen05.st traffic ran at ~160
  // cycles each (DESIGN finding 24)
  g.ok = g.nslots >= 2 && g.nbst >= 3 && tune("fct1", 0) == 1;
  return g;
}

}  // namespace

bool fct1_supports(int op, const ConvShape& s) {
  if (op != 0 && op != 1) return false;
  return make_g1(op, s).ok;
}

std::int64_t fct1_workspace(int op, const ConvShape& s) {
  return op == 1 ? (s.w_elems() * 4 + 255) / 256 * 256 : 0;
}

cudaError_t fct1_run(int op, const ConvShape& s, const float* in, const float* w, float* out, void* ws, float alpha,
                     float beta, cudaStream_t st, int flags) {
  const G1 g = make_g1(op, s);
  if (!g.ok) return cudaErrorInvalidValue;
  const float* bmat = w;
  if (op == 1) {
    float* b = static_cast<float*>(ws);
    if (!(flags & kFilterReady)) {
      count_launch();
      fct1_pack_bd_kernel<<<int(std::min<std::int64_t>((s.w_elems() + 255) / 256, 4 * sm_count1())), 256, 0, st>>>(
          w, b, s.K, s.C, s.R, s.S);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    bmat = b;
  }
  CUtensorMap bmap;
  const cuuint64_t dims[2] = {cuuint64_t(g.kred), cuuint64_t(g.Nout)};
  const cuuint64_t strides[1] = {cuuint64_t(g.kred) * 4};
  const cuuint32_t box[2] = {32, cuuint32_t(g.BN)};
  const cuuint32_t es[2] = {1, 1};
  if (encode_tiled1()(&bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(bmat), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  P1 p{};
  p.in = in; p.out = out; p.alpha = alpha; p.beta = beta;
  p.Cin = g.Cin; p.Hi = g.Hi; p.Wi = g.Wi; p.Nout = g.Nout; p.R = s.R; p.S = s.S; p.ph = g.ph; p.pw = g.pw;
  p.Ho = g.Ho; p.Wo = g.Wo;
  p.TRo = g.TRo; p.np = g.np; p.msub = g.msub; p.tiles_per_img = g.tiles_per_img; p.units = g.units;
  p.nchunks = g.nchunks; p.PH = g.PH; p.XW = g.XW; p.spc = g.spc;
  p.BN = g.BN; p.nslots = g.nslots; p.nbst = g.nbst; p.nacc = g.nacc;
  p.in_img = std::int64_t(g.Cin) * g.Hi * g.Wi;
  p.out_img = std::int64_t(g.Nout) * g.Ho * g.Wo;
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(fct1_kernel), int(g.smem));
  if (e != cudaSuccess) return e;
  trace_variant("fct1 op=%d units=%d grid=%d TRo=%d np=%d msub=%d chunks=%d PH=%d XW=%d BN=%d slots=%d bst=%d acc=%d",
                op, g.units, g.grid, g.TRo, g.np, g.msub, g.nchunks, g.PH, g.XW, g.BN, g.nslots, g.nbst, g.nacc);
  return launch_pdl(fct1_kernel, dim3(g.grid), dim3(kThreads1), g.smem, st, bmap, p);
}

}  // namespace ucudnn
