// UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM, BackwardFilter, load-store-unit-fed
// variant: the tcgen05 GEMM reads x and dy straight from their NCHW tensors.
//
//   dW[k][c][r][s] += alpha * sum_{n,oh,ow} dy[n][k][oh][ow] * x[n][c][oh*sh-ph+r][ow*sw-pw+s]
//   (reference_conv.hpp:141-171; beta applied once, :173-180)
//
// Why not TMA here (bfilter.cu): the reduction axis -- output pixels -- has
// to be K-major in shared memory, and a tap (r, s) shifts it by a non-16-byte
// multiple, which TMA cannot start at. bfilter.cu pays for that with
// re-laid-out, 4x-replicated copies of x in the workspace (AlexNet conv1: 687
// MB for 256 images), so under a 64 MiB limit the planner has to cut the
// batch into 16-image micro-batches and pay each call's ramp and
// re-layout again. Here producer warps gather the operands themselves with
// 4-byte cp.async (any alignment, zero fill through the ignore-src
// predicate), lane = pixel, so:
//   * no re-layout pass and no workspace beyond the small GEMM-layout RED
//     scratch -- every batch size fits, one call covers the whole batch;
//   * strides and padding are handled in the gather (per-lane bounds), GEMM
//     rows are exactly the C*R*S filter taps (no phase padding);
//   * 32-pixel reduction chunks run across image boundaries (the flat
//     pixel index n*OH*OW + p), so 13x13 layers waste no MMA K-steps.
// The store pattern is the SWIZZLE_128B K-major UMMA layout: row q at
// q*128 B, 16-byte chunk (lane/4) ^ (q%8).
//
// GEMM rows of x are ordered (r, s, c) so that 8-row groups share one tap
// (C % 8 == 0; fewer channels use a per-row (offset, tap) table):
// the bounds test and base offset are computed once per tap run, and each
// row is one cp.async plus a pointer step. Roles as in bfilter.cu: K <= 128
// output channels -> MMA rows = k (one 128-row tile of dy), columns = x rows.
//
// Persistent, one CTA per SM: warps 0-3 epilogue (TMEM -> fp32 RED into
// the scratch), warp 4 TMEM owner + MMA issuer, warps 5.. producers (12 in
// the 1-SM kernel, 16 in the CTA-pair kernel bfl2_kernel, K > 128). A producer never waits for its own gathers: each thread's
// cp.async.mbarrier.arrive fires when its copies land, and the MMA thread
// issues the generic->async proxy fence after observing the full barrier.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "bflsu.h"
#include "conv_common.h"
#include "igemm.h"
#include "launch.h"
#include "sm100.cuh"

namespace ucudnn {
using namespace sm100;

namespace {

constexpr int kBM = 128;
constexpr int kMaxBN = 256;
constexpr int kMaxStages = 8;
// producer warps: the gathers are latency-bound, more warps keep more rows
// in flight; measured best 12 for the 1-SM kernel (AlexNet conv1 BF 542 us
// vs 615 with 16) and 16 for the CTA pairs (conv2-5 4-7 % faster than 12)
constexpr int kProd1 = 12, kProd2 = 16;
template <int NP>
constexpr int threads_for() { return (5 + NP) * 32; }

struct LGeo {
  int N, C, H, W, K, R, S, ph, pw, sh, sw, OH, OW;
  int M;  // C*R*S GEMM rows of x
  int swap, BN, m_tiles, n_tiles;
  int two;        // CTA pairs (cta_group::2): m_tiles counts 256-row pair tiles
  int dual;       // pairs with two pair tiles per unit: m_tiles counts 512-row tiles
  long long npx;  // N*OH*OW
  int steps;      // 32-pixel chunks
};

int round_up(int a, int b) { return (a + b - 1) / b * b; }

LGeo make_lgeo(const ConvShape& s) {
  LGeo g{};
  g.N = s.N; g.C = s.C; g.H = s.H; g.W = s.W; g.K = s.K; g.R = s.R; g.S = s.S;
  g.ph = s.ph; g.pw = s.pw; g.sh = s.sh; g.sw = s.sw; g.OH = s.OH(); g.OW = s.OW();
  g.M = s.C * s.R * s.S;
  g.npx = std::int64_t(s.N) * g.OH * g.OW;
  g.steps = int((g.npx + 31) / 32);
  g.swap = s.K <= 128 && g.M > 128;
  if (g.swap) {
    int nt = (g.M + kMaxBN - 1) / kMaxBN;
    // few channels: the x rows may land MN-major (whole 32-row blocks)
    g.BN = round_up((g.M + nt - 1) / nt, s.C % 8 != 0 ? 32 : 16);
    g.n_tiles = (g.M + g.BN - 1) / g.BN;
    g.m_tiles = 1;
  } else {
    const int nt = (s.K + kMaxBN - 1) / kMaxBN;
    g.BN = round_up((s.K + nt - 1) / nt, 16);
    g.n_tiles = (s.K + g.BN - 1) / g.BN;
    g.m_tiles = (g.M + kBM - 1) / kBM;
    // pairs: each CTA gathers its own 128 x rows and half of the dy rows
    g.two = tune("bfl2", 1) && g.m_tiles >= 2;
    // one dy gather for 512 x rows (TMEM: 2 x BN <= 512 columns, C % 8 == 0 path)
    g.dual = g.two && s.C % 8 == 0 && g.m_tiles >= 4 && tune("bfl_dual", 1);
    if (g.two) g.m_tiles = (g.M + (g.dual ? 4 : 2) * kBM - 1) / ((g.dual ? 4 : 2) * kBM);
  }
  return g;
}

// RED scratch in the GEMM's own layout: non-swap [k][x row] (pitch rows_pad),
// swap [x row][k] (pitch 128); 32 lanes reduce into 32 consecutive floats.
int rows_pad(const LGeo& g) { return g.swap ? g.n_tiles * g.BN : g.m_tiles * kBM * (g.dual ? 4 : g.two ? 2 : 1); }
int cols_pad(const LGeo& g) { return g.swap ? kBM : g.n_tiles * g.BN; }
std::size_t scratch_bytes(const LGeo& g) { return (std::size_t(rows_pad(g)) * cols_pad(g) * 4 + 255) / 256 * 256; }

struct LParams {
  const float* x;
  const float* dy;
  float* acc;
  int C, H, W, K, R, S, sh, sw, ph, pw, OW, OHW, HW, M;
  long long npx, CHW, KOHW;
  int swap, BN, m_tiles, tiles, splits, steps, steps_per_unit, stages, rpad;
  int dbg;  // diagnostic (UCUDNN_TUNE=bfl_dbg): 1 skip the gathers, 2 skip the MMAs
  FastDiv fd_ohw, fd_ow, fd_C, fd_S, fd_RS, fd_sgs;
  int crs;  // x row order: 1 (c, r, s) = dW order, 0 (r, s, c)
  int sg, ngroups, sgs;
  int dual;  // CTA-pair kernel: two pair tiles per unit  // strided few-channel gather: groups of sw taps, count, ceil(S / sw)
  // direct (IMPLICIT_GEMM, zero workspace): RED alpha * partial straight into
  // dW[k][c][r][s] (`acc` = dw, beta applied by a scale pass first) instead
  // of into the GEMM-layout scratch + finalize; a warp's REDs then scatter
  // over 32 filter rows (DESIGN finding 8: ~8-18 us per call)
  int direct;
  float vscale;
  // xmn (swapped roles, few channels): x rows land MN-major (the 128B/32B-atom
  // swizzle, DESIGN finding 5) with lane = x row (c, r, s) at a fixed pixel,
  // so a warp's 32 cp.async read the S consecutive input columns of ~3 filter
  // rows -- a few sectors -- instead of 32 pixels at stride sw (AlexNet conv1:
  // 512 B, 16 sectors per instruction). Exact, but measured 2x slower on
  // AlexNet conv1 BF (1117 vs 591 us at 256 images; ncu: L1 35 % vs 64 %,
  // producer warps latency-bound on the per-pixel decode), so off by default
  // (UCUDNN_TUNE=bfl_xmn=1; profiles/r02_ncu_bfl_xmn_conv1_bf.txt)
  int xmn;
};

// RED target of partial (x row m, output channel k)
__device__ __forceinline__ float* red_target(const LParams& p, int m, int k) {
  if (p.direct) {
    int off = m;
    if (!p.crs) {  // row (r, s, c) -> dW offset c*R*S + r*S + s
      std::uint32_t rs, c, r, s;
      p.fd_C.divmod(std::uint32_t(m), rs, c);
      p.fd_S.divmod(rs, r, s);
      off = int(c) * p.R * p.S + int(r) * p.S + int(s);
    }
    return p.acc + std::int64_t(k) * p.M + off;
  }
  return p.swap ? p.acc + std::int64_t(m) * kBM + k : p.acc + std::int64_t(k) * p.rpad + m;
}

// 4-byte gather; src_size 0 writes a zero (src is then never dereferenced)
__device__ __forceinline__ void cp_async4a(std::uint32_t dst, std::uint64_t src, std::uint32_t src_size) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_size) : "memory");
}
// mbarrier arrive (without a pending-count increment) triggered when all of
// this thread's earlier cp.async have completed
__device__ __forceinline__ void cp_async_arrive(std::uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Waits that last a whole unit (the epilogue's) back off so their spinning
// does not steal issue slots from the gather warps.
__device__ __forceinline__ void mbar_wait_backoff(std::uint64_t* bar, std::uint32_t parity) {
  std::uint32_t ok = 0, ns = 128;
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
    if (ns < 4096) ns <<= 1;
  }
}
// MN-major 128B / 32 B-atom descriptor: LBO 4096 B between 32-row blocks
// (32 K-rows x 128 B), SBO 512 B (bfnhwc.cu desc_mn32)
__device__ __forceinline__ std::uint64_t desc_mn32(std::uint32_t saddr) {
  std::uint64_t d = 0;
  d |= std::uint64_t((saddr >> 4) & 0x3FFF);
  d |= std::uint64_t(4096 >> 4) << 16;
  d |= std::uint64_t(512 >> 4) << 32;
  d |= std::uint64_t(1) << 46;
  d |= std::uint64_t(1) << 61;
  return d;
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// bits t in [lo, hi) of a width-n tap mask (n <= 32)
__device__ __forceinline__ std::uint32_t range_mask(int lo, int hi, int n) {
  lo = max(lo, 0);
  hi = min(hi, n);
  if (hi <= lo) return 0u;
  const std::uint32_t h = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
  return h & ~((1u << lo) - 1u);
}

// The gather side shared by both kernels: per-thread constants, the
// per-unit row table (few-channel path) and one 32-pixel step into a stage.
template <int kProd>
struct Gatherer {
  const LParams& p;
  int lane, pw;
  bool c8;                 // C % 8 == 0: an 8-row group is 8 channels of one tap
  bool sg;                 // stride 2 / 4 with few channels: lane = (pixel, tap offset s')
  std::uint32_t swz[8];    // this lane's byte offset in an 8-row swizzle atom, per row q % 8
  std::uint32_t xj[8], dj[8];  // byte offsets of rows j of a group (independent adds)
  int2* xtab;
  int xm0, xrows, dk0, drows;  // current unit: x rows [xm0, +xrows), dy rows [dk0, +drows)

  __device__ __forceinline__ Gatherer(const LParams& p_, int lane_, int pw_, int2* tab)
      : p(p_), lane(lane_), pw(pw_), c8(!p_.crs && p_.C % 8 == 0 && !p_.xmn), sg(p_.sg != 0), xtab(tab) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      swz[j] = j * 128 + ((std::uint32_t(lane >> 2) ^ j) << 4) + (lane & 3) * 4;
      xj[j] = std::uint32_t(j * p.HW * 4);
      dj[j] = std::uint32_t(j * p.OHW * 4);
    }
  }

  __device__ __forceinline__ void unit(int xm0_, int xrows_, int dk0_, int drows_, int xrows2 = 0) {
    xm0 = xm0_;
    xrows = xrows_;
    dk0 = dk0_;
    drows = drows_;
    if (p.xmn) {
      // every producer warp reads every row's entry: (c*HW + r*W + s, r << 8 | s)
      named_sync(1, kProd * 32);  // all producers are done with the previous unit's table
      for (int j = pw * 32 + lane; j < xrows; j += kProd * 32) {
        std::uint32_t rs, c, r, s;
        if (p.crs) {
          p.fd_RS.divmod(std::uint32_t(xm0 + j), c, rs);
        } else {
          p.fd_C.divmod(std::uint32_t(xm0 + j), rs, c);
        }
        p.fd_S.divmod(rs, r, s);
        xtab[j] = make_int2(int(c) * p.HW + int(r) * p.W + int(s), int(r << 8 | s));
      }
      named_sync(1, kProd * 32);
    } else if (c8) {
      // this warp's 8-row groups (tile t, group q0/8): (c*HW + r*W + s, r << 16 | s),
      // so a step reads one smem word pair per group instead of two divisions
      for (int t = 0; t < (xrows2 > 0 ? 2 : 1); ++t) {
        const int rows = t ? xrows2 : xrows;
        const int q0 = pw * 8 + lane * kProd * 8;  // rows <= 256 (B tile of the swapped roles)
        if (q0 < rows) {
          std::uint32_t rs, c, r, s;
          p.fd_C.divmod(std::uint32_t(xm0 + t * 256 + q0), rs, c);
          p.fd_S.divmod(rs, r, s);
          xtab[t * 32 + q0 / 8] = make_int2(int(c) * p.HW + int(r) * p.W + int(s), int(r << 16 | s));
        }
      }
      __syncwarp();
    } else if (sg) {
      // this warp's tap groups (r, s0 = sgrp*sw, c): (c*HW + r*W + s0, r << 16 | s0 << 8 | c)
      // (built by the warp that reads it: gi = pw (mod kProd))
      for (int gi = pw + kProd * lane; gi < p.ngroups; gi += kProd * 32) {
        std::uint32_t rg, c, r, sgrp;
        p.fd_C.divmod(std::uint32_t(gi), rg, c);
        p.fd_sgs.divmod(rg, r, sgrp);
        const int s0 = int(sgrp) * p.sw;
        xtab[gi] = make_int2(int(c) * p.HW + int(r) * p.W + s0, int(r << 16 | s0 << 8 | c));
      }
      __syncwarp();
    } else if (!c8) {
      // this warp's rows of the tile: (c*HW + r*W + s, r << 8 | s)
      // (few channels, or (c, r, s) order)
      for (int q0 = pw * 8; q0 < xrows; q0 += kProd * 8)
        if (lane < 8 && q0 + lane < xrows) {
          std::uint32_t rs, c, r, s;
          if (p.crs) {
            p.fd_RS.divmod(std::uint32_t(xm0 + q0 + lane), c, rs);
          } else {
            p.fd_C.divmod(std::uint32_t(xm0 + q0 + lane), rs, c);
          }
          p.fd_S.divmod(rs, r, s);
          xtab[q0 + lane] = make_int2(int(c) * p.HW + int(r) * p.W + int(s), int(r << 8 | s));
        }
      __syncwarp();
    }
  }

  // Stride-2 / 4 x rows with few channels: row (r, s, c) of a 32-pixel step
  // reads x at stride sw along the pixels, i.e. 32 lanes would span 32*sw
  // floats. Instead lane = (pixel j, tap offset s' < sw): one cp.async covers
  // the sw taps s0 + s' of 32/sw consecutive pixels -- 32 *consecutive* x
  // floats -- and a group (r, s0, c) takes sw instructions (pixel subsets u).
  __device__ __forceinline__ void step_strided(int g, std::uint32_t xs) const {
    const int sw = p.sw, per = 32 / sw, sp = lane % sw, jl = lane / sw;
    const float* xl[4];
    int ihb[4], iwb[4];
    bool val[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u < sw) {
        const long long pg = (long long)g * 32 + u * per + jl;
        val[u] = pg < p.npx;
        std::uint32_t n, pix, oh, ow;
        p.fd_ohw.divmod(std::uint32_t(val[u] ? pg : 0), n, pix);
        p.fd_ow.divmod(pix, oh, ow);
        ihb[u] = int(oh) * p.sh - p.ph;
        iwb[u] = int(ow) * p.sw - p.pw;
        xl[u] = p.x + (long long)n * p.CHW + (long long)ihb[u] * p.W + iwb[u] + sp;
      }
    }
    for (int gi = pw; gi < p.ngroups; gi += kProd) {
      const int2 e = xtab[gi];
      const int r = e.y >> 16, s0 = (e.y >> 8) & 255, c = e.y & 255;
      const int s = s0 + sp;
      const int q = (r * p.S + s) * p.C + c - xm0;  // this lane's tile row
      const bool in = s < p.S && unsigned(q) < unsigned(xrows);
      if (!__any_sync(0xffffffffu, in)) continue;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (u < sw) {
          const int kk = u * per + jl;
          const bool ok = val[u] && unsigned(ihb[u] + r) < unsigned(p.H) && unsigned(iwb[u] + s) < unsigned(p.W);
          const std::uint32_t dst =
              xs + std::uint32_t(q) * 128 + ((std::uint32_t(kk >> 2) ^ (q & 7)) << 4) + (kk & 3) * 4;
          if (in) cp_async4a(dst, reinterpret_cast<std::uint64_t>(xl[u] + e.x), ok ? 4u : 0u);
        }
      }
    }
  }

  // x rows MN-major: block i of 32 rows at xs + i*4096, pixel k at K-row k
  __device__ __forceinline__ void step_xmn(int g, std::uint32_t xs) const {
    const std::uint32_t lsw = std::uint32_t(lane & 7) * 4, lg = std::uint32_t(lane >> 3);
    const int nblk = (xrows + 31) >> 5;
    for (int k = pw; k < 32; k += kProd) {
      const long long pg = (long long)g * 32 + k;
      const bool valid = pg < p.npx;
      std::uint32_t n, pix, oh, ow;
      p.fd_ohw.divmod(std::uint32_t(valid ? pg : 0), n, pix);
      p.fd_ow.divmod(pix, oh, ow);
      const int ihb = int(oh) * p.sh - p.ph, iwb = int(ow) * p.sw - p.pw;
      const float* xl = p.x + (long long)n * p.CHW + (long long)ihb * p.W + iwb;
      const std::uint32_t krow = xs + std::uint32_t(k) * 128 + ((lg ^ std::uint32_t(k & 3)) << 5) + lsw;
      for (int i = 0; i < nblk; ++i) {
        const int j = i * 32 + lane;
        std::uint32_t ok = 0;
        int off = 0;
        if (j < xrows) {
          const int2 e = xtab[j];
          const int r = e.y >> 8, s = e.y & 255;
          ok = (valid && unsigned(ihb + r) < unsigned(p.H) && unsigned(iwb + s) < unsigned(p.W)) ? 1u : 0u;
          off = e.x;
        }
        cp_async4a(krow + std::uint32_t(i) * 4096, reinterpret_cast<std::uint64_t>(ok ? xl + off : p.x), ok * 4u);
      }
    }
  }

  // x rows -> smem at xs, dy rows -> smem at ds (SW128 K-major, row q at q*128)
  // xs2 != 0 (CTA-pair kernel, C % 8 == 0): a second x tile, rows
  // [xm0 + 256, + xrows2), into xs2 -- the dy rows are gathered once for both
  __device__ __forceinline__ void step(int g, std::uint32_t xs, std::uint32_t ds, std::uint32_t xs2 = 0,
                                       int xrows2 = 0) const {
    const long long pg = (long long)g * 32 + lane;  // this lane's pixel
    const bool valid = pg < p.npx;
    std::uint32_t n, pix, oh, ow;
    p.fd_ohw.divmod(std::uint32_t(valid ? pg : 0), n, pix);
    p.fd_ow.divmod(pix, oh, ow);
    const int ihb = int(oh) * p.sh - p.ph, iwb = int(ow) * p.sw - p.pw;
    const float* xl = p.x + (long long)n * p.CHW + (long long)ihb * p.W + iwb;
    if (p.xmn) {
      step_xmn(g, xs);
    } else if (sg) {
      step_strided(g, xs);
    } else if (c8) {
      // one bounds test per group, then consecutive channel planes
      for (int t = 0; t < (xs2 ? 2 : 1); ++t) {
        const int rows = t ? xrows2 : xrows;
        const std::uint32_t base = t ? xs2 : xs;
        for (int q0 = pw * 8; q0 < rows; q0 += kProd * 8) {
          const int2 e = xtab[t * 32 + q0 / 8];
          const int r = e.y >> 16, s = e.y & 0xffff;
          const bool ok = valid && unsigned(ihb + r) < unsigned(p.H) && unsigned(iwb + s) < unsigned(p.W);
          const std::uint32_t sz = ok ? 4u : 0u, dst = base + q0 * 128;
          const std::uint64_t a = reinterpret_cast<std::uint64_t>(xl + e.x);
          const int qn = min(8, rows - q0);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < qn) cp_async4a(dst + swz[j], a + xj[j], sz);
        }
      }
    } else {
      // few channels (taps straddle groups): per-row (offset, tap) from the
      // smem table, bounds from this lane's valid-tap bitmasks
      const std::uint32_t vr = valid ? range_mask(-ihb, p.H - ihb, p.R) : 0u;
      const std::uint32_t vs = range_mask(-iwb, p.W - iwb, p.S);
      const std::uint64_t xa = reinterpret_cast<std::uint64_t>(xl);
      for (int q0 = pw * 8; q0 < xrows; q0 += kProd * 8) {
        const std::uint32_t dst = xs + q0 * 128;
        const int qn = min(8, xrows - q0);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < qn) {
            const int2 e = xtab[q0 + j];
            const std::uint32_t ok = (vr >> (e.y >> 8)) & (vs >> (e.y & 255)) & 1u;
            cp_async4a(dst + swz[j], xa + std::int64_t(e.x) * 4, ok * 4u);
          }
        }
      }
    }
    const float* dl = p.dy + (long long)n * p.KOHW + pix;
    const std::uint32_t sz = valid ? 4u : 0u;
    for (int q0 = pw * 8; q0 < drows; q0 += kProd * 8) {
      const std::uint64_t a = reinterpret_cast<std::uint64_t>(dl + (long long)(dk0 + q0) * p.OHW);
      const std::uint32_t dst = ds + q0 * 128;
      const int qn = min(8, drows - q0);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < qn) cp_async4a(dst + swz[j], a + dj[j], sz);
    }
  }
};

__global__ void __launch_bounds__(threads_for<kProd1>(), 1) bfl_kernel(const LParams p) {
  constexpr int kProd = kProd1;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t a_bytes = kBM * 128;
  const std::uint32_t stage_bytes = a_bytes + ((std::uint32_t(p.BN) * 128 + 1023) & ~1023u);
  const int kStages = p.stages;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kStages * stage_bytes);
  std::uint64_t* empty = full + kMaxStages;
  std::uint64_t* tfull = empty + kMaxStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  __shared__ int2 xtab[kMaxBN];  // few-channel path: per x row of the tile

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], kProd * 32);  // every producer thread, cp.async arrive
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
  const int units = p.tiles * p.splits;

  if (warp >= 5) {
    // ------------------------------------------------ gather producers
    Gatherer<kProd> ga(p, lane, warp - 5, xtab);
    const std::uint32_t sbase = smem_u32(smem);
    // x rows go to A (non-swap) or B (swap); dy rows to the other
    const std::uint32_t x_off = p.swap ? a_bytes : 0, d_off = p.swap ? 0 : a_bytes;
    int st = 0;
    std::uint32_t ph = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int tile = u % p.tiles, split = u / p.tiles;
      const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
      const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
      const int xm0 = p.swap ? nt * p.BN : mt * kBM;  // first x row of the tile
      const int dk0 = p.swap ? 0 : nt * p.BN;
      ga.unit(xm0, min(p.swap ? p.BN : kBM, p.M - xm0), dk0, min(p.swap ? kBM : p.BN, p.K - dk0));
      for (int g = g0; g < g1; ++g) {
        mbar_wait(&empty[st], ph ^ 1);
        const std::uint32_t sst = sbase + st * stage_bytes;
        if (p.dbg != 1) ga.step(g, sst + x_off, sst + d_off);
        // arrives once every cp.async this thread issued so far has landed
        cp_async_arrive(&full[st]);
        if (++st == kStages) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------------ MMA issuer
    // xmn: B (the x rows) MN-major -- instruction-descriptor bit 16
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN) | (p.xmn ? (1u << 16) : 0u);
    const std::uint32_t sbase = smem_u32(smem);
    int it = 0, tl = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
      const int split = u / p.tiles;
      const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
      const int acc = tl & 1;
      mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
      tc_fence_after();
      const std::uint32_t dtm = tmem + std::uint32_t(acc * kMaxBN);
      for (int g = g0; g < g1; ++g, ++it) {
        const int st = it % kStages;
        mbar_wait(&full[st], (it / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          // the operands were written through the generic proxy (cp.async):
          // order them before the tensor core's async-proxy reads
          fence_async_smem();
          const std::uint32_t sa = sbase + st * stage_bytes, sb = sa + a_bytes;
          if (p.dbg != 2)
#pragma unroll
            for (int q = 0; q < 4; ++q)
              mma_tf32(dtm, umma_desc_sw128(sa + q * 32), p.xmn ? desc_mn32(sb + q * 1024) : umma_desc_sw128(sb + q * 32),
                       idesc,
                       (g != g0 || q != 0) ? 1u : 0u);
          mma_commit(&empty[st]);
          if (g + 1 >= g1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
      if (g1 <= g0 && lane == 0) mma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------ epilogue: RED into the scratch
    const int ew = warp;
    int tl = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
      const int tile = u % p.tiles, split = u / p.tiles;
      const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
      const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
      const int acc = tl & 1;
      mbar_wait_backoff(&tfull[acc], (tl >> 1) & 1);
      tc_fence_after();
      const std::uint32_t tbase = tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t(acc * kMaxBN);
      if (p.swap) {
        // TMEM lane = output channel k, column = x row nt*BN + j
        const int k = ew * 32 + lane;
        const bool live = k < p.K && g1 > g0;
        for (int c0 = 0; c0 < p.BN; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + std::uint32_t(c0), v);
          if (!live) continue;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int m = nt * p.BN + c0 + j;
            if (c0 + j >= p.BN || m >= p.M) break;
            red_add(red_target(p, m, k), p.vscale * v[j]);
          }
        }
      } else {
        const int m = mt * kBM + ew * 32 + lane;
        const bool live = m < p.M && g1 > g0;
        for (int c0 = 0; c0 < p.BN; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + std::uint32_t(c0), v);
          if (!live) continue;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int k = nt * p.BN + c0 + j;
            if (c0 + j >= p.BN || k >= p.K) break;
            red_add(red_target(p, m, k), p.vscale * v[j]);
          }
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

// CTA-pair variant (K > 128, roles not swapped): tcgen05.mma.cta_group::2,
// M = 256 x rows (128 gathered by each CTA into its own smem) x BN output
// channels, the dy rows split along N (BN/2 gathered by each CTA) -- half
// the dy gather per SM of the 1-SM kernel. Rank 0 issues the MMAs; rank 1's
// warp 4 relays its producers' completion (its own cp.async full barrier)
// to rank 0's full barrier after the proxy fence. Commits multicast to both
// CTAs; both epilogues release rank 0's accumulator barrier.
__global__ void __launch_bounds__(threads_for<kProd2>(), 1) bfl2_kernel(const LParams p) {
  constexpr int kProd = kProd2;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t rank = cluster_rank();
  const int bh = p.BN / 2;
  const std::uint32_t a_bytes = kBM * 128;
  // dual: two 256-row pair tiles per unit (acc 0 / 1 at TMEM columns 0 / 256)
  // sharing one dy gather; the accumulators then fill TMEM, so units are
  // not double-buffered
  const int nsub = p.dual ? 2 : 1;
  const std::uint32_t stage_bytes = nsub * a_bytes + ((std::uint32_t(bh) * 128 + 1023) & ~1023u);
  const int kStages = p.stages;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kStages * stage_bytes);
  std::uint64_t* empty = full + kMaxStages;
  std::uint64_t* tfull = empty + kMaxStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  __shared__ int2 xtab[kMaxBN];

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], kProd * 32 + (rank == 0 ? 1 : 0));  // + rank 1's relay
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 256);
    }
    mbar_fence_init();
  }
  if (warp == 4) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const std::uint32_t tmem = tmem_base_uniform(tmem_slot);
  const int units = p.tiles * p.splits;  // tiles = pair tiles x n tiles
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp >= 5) {
    // ------------------------------------------------ gather producers
    Gatherer<kProd> ga(p, lane, warp - 5, xtab);
    const std::uint32_t sbase = smem_u32(smem);
    int st = 0;
    std::uint32_t ph = 0;
    for (int u = cid; u < units; u += ncl) {
      const int tile = u % p.tiles, split = u / p.tiles;
      const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
      const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
      const int xm0 = mt * 2 * nsub * kBM + int(rank) * kBM, dk0 = nt * p.BN + int(rank) * bh;
      const int xrows2 = min(kBM, p.M - xm0 - 2 * kBM);
      ga.unit(xm0, min(kBM, p.M - xm0), dk0, min(bh, p.K - dk0), p.dual ? xrows2 : 0);
      for (int g = g0; g < g1; ++g) {
        mbar_wait(&empty[st], ph ^ 1);
        const std::uint32_t sst = sbase + st * stage_bytes;
        if (p.dbg != 1) {
          if (p.dual) ga.step(g, sst, sst + 2 * a_bytes, sst + a_bytes, xrows2);
          else ga.step(g, sst, sst + a_bytes);
        }
        cp_async_arrive(&full[st]);
        if (++st == kStages) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 4) {
    if (rank == 0) {
      // ------------------------------------------------ MMA issuer (pair)
      const std::uint32_t idesc = idesc_tf32(2 * kBM, p.BN);
      const std::uint32_t sbase = smem_u32(smem);
      int it = 0, tl = 0;
      for (int u = cid; u < units; u += ncl, ++tl) {
        const int split = u / p.tiles;
        const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
        const int acc = p.dual ? 0 : (tl & 1);
        const std::uint32_t tpar = p.dual ? ((tl & 1) ^ 1) : (((tl >> 1) & 1) ^ 1);
        mbar_wait(&tempty[acc], tpar);
        tc_fence_after();
        const std::uint32_t dtm = tmem + std::uint32_t(acc * kMaxBN);
        for (int g = g0; g < g1; ++g, ++it) {
          const int st = it % kStages;
          mbar_wait(&full[st], (it / kStages) & 1);
          tc_fence_after();
          if (lane == 0) {
            fence_async_smem();
            const std::uint32_t sa = sbase + st * stage_bytes, sb = sa + nsub * a_bytes;
            if (p.dbg != 2)
              for (int t = 0; t < nsub; ++t)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  mma_tf32_2sm(dtm + std::uint32_t(t * kMaxBN), umma_desc_sw128(sa + t * a_bytes + q * 32),
                               umma_desc_sw128(sb + q * 32), idesc, (g != g0 || q != 0) ? 1u : 0u);
            mma_commit_2sm(&empty[st], 3);
            if (g + 1 >= g1) mma_commit_2sm(&tfull[acc], 3);
          }
          __syncwarp();
        }
        if (g1 <= g0 && lane == 0) mma_commit_2sm(&tfull[acc], 3);
        __syncwarp();
      }
    } else if (lane == 0) {
      // ------------------------------------------------ relay (rank 1)
      const std::uint32_t full0 = mapa(smem_u32(&full[0]), 0);
      int it = 0;
      for (int u = cid; u < units; u += ncl) {
        const int split = u / p.tiles;
        const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
        for (int g = g0; g < g1; ++g, ++it) {
          const int st = it % kStages;
          mbar_wait(&full[st], (it / kStages) & 1);
          fence_async_smem();
          mbar_arrive_remote(full0 + std::uint32_t(st) * 8);
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ epilogue: RED into the scratch
    const int ew = warp;
    const std::uint32_t tempty0 = mapa(smem_u32(&tempty[0]), 0);
    int tl = 0;
    for (int u = cid; u < units; u += ncl, ++tl) {
      const int tile = u % p.tiles, split = u / p.tiles;
      const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
      const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
      const int acc = p.dual ? 0 : (tl & 1);
      mbar_wait_backoff(&tfull[acc], p.dual ? (tl & 1) : ((tl >> 1) & 1));
      tc_fence_after();
      for (int t = 0; t < nsub; ++t) {
        const std::uint32_t tbase =
            tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t((acc + t) * kMaxBN);
        const int m = mt * 2 * nsub * kBM + t * 2 * kBM + int(rank) * kBM + ew * 32 + lane;
        const bool live = m < p.M && g1 > g0;
        for (int c0 = 0; c0 < p.BN; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + std::uint32_t(c0), v);
          if (!live) continue;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int k = nt * p.BN + c0 + j;
            if (c0 + j >= p.BN || k >= p.K) break;
            red_add(red_target(p, m, k), p.vscale * v[j]);
          }
        }
      }
      tc_fence_before();
      if (rank == 0) mbar_arrive(&tempty[acc]);
      else mbar_arrive_remote(tempty0 + std::uint32_t(acc) * 8);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 4) {
    tc_fence_after();
    tmem_free_2sm<512>(tmem);
  }
}

// dW[k][c][r][s] = beta * dW + alpha * scratch(row = (r*S + s)*C + c, k)
struct LFinal {
  const float* acc;
  float* dw;
  float alpha, beta;
  int C, R, S, rpad, swap, crs;
  std::int64_t n;  // K*C*R*S
};
__global__ void __launch_bounds__(256) bfl_finalize_kernel(const LFinal f) {
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < f.n;
       i += std::int64_t(gridDim.x) * blockDim.x) {
    const int s = int(i % f.S);
    std::int64_t t = i / f.S;
    const int r = int(t % f.R);
    t /= f.R;
    const int c = int(t % f.C), k = int(t / f.C);
    const int row = f.crs ? int(i % (std::int64_t(f.C) * f.R * f.S)) : (r * f.S + s) * f.C + c;
    const float v = f.swap ? f.acc[std::int64_t(row) * kBM + k] : f.acc[std::int64_t(k) * f.rpad + row];
    f.dw[i] = f.beta == 0.f ? f.alpha * v : f.alpha * v + f.beta * f.dw[i];
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

}  // namespace

bool bfl_supports(const ConvShape& s) {
  const LGeo g = make_lgeo(s);
  // few-channel path: tap masks are 32 bits, table offsets int32
  const bool few_ok = (s.C % 8 == 0 && !tune("bfl_crs", 0)) ||
                      (s.R <= 32 && s.S <= 32 && std::int64_t(s.C) * s.H * s.W < (1ll << 31));
  return few_ok && g.npx + 64 < (std::int64_t(1) << 31) && g.M < (1 << 24) && s.K < (1 << 24);
}

std::int64_t bfl_workspace(const ConvShape& s) { return std::int64_t(scratch_bytes(make_lgeo(s))); }

cudaError_t bfl_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha, float beta,
                    cudaStream_t st, bool direct) {
  const LGeo g = make_lgeo(s);
  float* acc = direct ? dw : static_cast<float*>(ws);
  cudaError_t e = direct ? scale_tensor(dw, s.w_elems(), beta, st)
                         : cudaMemsetAsync(acc, 0, std::size_t(rows_pad(g)) * cols_pad(g) * 4, st);
  if (e != cudaSuccess) return e;
  const int sms = sm_count();
  LParams p{};
  p.x = x;
  p.dy = dy;
  p.acc = acc;
  p.C = g.C; p.H = g.H; p.W = g.W; p.K = g.K; p.R = g.R; p.S = g.S;
  p.sh = g.sh; p.sw = g.sw; p.ph = g.ph; p.pw = g.pw; p.OW = g.OW;
  p.OHW = g.OH * g.OW;
  p.HW = g.H * g.W;
  p.M = g.M;
  p.npx = g.npx;
  p.CHW = std::int64_t(g.C) * p.HW;
  p.KOHW = std::int64_t(g.K) * p.OHW;
  p.swap = g.swap;
  p.BN = g.BN;
  p.m_tiles = g.m_tiles;
  p.tiles = g.m_tiles * g.n_tiles;
  p.steps = g.steps;
  p.rpad = rows_pad(g);
  p.dbg = tune("bfl_dbg", 0);
  p.direct = direct ? 1 : 0;
  p.vscale = direct ? alpha : 1.f;
  p.fd_ohw = FastDiv(std::uint32_t(p.OHW));
  p.fd_ow = FastDiv(std::uint32_t(g.OW));
  p.fd_C = FastDiv(std::uint32_t(g.C));
  p.fd_S = FastDiv(std::uint32_t(g.S));
  p.fd_RS = FastDiv(std::uint32_t(g.R * g.S));
  // (c, r, s) rows (UCUDNN_TUNE=bfl_crs=1): a tile then holds every tap of a
  // few channels and the taps' overlapping x reads hit L1 (hit rate 35 -> 58 %,
  // L2 throughput halved), but every row needs the table path and AlexNet
  // conv2 at 256 images measured 503 -> 787 us, so (r, s, c) stays
  p.crs = tune("bfl_crs", 0);
  p.dual = g.dual;
  // strided few-channel x gather (AlexNet / ResNet conv1)
  p.sgs = (g.S + g.sw - 1) / g.sw;
  p.ngroups = g.R * p.sgs * g.C;
  p.sg = !p.crs && g.C % 8 != 0 && (g.sw == 2 || g.sw == 4) && g.C < 256 && p.ngroups <= kMaxBN &&
         tune("bfl_sg", 0);  // exact, but issue-bound: AlexNet conv1 BF 542 -> 876 us, ResNet conv1 1031 -> 1601
  p.fd_sgs = FastDiv(std::uint32_t(p.sgs));
  p.xmn = g.swap && !p.sg && (g.C % 8 != 0 || p.crs) && tune("bfl_xmn", 0);
  // split the reduction so the tiles fill the SMs once, >= 8 steps per unit
  const int slots = g.two ? sms / 2 : sms;
  const int splits =
      deterministic() ? 1 : std::max(1, std::min(p.steps / 8, tune("bfl_waves", 1) * slots / p.tiles));
  p.steps_per_unit = (p.steps + splits - 1) / splits;
  p.splits = (p.steps + p.steps_per_unit - 1) / p.steps_per_unit;
  const int stage_bytes = (g.dual ? 2 : 1) * kBM * 128 + (((g.two ? g.BN / 2 : g.BN) * 128 + 1023) & ~1023);
  p.stages = std::max(2, std::min({kMaxStages, tune("bfl_stages", 4), (200 * 1024) / stage_bytes}));
  // 4 stages: the rest of the 228 KB stays L1, which catches the taps' re-reads
  // of x (AlexNet conv3-5 at 256 images: 8 stages 282/312/208 us, 4 stages
  // 249/265/175 us)
  const int smem = p.stages * stage_bytes + 1024 + 256;
  // + 2 KB static xtab
  e = set_smem_attr(reinterpret_cast<const void*>(bfl_kernel), 220 * 1024);
  if (e == cudaSuccess) e = set_smem_attr(reinterpret_cast<const void*>(bfl2_kernel), 220 * 1024);
  if (e != cudaSuccess) return e;
  trace_variant("%s tiles=%d splits=%d swap=%d dual=%d direct=%d xmn=%d", g.two ? "bfl2" : "bfl", p.tiles,
                p.splits, int(g.swap), int(g.dual), p.direct, p.xmn);
  if (g.two) {
    count_launch();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * std::min(sms / 2, p.tiles * p.splits));
    cfg.blockDim = dim3(threads_for<kProd2>());
    cfg.dynamicSmemBytes = std::size_t(smem);
    cfg.stream = st;
    cudaLaunchAttribute cat[1];
    cat[0].id = cudaLaunchAttributeClusterDimension;
    cat[0].val.clusterDim.x = 2;
    cat[0].val.clusterDim.y = 1;
    cat[0].val.clusterDim.z = 1;
    cfg.attrs = cat;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, bfl2_kernel, p);
  } else {
    e = launch_pdl(bfl_kernel, dim3(std::min(sms, p.tiles * p.splits)), dim3(threads_for<kProd1>()),
                   std::size_t(smem), st, p);
  }
  if (e != cudaSuccess || direct) return e;
  LFinal f{acc, dw, alpha, beta, g.C, g.R, g.S, rows_pad(g), g.swap, p.crs, s.w_elems()};
  return launch_pdl(bfl_finalize_kernel, dim3(int(std::min<std::int64_t>((f.n + 255) / 256, 8 * sms))), dim3(256), 0,
                    st, f);
}

}  // namespace ucudnn
