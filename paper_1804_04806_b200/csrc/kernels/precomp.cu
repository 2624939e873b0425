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
#include <cstdlib>
#include <mutex>

#include "bfilter.h"
#include "z1x1.h"
#include "conv_common.h"
#include "launch.h"
#include "precomp.h"
#include "sm100.cuh"

namespace ucudnn {
using namespace sm100;

namespace {

constexpr int kBM = 128;
// ring depth that splits evenly over 3 or 2 producer threads
inline int ring_stages(int fit) { return fit > 8 ? 8 : fit < 2 ? 2 : fit; }
constexpr int kMaxStages = 8;
// 32-deep reduction chunks per pipeline stage: a tcgen05.commit costs
// several hundred cycles of issue time, so each commit covers 8 MMAs
// (scripts/mma_probe.cu)
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
  // phase scatter epilogue (strided BackwardData): column (a, b, c) of
  // output pixel (n, i, j) is dx[n][c][i*ssh + a - sph][j*ssw + b - spw]
  int phase, Cr, Hr, Wr, ssh, ssw, sph, spw;
  int pair;      // 1x1 stride-2 block stores (phase_store)
  int bp;        // blocked phase BD: phase-grid columns per GEMM row (column = (pb, a, b, c))
  FastDiv fd_blk;  // Ah * Bw * C
  int sAh, sBw;  // phases with taps (< ssh, ssw when the filter is narrower than the stride)
  int ph32;      // phase chunks of 32 columns are one (a, b): phase_store32
  int stages, ksub, prof, cps;
  int nacc2;  // precomp2: accumulator sets (2 when 2 * msub * BN <= 512)
  int msub;      // 1-SM kernel: 128-pixel MMA sub-tiles per tile sharing each B (filter) chunk
  FastDiv fd_Cr, fd_ssw;
};

// Stride-phase BackwardData when the filter is narrower than the stride (1x1
// stride-2 shortcuts): only phases a < sAh, b < sBw have taps and are GEMM
// columns; dx at the other phases gets beta * dx (0 for beta = 0), written
// by whoever owns column (0, 0, c) of the same pixel.
template <typename P>
__device__ __forceinline__ void tapless_phases(const P& p, float* base, int c, int hb, int wb) {
  if (p.sAh >= p.ssh && p.sBw >= p.ssw) return;
  for (int a = 0; a < p.ssh; ++a)
    for (int b = 0; b < p.ssw; ++b) {
      if (a < p.sAh && b < p.sBw) continue;
      const int h = hb + a, w = wb + b;
      if (unsigned(h) >= unsigned(p.Hr) || unsigned(w) >= unsigned(p.Wr)) continue;
      float* dst = base + (std::int64_t(c) * p.Hr + h) * p.Wr + w;
      *dst = p.beta == 0.f ? 0.f : p.beta * *dst;
    }
}

// One stride-phase BackwardData output: column col of the pixel whose dx
// block starts at (hb, wb). pair = 1x1 stride-2 unpadded with even dx extents
// (ResNet shortcuts): only (0, 0) of the 2x2 block has a tap, so the thread
// writes the whole block as two float2 rows -- warp-contiguous along j,
// instead of four scattered stride-2 scalars per column.
template <typename P>
__device__ __forceinline__ void phase_store(const P& p, std::int64_t obase, int col, int hb, int wb, float val) {
  if (p.pair) {
    float2* d0 = reinterpret_cast<float2*>(p.out + obase + (std::int64_t(col) * p.Hr + hb) * p.Wr + wb);
    float2* d1 = d0 + (p.Wr >> 1);
    if (p.beta == 0.f) {
      *d0 = make_float2(val, 0.f);
      *d1 = make_float2(0.f, 0.f);
    } else {
      const float2 o0 = *d0, o1 = *d1;
      *d0 = make_float2(val + p.beta * o0.x, p.beta * o0.y);
      *d1 = make_float2(p.beta * o1.x, p.beta * o1.y);
    }
    return;
  }
  if (p.bp > 1) {  // blocked: column (pb, a, b, c) belongs to phase-grid column j + pb
    std::uint32_t pb, rem;
    p.fd_blk.divmod(std::uint32_t(col), pb, rem);
    col = int(rem);
    wb += int(pb) * p.ssw;
  }
  std::uint32_t ab, c, a, b;
  p.fd_Cr.divmod(std::uint32_t(col), ab, c);
  p.fd_ssw.divmod(ab, a, b);
  if (ab == 0) tapless_phases(p, p.out + obase, int(c), hb, wb);
  const int h = hb + int(a), w = wb + int(b);
  if (unsigned(h) >= unsigned(p.Hr) || unsigned(w) >= unsigned(p.Wr)) return;
  float* dst = p.out + obase + (std::int64_t(c) * p.Hr + h) * p.Wr + w;
  *dst = p.beta == 0.f ? val : val + p.beta * *dst;
}

// 32 output columns of one row (column j at base[j * pitch], n valid):
// beta == 0 stores; otherwise every old value is loaded before the first
// store, so the 32 load latencies overlap instead of serialising behind
// the stores (the sliced algorithm runs most of its calls with beta = 1)
template <typename P>
__device__ __forceinline__ void store_row32(const P& p, float* base, int n, std::int64_t pitch, const float (&v)[32]) {
  if (p.beta == 0.f) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < n) base[j * pitch] = p.alpha * v[j];
  } else {
    // 8 loads in flight at a time: the 1-SM kernel must stay <= 128
    // registers to run two CTAs per SM
#pragma unroll
    for (int j0 = 0; j0 < 32; j0 += 8) {
      float o[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = j0 + j < n ? base[(j0 + j) * pitch] : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j0 + j < n) base[(j0 + j) * pitch] = p.alpha * v[j0 + j] + p.beta * o[j];
    }
  }
}

// Stride-phase scatter of one pixel's 32-column chunk when every chunk is a
// single phase (a, b): the phase-channel count is a multiple of 32 and there
// are no blocked columns, pair stores or tapless phases (p.ph32, set on the
// host). The chunk's (a, b, c) is decoded once and its channels are strided
// stores (store_row32) -- instead of a divmod pair, a tapless test and a
// bounds test per value, which made the epilogue the bound of the strided
// BackwardData (30 M warp instructions for ResNet-18 l2b1c1 at 64 images).
template <typename P>
__device__ __forceinline__ void phase_store32(const P& p, std::int64_t obase, int col0, int n, int hb, int wb,
                                              const float (&v)[32]) {
  std::uint32_t ab, c, a, b;
  p.fd_Cr.divmod(std::uint32_t(col0), ab, c);
  p.fd_ssw.divmod(ab, a, b);
  const int h = hb + int(a), w = wb + int(b);
  if (unsigned(h) >= unsigned(p.Hr) || unsigned(w) >= unsigned(p.Wr)) return;
  store_row32(p, p.out + obase + (std::int64_t(c) * p.Hr + h) * p.Wr + w, n, std::int64_t(p.Hr) * p.Wr, v);
}

__device__ __forceinline__ void tile_coords(const PrecompParams& p, int t, int& mt, int& nt) {
  std::uint32_t q, r;
  p.fd_mt.divmod(std::uint32_t(t), q, r);
  nt = int(q);
  mt = int(r);
}

// UCUDNN_TUNE=prof=1: per-CTA cycle counters of the MMA warp (wait-for-data,
// issue, wait-for-accumulator) -- a diagnostic, read by ucudnnDebugProfile.
__device__ unsigned long long g_prof[1024 * 4];

__global__ void __launch_bounds__(kThreads, 1)
    precomp_kernel(const __grid_constant__ CUtensorMap amap, const PrecompParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t a_bytes = kBM * 128;
  const std::uint32_t b_bytes = std::uint32_t(p.BN) * 128;
  const int msub = p.msub;
  const std::uint32_t sub_bytes = msub * a_bytes + ((b_bytes + 1023) & ~1023u);
  const int kSub = p.ksub;
  const std::uint32_t stage_bytes = kSub * sub_bytes;
  const int kStages = p.stages;
  const int jsteps = (p.ksteps + kSub - 1) / kSub;  // pipeline stages per tile
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kStages * stage_bytes);
  std::uint64_t* empty = full + kMaxStages;
  std::uint64_t* tfull = empty + kMaxStages;
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
  // cps == 2: two CTAs share the SM (256 TMEM columns each; one accumulator
  // when BN > 128, so the other CTA's MMAs cover this one's epilogue)
  if (warp == 1) {
    if (p.cps == 2) tmem_alloc<256>(tmem_slot);
    else tmem_alloc<512>(tmem_slot);
  }
  const int nacc = p.cps == 2 && p.BN > 128 ? 1 : 2;
  const std::uint32_t acc_cols = p.cps == 2 ? 128u : std::uint32_t(kMaxBN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = tmem_base_uniform(tmem_slot);
  pdl_wait();  // everything above touched only smem / TMEM / the param-space tensor map
  pdl_trigger();
  const int total_tiles = p.m_tiles * p.n_tiles;

  if (warp == 0 || warp == 2 || warp == 3) {
    // up to three producer threads, stage s owned by thread s % 3 (one
    // thread's TMA issue stream keeps only about one stage in flight:
    // scripts/tma_probe.cu). Fixed ownership keeps every stage's parity
    // waits in order, so no producer can run two rounds ahead on a stage.
    const int pq = warp == 0 ? 0 : warp - 1;
    const int nprod = kStages < 3 ? kStages : 3;
    if (lane == 0) {
      // ------------------------------------------------ producer
      int it = 0;
      RingOwner ro;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        int mt, nt;
        tile_coords(p, t, mt, nt);
        // TMA start coordinates of each sub-tile's first output pixel (raster order)
        // (two sub-tiles at most: scalars, not an indexed array -- no stack frame)
        int cw0, ch0, n0, cw1 = 0, ch1 = 0, n1 = 0;
        {
          std::uint32_t n, pix, oh, ow;
          p.fd_P.divmod(std::uint32_t(mt * msub * kBM), n, pix);
          p.fd_OW.divmod(pix, oh, ow);
          cw0 = int(ow) * p.sw - p.pw;
          ch0 = int(oh) * p.sh - p.ph;
          n0 = int(n);
          if (msub == 2) {
            p.fd_P.divmod(std::uint32_t((mt * 2 + 1) * kBM), n, pix);
            p.fd_OW.divmod(pix, oh, ow);
            cw1 = int(ow) * p.sw - p.pw;
            ch1 = int(oh) * p.sh - p.ph;
            n1 = int(n);
          }
        }
        const float* bsrc = p.btiles + std::size_t(nt) * p.ksteps * (b_bytes / 4);
        for (int j = 0; j < jsteps; ++j, ++it, ro.step(kStages, nprod)) {
          if (ro.own != pq) continue;
          const int s = ro.slot;
          mbar_wait(&empty[s], ro.ph ^ 1);
          const int k0 = j * kSub, nsub = min(kSub, p.ksteps - k0);
          mbar_expect_tx(&full[s], nsub * (msub * a_bytes + b_bytes));
          for (int sub = 0; sub < nsub; ++sub) {
            const int k = k0 + sub;
            for (int m = 0; m < msub; ++m) {
              unsigned char* sa = smem + s * stage_bytes + sub * sub_bytes + m * a_bytes;
              const int cwm = m ? cw1 : cw0, chm = m ? ch1 : ch0, nm = m ? n1 : n0;
              if (p.small_c) {
#pragma unroll 1
                for (int g = 0; g < 8; ++g) {
                  int tap = k * 8 + g;
                  if (tap >= p.taps) tap = p.taps - 1;  // its B rows are zero
                  const int r = tap / p.S, q = tap - r * p.S;
                  tma_im2col_4d(sa + g * (kBM * 16), &amap, &full[s], 0, cwm, chm, nm, (unsigned short)q,
                                (unsigned short)r);
                }
              } else {
                const int tap = k / p.c_chunks, cc = k - tap * p.c_chunks;
                const int r = tap / p.S, q = tap - r * p.S;
                tma_im2col_4d(sa, &amap, &full[s], cc * 32, cwm, chm, nm, (unsigned short)q,
                              (unsigned short)r);
              }
            }
            bulk_g2s(smem + s * stage_bytes + sub * sub_bytes + msub * a_bytes,
                     bsrc + std::size_t(k) * (b_bytes / 4), b_bytes, &full[s]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN);
    const std::uint32_t sbase = smem_u32(smem);
    int it = 0, tl = 0;
    RingPos rp;
    long long c_data = 0, c_issue = 0, c_acc = 0, t_start = clock64();
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++tl) {
      const int acc = tl % nacc;
      long long c0 = p.prof ? clock64() : 0;
      mbar_wait(&tempty[acc], ((tl / nacc) & 1) ^ 1);
      tc_fence_after();
      if (p.prof) c_acc += clock64() - c0;
      const std::uint32_t dtm = tmem + std::uint32_t(acc) * acc_cols;
      for (int j = 0; j < jsteps; ++j, ++it, rp.step(kStages)) {
        const int s = rp.slot;
        long long c1 = p.prof ? clock64() : 0;
        mbar_wait(&full[s], rp.ph);
        tc_fence_after();
        long long c2 = p.prof ? clock64() : 0;
        if (p.prof) c_data += c2 - c1;
        const int k0 = j * kSub, nsub = min(kSub, p.ksteps - k0);
        {  // whole warp, one elected lane issues (sm100.cuh mma_tf32_w)
          for (int sub = 0; sub < nsub; ++sub) {
            const std::uint32_t sa0 = sbase + s * stage_bytes + sub * sub_bytes, sb = sa0 + msub * a_bytes;
            for (int m = 0; m < msub; ++m) {
              const std::uint32_t sa = sa0 + m * a_bytes;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                std::uint64_t ad = p.small_c ? umma_desc(sa + 2 * q * (kBM * 16), kBM * 16, 128)
                                             : umma_desc_sw128(sa + q * 32);
                std::uint64_t bd = umma_desc_sw128(sb + q * 32);
                mma_tf32_w(dtm + std::uint32_t(m * p.BN), ad, bd, idesc, ((k0 + sub) | q) != 0);
              }
            }
          }
          mma_commit_w(&empty[s]);
          if (j == jsteps - 1) mma_commit_w(&tfull[acc]);
        }
        __syncwarp();
        if (p.prof) c_issue += clock64() - c2;
      }
    }
    if (p.prof && lane == 0 && blockIdx.x < 1024) {
      g_prof[blockIdx.x * 4 + 0] = c_data;
      g_prof[blockIdx.x * 4 + 1] = c_issue;
      g_prof[blockIdx.x * 4 + 2] = c_acc;
      g_prof[blockIdx.x * 4 + 3] = clock64() - t_start;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue
    const int ew = warp - 4;
    // Stride-phase scatter without tapless phases or pair stores: every
    // column's (a, pb * ssw + b, c) decode depends on the column only, so it
    // is tabulated once per column tile (the per-element decode -- three fast
    // divisions -- kept the epilogue behind the MMAs: AlexNet conv1 BD's MMA
    // warp waited 27 % of its time for a free accumulator)
    __shared__ int ptab_dh[kMaxBN], ptab_dw[kMaxBN];
    __shared__ std::int64_t ptab_off[kMaxBN];
    const bool ptab = p.phase && !p.pair && p.sAh >= p.ssh && p.sBw >= p.ssw;
    int tab_nt = -1;
    int tl = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++tl) {
      int mt, nt;
      tile_coords(p, t, mt, nt);
      if (ptab && nt != tab_nt) {
        asm volatile("bar.sync 1, 128;" ::: "memory");  // previous tile done with the table
        for (int j = ew * 32 + lane; j < p.BN; j += 128) {
          std::uint32_t col = std::uint32_t(nt * p.BN + j), pb = 0, rem = col;
          if (p.bp > 1) p.fd_blk.divmod(col, pb, rem);
          std::uint32_t ab, c, a, b;
          p.fd_Cr.divmod(rem, ab, c);
          p.fd_ssw.divmod(ab, a, b);
          ptab_dh[j] = int(a);
          ptab_dw[j] = int(pb) * p.ssw + int(b);
          ptab_off[j] = std::int64_t(c) * p.Hr * p.Wr;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        tab_nt = nt;
      }
      const int acc = tl % nacc;
      mbar_wait(&tfull[acc], (tl / nacc) & 1);
      tc_fence_after();
      for (int m = 0; m < msub; ++m) {
      const int row = (mt * msub + m) * kBM + ew * 32 + lane;
      const bool ok = row < p.M;
      std::int64_t obase = 0;
      int hb = 0, wb = 0;
      if (ok) {
        std::uint32_t n, pix;
        p.fd_P.divmod(std::uint32_t(row), n, pix);
        obase = std::int64_t(n) * p.Nout * p.P + pix;
        if (p.phase) {
          std::uint32_t i, j;
          p.fd_OW.divmod(pix, i, j);
          obase = std::int64_t(n) * p.Cr * p.Hr * p.Wr;
          hb = int(i) * p.ssh - p.sph;
          wb = int(j) * p.bp * p.ssw - p.spw;
        }
      }
      const std::uint32_t tbase =
          tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t(acc) * acc_cols + std::uint32_t(m * p.BN);
      for (int c0 = 0; c0 < p.BN; c0 += 32) {
        float v[32];
        tmem_ld32(tbase + std::uint32_t(c0), v);
        if (!ok) continue;
        if (p.ph32) {
          const int col0 = nt * p.BN + c0;
          phase_store32(p, obase, col0, min(32, min(p.BN - c0, p.Nout - col0)), hb, wb, v);
          continue;
        }
        if (ptab) {
          const int nv = min(32, min(p.BN - c0, p.Nout - nt * p.BN - c0));
#pragma unroll 4
          for (int j = 0; j < 32; ++j) {
            if (j >= nv) break;
            const int h = hb + ptab_dh[c0 + j], w = wb + ptab_dw[c0 + j];
            if (unsigned(h) >= unsigned(p.Hr) || unsigned(w) >= unsigned(p.Wr)) continue;
            float* dst = p.out + obase + ptab_off[c0 + j] + std::int64_t(h) * p.Wr + w;
            *dst = p.beta == 0.f ? p.alpha * v[j] : p.alpha * v[j] + p.beta * *dst;
          }
          continue;
        }
        if (p.phase) {
#pragma unroll 4
          for (int j = 0; j < 32; ++j) {
            const int col = nt * p.BN + c0 + j;
            if (c0 + j >= p.BN || col >= p.Nout) break;
            phase_store(p, obase, col, hb, wb, p.alpha * v[j]);
          }
          continue;
        }
        {
          const int col0 = nt * p.BN + c0;
          store_row32(p, p.out + obase + std::int64_t(col0) * p.P, min(32, min(p.BN - c0, p.Nout - col0)),
                      std::int64_t(p.P), v);
        }
      }
      }  // sub-tiles
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (p.cps == 2) tmem_free<256>(tmem);
    else tmem_free<512>(tmem);
  }
}


// ---------------------------------------------------------------- 2-SM
// The same implicit GEMM on CTA pairs (cluster of 2) with tcgen05.mma
// cta_group::2: one MMA covers 256 output pixels (128 per CTA, each CTA's
// own TMA im2col box) x BN channels, B split along N (each CTA loads BN/2
// filter rows). Per CTA that halves the filter bytes per MMA and doubles the
// work per MMA instruction, so the same shared-memory ring keeps twice as
// much MMA work in flight -- the ring's round trip (MMA completion ->
// producer -> TMA -> MMA issue) is what bounded the 1-SM kernel. The pair's
// rank 0 issues every MMA; both CTAs' TMA transactions count on rank 0's
// "full" barriers, its commits multicast to both CTAs, and both epilogues
// release the accumulator on rank 0's "tempty" barrier (256 arrivals).
__global__ void __launch_bounds__(kThreads, 1)
    precomp2_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                    const PrecompParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t rank = cluster_rank();
  const int bh = p.BN / 2;  // filter rows per CTA
  const std::uint32_t a_bytes = kBM * 128;
  const std::uint32_t b_bytes = std::uint32_t(bh) * 128;
  // msub == 2: two pair sub-tiles (rows mt*512 + m*256 + rank*128 ..) share
  // each filter box, so a stage carries twice the MMA work for 1.6x the bytes
  const int msub = p.msub;
  const std::uint32_t sub_bytes = msub * a_bytes + ((b_bytes + 1023) & ~1023u);
  const int kSub = p.ksub;
  const std::uint32_t stage_bytes = kSub * sub_bytes;
  const int kStages = p.stages;
  const int jsteps = (p.ksteps + kSub - 1) / kSub;
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
  if (warp == 1) tmem_alloc_2sm<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' barriers initialised before any remote arrive / TMA
  tc_fence_after();
  const std::uint32_t tmem = tmem_base_uniform(tmem_slot);
  const int total_tiles = p.m_tiles * p.n_tiles;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0 || warp == 2 || warp == 3) {
    const int pq = warp == 0 ? 0 : warp - 1;
    const int nprod = kStages < 3 ? kStages : 3;
    if (lane == 0) {
      int it = 0;
      RingOwner ro;
      for (int t = cid; t < total_tiles; t += ncl) {
        int mt, nt;
        tile_coords(p, t, mt, nt);
        int cws[2], chs[2], ns[2];
        for (int m = 0; m < msub; ++m) {
          std::uint32_t n, pix, oh, ow;
          p.fd_P.divmod(std::uint32_t(mt * 2 * msub * kBM + m * 2 * kBM + int(rank) * kBM), n, pix);
          p.fd_OW.divmod(pix, oh, ow);
          cws[m] = int(ow) * p.sw - p.pw;
          chs[m] = int(oh) * p.sh - p.ph;
          ns[m] = int(n);
        }
        const int brow0 = nt * p.ksteps * p.BN + int(rank) * bh;
        for (int j = 0; j < jsteps; ++j, ++it, ro.step(kStages, nprod)) {
          if (ro.own != pq) continue;
          const int s = ro.slot;
          mbar_wait(&empty[s], ro.ph ^ 1);
          const int k0 = j * kSub, nsub = min(kSub, p.ksteps - k0);
          if (rank == 0) mbar_expect_tx(&full[s], 2u * nsub * (msub * a_bytes + b_bytes));
          const std::uint32_t bar = mapa(smem_u32(&full[s]), 0);
          for (int sub = 0; sub < nsub; ++sub) {
            const int k = k0 + sub;
            unsigned char* sa = smem + s * stage_bytes + sub * sub_bytes;
            const int tap = k / p.c_chunks, cc = k - tap * p.c_chunks;
            const int r = tap / p.S, q = tap - r * p.S;
            for (int m = 0; m < msub; ++m)
              tma_im2col_4d_2sm(sa + m * a_bytes, &amap, bar, cc * 32, cws[m], chs[m], ns[m], (unsigned short)q,
                                (unsigned short)r);
            tma_2d_2sm(sa + msub * a_bytes, &bmap, bar, 0, brow0 + k * p.BN);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (rank == 0) {
      // ---------------------------------------------- MMA issuer (pair leader)
      const std::uint32_t idesc = idesc_tf32(2 * kBM, p.BN);
      const std::uint32_t sbase = smem_u32(smem);
      const std::uint64_t da0 = umma_desc_sw128(sbase), db0 = umma_desc_sw128(sbase + msub * a_bytes);
      const int nacc = p.nacc2;
      int it = 0, tl = 0;
    RingPos rp;
      for (int t = cid; t < total_tiles; t += ncl, ++tl) {
        const int acc = tl % nacc, use = tl / nacc;
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const std::uint32_t dtm = tmem + std::uint32_t(acc * msub * p.BN);
        for (int j = 0; j < jsteps; ++j, ++it, rp.step(kStages)) {
          const int s = rp.slot;
          mbar_wait(&full[s], rp.ph);
          tc_fence_after();
          const int k0 = j * kSub, nsub = min(kSub, p.ksteps - k0);
          {  // whole warp, one elected lane issues
            const std::uint32_t so = (std::uint32_t(s) * stage_bytes) >> 4;
            for (int sub = 0; sub < nsub; ++sub) {
              const std::uint32_t o = so + ((std::uint32_t(sub) * sub_bytes) >> 4);
              const std::uint32_t first = (k0 + sub) != 0;
              for (int m = 0; m < msub; ++m) {
                const std::uint32_t oa = o + ((std::uint32_t(m) * a_bytes) >> 4);
                const std::uint32_t dm = dtm + std::uint32_t(m * p.BN);
                mma_tf32_2sm_w(dm, da0 + oa, db0 + o, idesc, first);
                mma_tf32_2sm_w(dm, da0 + oa + 2, db0 + o + 2, idesc, 1u);
                mma_tf32_2sm_w(dm, da0 + oa + 4, db0 + o + 4, idesc, 1u);
                mma_tf32_2sm_w(dm, da0 + oa + 6, db0 + o + 6, idesc, 1u);
              }
            }
            mma_commit_2sm_w(&empty[s], 3);
            if (j == jsteps - 1) mma_commit_2sm_w(&tfull[acc], 3);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue (both CTAs)
    const int ew = warp - 4;
    const std::uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), 0);
    int tl = 0;
    for (int t = cid; t < total_tiles; t += ncl, ++tl) {
      int mt, nt;
      tile_coords(p, t, mt, nt);
      const int acc = tl % p.nacc2, use = tl / p.nacc2;
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      for (int m = 0; m < msub; ++m) {
      const int row = mt * 2 * msub * kBM + m * 2 * kBM + int(rank) * kBM + ew * 32 + lane;
      const bool ok = row < p.M;
      std::int64_t obase = 0;
      int hb = 0, wb = 0;
      if (ok) {
        std::uint32_t n, pix;
        p.fd_P.divmod(std::uint32_t(row), n, pix);
        obase = std::int64_t(n) * p.Nout * p.P + pix;
        if (p.phase) {
          std::uint32_t i, j;
          p.fd_OW.divmod(pix, i, j);
          obase = std::int64_t(n) * p.Cr * p.Hr * p.Wr;
          hb = int(i) * p.ssh - p.sph;
          wb = int(j) * p.bp * p.ssw - p.spw;
        }
      }
      const std::uint32_t tbase =
          tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t((acc * msub + m) * p.BN);
      for (int c0 = 0; c0 < p.BN; c0 += 32) {
        float v[32];
        tmem_ld32(tbase + std::uint32_t(c0), v);
        if (!ok) continue;
        if (p.ph32) {
          const int col0 = nt * p.BN + c0;
          phase_store32(p, obase, col0, min(32, min(p.BN - c0, p.Nout - col0)), hb, wb, v);
          continue;
        }
        if (p.phase) {
#pragma unroll 4
          for (int j = 0; j < 32; ++j) {
            const int col = nt * p.BN + c0 + j;
            if (c0 + j >= p.BN || col >= p.Nout) break;
            phase_store(p, obase, col, hb, wb, p.alpha * v[j]);
          }
          continue;
        }
        {
          const int col0 = nt * p.BN + c0;
          store_row32(p, p.out + obase + std::int64_t(col0) * p.P, min(32, min(p.BN - c0, p.Nout - col0)),
                      std::int64_t(p.P), v);
        }
      }
      }
      tc_fence_before();
      if (rank == 0) mbar_arrive(&tempty[acc]);
      else mbar_arrive_remote(tempty_leader0 + std::uint32_t(acc) * 8);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still signal its barriers
  if (warp == 1) {
    tc_fence_after();
    tmem_free_2sm<512>(tmem);
  }
}

// NCHW -> N(HW)Cp, zero-filling channels C..Cp-1 (32 x 32 smem transpose).
// img: elements between images of src (C * HW, or more for a channel slice)
// 64 pixels x 32 channels per 256-thread block: coalesced 128 B reads along
// pixels, float4 stores of 4 channels (the 32 x 32 / 4-byte-store version
// ran at ~3 TB/s)
__global__ void __launch_bounds__(256) to_nhwc_kernel(const float* __restrict__ src, float* __restrict__ dst, int C,
                                                      int HW, int Cp, std::int64_t img) {
  pdl_wait();
  pdl_trigger();
  __shared__ float tile[32][65];
  const int n = blockIdx.z;
  const int p0 = blockIdx.x * 64, c0 = blockIdx.y * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* s = src + std::int64_t(n) * img;
  float* d = dst + std::int64_t(n) * HW * Cp;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = c0 + warp + 8 * i;
    const float* row = s + std::int64_t(c) * HW;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int pp = p0 + lane + 32 * h;
      tile[warp + 8 * i][lane + 32 * h] = (c < C && pp < HW) ? __ldg(row + pp) : 0.f;
    }
  }
  __syncthreads();
  const int q = threadIdx.x & 7;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int pl = (threadIdx.x >> 3) + 32 * k, pp = p0 + pl;
    if (pp < HW && c0 + 4 * q < Cp)
      *reinterpret_cast<float4*>(d + std::int64_t(pp) * Cp + c0 + 4 * q) =
          make_float4(tile[4 * q][pl], tile[4 * q + 1][pl], tile[4 * q + 2][pl], tile[4 * q + 3][pl]);
  }
}

// Space-to-depth for strided Forward: x (NCHW) -> xs[n][i][j][Cp] with
// channel cc = (a*Bw + b)*C + c holding x[n][c][i*sh + a - ph][j*sw + b - pw]
// (0 off the image or for cc >= Ah*Bw*C). 32 x 32 smem transpose per block.
struct S2D {
  int C, H, W, sh, sw, ph, pw, Bw, CC, Hq, Wq, Cp;
};
__global__ void s2d_nhwc_kernel(const float* __restrict__ x, float* __restrict__ out, S2D d) {
  pdl_wait();
  pdl_trigger();
  __shared__ float tile[32][33];
  const int n = blockIdx.z / d.Hq, i = blockIdx.z - n * d.Hq;
  const int j0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int iy = threadIdx.y; iy < 32; iy += blockDim.y) {
    const int cc = c0 + iy, j = j0 + threadIdx.x;
    float v = 0.f;
    if (cc < d.CC && j < d.Wq) {
      const int ab = cc / d.C, c = cc - ab * d.C, a = ab / d.Bw, b = ab - a * d.Bw;
      const int h = i * d.sh + a - d.ph, w = j * d.sw + b - d.pw;
      if (unsigned(h) < unsigned(d.H) && unsigned(w) < unsigned(d.W))
        v = __ldg(x + ((std::int64_t(n) * d.C + c) * d.H + h) * d.W + w);
    }
    tile[iy][threadIdx.x] = v;
  }
  __syncthreads();
  float* o = out + (std::int64_t(n) * d.Hq + i) * d.Wq * d.Cp;
  for (int iy = threadIdx.y; iy < 32; iy += blockDim.y) {
    const int j = j0 + iy, cc = c0 + threadIdx.x;
    if (j < d.Wq && cc < d.Cp) o[std::int64_t(j) * d.Cp + cc] = tile[threadIdx.x][iy];
  }
}

// The same copy one output row (n, i) per block: the Ah input rows of each
// channel it needs are read whole (coalesced, zero-padded to Wq*sw columns)
// into shared memory, then the [Wq][Cp] output row is written contiguously.
// The 32 x 32 tile version reads x at stride sw along a warp (4x the sectors
// for AlexNet conv1: 67 us per 64 images, ~1.4 TB/s).
// Per-geometry constants of the row copy, computed on the host: the smem
// offset of channel cc's (c, a, b) source within a row group (-1: zero
// channel), so no thread divides (the per-thread decode was ~40 % of the
// instructions of this issue-bound kernel).
struct S2DTab {
  int Ah, Lp;
  short off[256];
};
// MinB = 6: 40 registers, six blocks per SM (the unbounded build used 60,
// four blocks, for an issue-bound copy)
template <int MinB>
__global__ void __launch_bounds__(256, MinB)
    s2d_rows_kernel(const float* __restrict__ x, float* __restrict__ out, S2D d, const __grid_constant__ S2DTab tab) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float rows[];  // [c][a][Wq * sw]
  const int n = blockIdx.x / d.Hq, i = blockIdx.x - n * d.Hq;
  // odd row pitch: the write phase reads rows (c, a) that differ by whole
  // rows, which would otherwise land on the same banks
  const int Ah = tab.Ah, L = d.Wq * d.sw, Lp = tab.Lp;
  // load: thread t takes column t of all C*Ah (<= 16) rows, every load
  // issued before the first smem store (a loop of load -> store per row
  // exposed one DRAM latency per row: 44 us per 64 AlexNet images)
  const int nr = d.C * Ah;
  // (only when every input column lands inside the row: with kernel ==
  // stride and W not a multiple of it, trailing columns no window reads
  // would run past the row pitch; the scalar loop below only writes t < L)
  if ((d.W & 3) == 0 && (reinterpret_cast<std::uintptr_t>(x) & 15) == 0 && d.pw + d.W <= L) {
    // float4 loads along w (the scalar loop below was issue-bound: 77 %
    // issue-active, ~1000 instructions per warp for AlexNet conv1); padding
    // columns and rows outside the image are zero-filled separately
    const int W4 = d.W >> 2, items = nr * W4, tail = L - d.pw - d.W;
    // four float4 loads in flight per thread before their smem stores (a
    // load -> store loop left one DRAM latency exposed per iteration); the
    // row bases come from a per-block table and (row, column) advance by
    // adds (two integer divisions per item made the copy issue-bound: 73 %
    // issue-active at ~2.3 TB/s for AlexNet conv1)
    __shared__ const float4* rowp[16];
    if (threadIdx.x < nr) {
      const int c = threadIdx.x / Ah, a = threadIdx.x - c * Ah;
      const int h = i * d.sh + a - d.ph;
      rowp[threadIdx.x] = unsigned(h) < unsigned(d.H)
                              ? reinterpret_cast<const float4*>(x + ((std::int64_t(n) * d.C + c) * d.H + h) * d.W)
                              : nullptr;
    }
    __syncthreads();
    constexpr int kU = 4;
    const int dk = blockDim.x / W4, dt = blockDim.x - dk * W4;
    int k = threadIdx.x / W4, t4 = threadIdx.x - k * W4;
    for (int base = 0; base < items; base += kU * blockDim.x) {
      float4 v[kU];
      int dst[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        dst[u] = -1;
        if (k < nr) {
          const float4* rp = rowp[k];
          if (rp) v[u] = __ldg(rp + t4);
          dst[u] = k * Lp + d.pw + 4 * t4;
        }
        t4 += dt;
        k += dk;
        if (t4 >= W4) {
          t4 -= W4;
          ++k;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (dst[u] >= 0) {
          float* r = rows + dst[u];
          r[0] = v[u].x;
          r[1] = v[u].y;
          r[2] = v[u].z;
          r[3] = v[u].w;
        }
    }
    const int pads = d.pw + (tail > 0 ? tail : 0);
    for (int idx = threadIdx.x; idx < nr * pads; idx += blockDim.x) {
      const int k = idx / pads, t = idx - k * pads;
      rows[k * Lp + (t < d.pw ? t : d.W + t)] = 0.f;
    }
  } else
  for (int t = threadIdx.x; t < L; t += blockDim.x) {
    const int w = t - d.pw;
    const bool win = unsigned(w) < unsigned(d.W);
    float v[16];
    int c = 0, a = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      v[k] = 0.f;
      if (k < nr) {
        const int h = i * d.sh + a - d.ph;
        if (win && unsigned(h) < unsigned(d.H)) v[k] = __ldg(x + ((std::int64_t(n) * d.C + c) * d.H + h) * d.W + w);
        if (++a == Ah) {
          a = 0;
          ++c;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < nr) rows[k * Lp + t] = v[k];
  }
  __syncthreads();
  // write: each thread owns 4 consecutive channels (one float4 store) for
  // every (256*4/Cp)-th column j; the (a, b, c) decode happens once
  const int c4 = d.Cp >> 2;  // Cp is a power of two here (1024 % Cp == 0)
  const int q4 = threadIdx.x & (c4 - 1), j0 = threadIdx.x / c4, js = blockDim.x / c4;
  int off[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) off[e] = tab.off[4 * q4 + e];
  float4* o = reinterpret_cast<float4*>(out + (std::int64_t(n) * d.Hq + i) * d.Wq * d.Cp) + q4 + j0 * c4;
  const int ostep = js * c4, jstep = js * d.sw;
  for (int j = j0, jo = j0 * d.sw; j < d.Wq; j += js, jo += jstep, o += ostep)
    *o = make_float4(off[0] >= 0 ? rows[off[0] + jo] : 0.f, off[1] >= 0 ? rows[off[1] + jo] : 0.f,
                     off[2] >= 0 ? rows[off[2] + jo] : 0.f, off[3] >= 0 ? rows[off[3] + jo] : 0.f);
}
std::size_t s2d_rows_smem(const S2D& d) {
  return std::size_t(d.CC / (d.Bw * d.C)) * d.C * ((d.Wq * d.sw) | 1) * 4;
}
// space-to-depth launch: the row kernel when its rows fit in 48 KB
cudaError_t launch_s2d(const float* x, float* out, const S2D& d, int N, cudaStream_t st) {
  const std::size_t sm = s2d_rows_smem(d);
  if (sm <= 48 * 1024 && d.Cp % 4 == 0 && 1024 % d.Cp == 0 && d.Cp <= 256 && d.CC / d.Bw <= 16 &&
      tune("s2d_rows", 1)) {
    S2DTab tab{};
    tab.Ah = d.CC / (d.Bw * d.C);
    tab.Lp = (d.Wq * d.sw) | 1;
    for (int cc = 0; cc < d.Cp; ++cc) {
      tab.off[cc] = -1;
      if (cc < d.CC) {
        const int ab = cc / d.C, c = cc - ab * d.C, aa = ab / d.Bw, bb = ab - aa * d.Bw;
        tab.off[cc] = short((c * tab.Ah + aa) * tab.Lp + bb);
      }
    }
    return tune("s2d_minb", 6) == 6
               ? launch_pdl(s2d_rows_kernel<6>, dim3(N * d.Hq), dim3(256), sm, st, x, out, d, tab)
               : launch_pdl(s2d_rows_kernel<1>, dim3(N * d.Hq), dim3(256), sm, st, x, out, d, tab);
  }
  return launch_pdl(s2d_nhwc_kernel, dim3((d.Wq + 31) / 32, (d.Cp + 31) / 32, N * d.Hq), dim3(32, 8), 0, st, x,
                    out, d);
}

// Filter -> B tiles [n_tile][kstep][BN rows][32 floats, SWIZZLE_128B]. Output channel o,
// reduction (tap, ch). Forward: W[o][ch][tap]; flip_transpose (stride-1
// BackwardData): W[ch][o][taps-1-tap] with rows o over C and ch over K;
// phase (strided BackwardData): o = (a, b, c), tap = (t, u) of a Th x Tw
// grid, ch = k -> W[k][c][a + (Th-1-t)*sh][b + (Tw-1-u)*sw] (0 off the filter).
struct PhaseFilter {
  int C, R, S, sh, sw, Tw;
  int bw = 0;  // stride-phase BD: phases kept along w (decode divisor of the column index)
  int P = 1;   // stride-phase BD blocked along w: P phase-grid columns per GEMM row
};
// ldi: input-channel pitch of w in Forward (flip 0) mode (I, or the full C
// for a channel slice)
__global__ void pack_filter_kernel(const float* __restrict__ w, float* __restrict__ out, int O, int I, int taps,
                                   int BN, int n_tiles, int ksteps, int small_c, int c_chunks, int flip,
                                   PhaseFilter pf, int swz, int ldi) {
  pdl_wait();
  pdl_trigger();
  // blockIdx.x = (column tile, k-step): BN rows x 8 16-byte chunks, spread
  // over gridDim.y blocks (one item per thread: the filter gather is
  // latency-bound, 50 single blocks took 7-12 us for a 1 MB filter)
  const int nt = blockIdx.x / ksteps, k = blockIdx.x - nt * ksteps;
  for (int idx = threadIdx.x + blockIdx.y * blockDim.x; idx < 8 * BN; idx += blockDim.x * gridDim.y) {
    const int row = idx >> 3, g = idx & 7;  // a row's 8 chunks from 8 adjacent threads: 128 B stores
    const std::int64_t u = (std::int64_t(blockIdx.x) * 8 + g) * BN + row;
    const int o = nt * BN + row;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      int tap, ch;
      if (small_c == 1) {
        tap = k * 8 + g;
        ch = e;
      } else if (small_c == 2) {  // strip kernel: k = chunk * taps + tap
        const int cc = k / taps;
        tap = k - cc * taps;
        ch = cc * 32 + g * 4 + e;
      } else {
        tap = k / c_chunks;
        ch = (k - tap * c_chunks) * 32 + g * 4 + e;
      }
      float x = 0.f;
      if (o < O && ch < I && tap < taps) {
        if (flip == 3) {  // space-to-depth Forward: o = k, tap = (t, u), ch = (a, b, c)
          const int ab = ch / pf.C, c = ch - ab * pf.C, a = ab / pf.sw, b = ab - a * pf.sw;
          const int t = tap / pf.Tw, u = tap - t * pf.Tw;
          const int r = t * pf.sh + a, q = u * pf.sw + b;
          if (a < pf.sh && r < pf.R && q < pf.S) x = w[((std::int64_t(o) * pf.C + c) * pf.R + r) * pf.S + q];
        } else if (flip == 2) {
          // column (pb, a, b, c), tap (t, u') of a Th x (Tw + P - 1) window:
          // phase-grid column pb of the block uses sub-filter tap u = u' - pb
          const int Twb = pf.Tw + pf.P - 1, nab = (o / pf.C) , Ah = min(pf.sh, pf.R);
          const int pb = nab / (Ah * pf.bw), ab = nab - pb * (Ah * pf.bw), c = o - nab * pf.C;
          const int a = ab / pf.bw, b = ab - a * pf.bw;
          const int t = tap / Twb, u = tap - t * Twb - pb, Th = taps / Twb;
          const int r = a + (Th - 1 - t) * pf.sh, q = b + (pf.Tw - 1 - u) * pf.sw;
          if (u >= 0 && u < pf.Tw && r < pf.R && q < pf.S)
            x = w[((std::int64_t(ch) * pf.C + c) * pf.R + r) * pf.S + q];
        } else {
          x = flip ? w[(std::int64_t(ch) * O + o) * taps + (taps - 1 - tap)]
                   : w[(std::int64_t(o) * ldi + ch) * taps + tap];
        }
      }
      v[e] = x;
    }
    // SWIZZLE_128B K-major block: row `row` holds its 8 16-byte chunks at
    // positions g ^ (row & 7) (the pattern TMA writes and UMMA reads)
    const std::int64_t blk = u / (8 * BN);
    // swz == 0: plain rows, for a TMA load that applies the swizzle itself
    reinterpret_cast<float4*>(out)[blk * 8 * BN + row * 8 + (swz ? (g ^ (row & 7)) : g)] =
        make_float4(v[0], v[1], v[2], v[3]);
  }
}


// ---------------------------------------------------------------- strip
// Stride-1 implicit GEMM that loads each input pixel once per 32-channel
// chunk instead of once per filter tap. The (padded, channels-last) input is
// read as a flat [rows = (n, h, w)][C] matrix with the padded row pitch Wp,
// and output pixel (oh, ow) of image n is flat position p = n*Hp*Wp + oh*Wp +
// ow (positions with ow >= OW or oh >= OH are computed and dropped). Tap
// (r, s) of positions [p0, p0+128) then reads input rows [p0 + r*Wp + s, ...),
// so one TMA "strip" of 128 + (R-1)*Wp + (S-1) rows per chunk feeds every tap:
// the UMMA descriptor simply starts r*Wp + s rows (x 128 B) into the strip --
// SWIZZLE_128B is a function of the absolute smem address, so any 128-byte
// row start is legal (scripts/offset_probe.cu). Compared with one TMA im2col
// box per (tap, chunk) this cuts the operand traffic from L2 by ~R*S for A.
//
// Roles: warp 3 lane 0 streams strips into a double buffer; warps 0 and 2
// stream the filter chunks of two taps per stage (8 MMAs per commit); warp 1
// issues tcgen05.mma; warps 4-7 run the epilogue (NCHW or stride-phase
// scatter) while the next tile accumulates in the other TMEM buffer.
constexpr int kTapsPerStage = 2;

struct StripParams {
  const float* btiles;  // [n_tile][chunk][tap][BN rows][32 floats, SW128]
  float* out;
  float alpha, beta;
  int BN, n_tiles, m_tiles, nimg;  // m_tiles: flat position tiles over all images
  int taps, S, c_chunks, Wp, HWp;
  int OH, OW, Nout, P;
  int box_rows, nboxes, stages;
  int phase, Cr, Hr, Wr, ssh, ssw, sph, spw;
  int sAh, sBw, pair, bp, ph32;
  FastDiv fd_blk;
  FastDiv fd_Cr, fd_ssw, fd_Wp, fd_HWp, fd_mt;
  int swap;  // 1: MMA rows = output channels (<= 128), N = 256 strip positions
  int msub;  // swap == 0: 128-position MMA sub-tiles per tile sharing each filter stage (1 .. 4)
  int prof;  // UCUDNN_TUNE=prof=1: MMA-warp cycle split into g_prof (strip wait, stage wait, acc wait, total);
             // prof=2: epilogue busy, last epilogue, TMEM-load share, whole CTA
  int nsb;   // strip buffers (2; 1 when a wide tile's strip would leave too few filter stages)
};

__global__ void __launch_bounds__(kThreads, 1)
    strip_kernel(const __grid_constant__ CUtensorMap xmap, const StripParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const long long t_entry = p.prof == 2 ? clock64() : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t strip_bytes = std::uint32_t(p.nboxes * p.box_rows) * 128;
  const std::uint32_t tap_bytes = std::uint32_t(p.BN) * 128;  // swap: BN = 128 filter rows
  const int tile_pos = p.swap ? 2 * kBM : p.msub * kBM;
  const std::uint32_t stage_bytes = kTapsPerStage * tap_bytes;
  const int kStages = p.stages;
  unsigned char* strips = smem;
  unsigned char* ring = smem + p.nsb * strip_bytes;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(ring + kStages * stage_bytes);
  std::uint64_t* empty = full + kMaxStages;
  std::uint64_t* sfull = empty + kMaxStages;
  std::uint64_t* sempty = sfull + 2;
  std::uint64_t* tfull = sempty + 2;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  float* xpose = reinterpret_cast<float*>(ring + kStages * stage_bytes + 256);  // swap epilogue: 4 x 32 x 33
  __shared__ std::uint32_t toff[64];  // tap -> strip row offset (r * Wp + s) in descriptor units (16 B)
  for (int tap = threadIdx.x; tap < p.taps && tap < 64; tap += blockDim.x) {
    const int r = tap / p.S, q = tap - r * p.S;
    toff[tap] = std::uint32_t(r * p.Wp + q) * 8;
  }
  if (threadIdx.x == 0) {
    prefetch_tmap(&xmap);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&sfull[a], 1);
      mbar_init(&sempty[a], 1);
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = tmem_base_uniform(tmem_slot);
  pdl_wait();  // everything above touched only smem / TMEM / the param-space tensor map
  pdl_trigger();
  const int total_tiles = p.m_tiles * p.n_tiles;
  const int tsteps = (p.taps + kTapsPerStage - 1) / kTapsPerStage;  // filter stages per chunk

  if (warp == 3) {
    if (lane == 0) {
      // ------------------------------------------------ strip producer
      int sc = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        std::uint32_t nt, mt;
        p.fd_mt.divmod(std::uint32_t(t), nt, mt);
        const int p0 = int(mt) * tile_pos;  // tiles run over the flat (n, hp, wp) rows, across images
        for (int cc = 0; cc < p.c_chunks; ++cc, ++sc) {
          const int sb = sc % p.nsb;
          mbar_wait(&sempty[sb], ((sc / p.nsb) & 1) ^ 1);
          mbar_expect_tx(&sfull[sb], strip_bytes);
          for (int bx = 0; bx < p.nboxes; ++bx)
            tma_2d(strips + sb * strip_bytes + bx * p.box_rows * 128, &xmap, &sfull[sb], cc * 32,
                   p0 + bx * p.box_rows);
        }
      }
    }
    __syncwarp();
  } else if (warp == 0 || warp == 2) {
    // ------------------------------------------------ filter producers
    const int pq = warp == 0 ? 0 : 1, nprod = kStages < 2 ? 1 : 2;
    if (lane == 0) {
      int it = 0;
      RingOwner ro;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const int nt = t / p.m_tiles;
        const float* bsrc = p.btiles + std::size_t(nt) * p.c_chunks * p.taps * (tap_bytes / 4);
        for (int cc = 0; cc < p.c_chunks; ++cc)
          for (int ts = 0; ts < tsteps; ++ts, ++it, ro.step(kStages, nprod)) {
            if (ro.own != pq) continue;
            const int st = ro.slot;
            const int tap0 = ts * kTapsPerStage, ntap = min(kTapsPerStage, p.taps - tap0);
            mbar_wait(&empty[st], ro.ph ^ 1);
            mbar_expect_tx(&full[st], ntap * tap_bytes);
            for (int i = 0; i < ntap; ++i)
              bulk_g2s(ring + st * stage_bytes + i * tap_bytes,
                       bsrc + (std::size_t(cc) * p.taps + tap0 + i) * (tap_bytes / 4), tap_bytes, &full[st]);
          }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const std::uint32_t idesc = idesc_tf32(kBM, p.swap ? 2 * kBM : p.BN);
    const std::uint32_t sbase = smem_u32(strips), rbase = smem_u32(ring);
    int it = 0, sc = 0, tl = 0;
    RingPos rp;
    long long c_strip = 0, c_stage = 0, c_acc = 0, t_start = clock64(), cq = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++tl) {
      const int acc = tl & 1;
      if (p.prof) cq = clock64();
      mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
      if (p.prof) c_acc += clock64() - cq;
      tc_fence_after();
      const std::uint32_t dtm = tmem + std::uint32_t(acc * kMaxBN);
      for (int cc = 0; cc < p.c_chunks; ++cc, ++sc) {
        const int sb = sc % p.nsb;
        if (p.prof) cq = clock64();
        mbar_wait(&sfull[sb], (sc / p.nsb) & 1);
        if (p.prof) c_strip += clock64() - cq;
        tc_fence_after();
        for (int ts = 0; ts < tsteps; ++ts, ++it, rp.step(kStages)) {
          const int st = rp.slot;
          const int tap0 = ts * kTapsPerStage, ntap = min(kTapsPerStage, p.taps - tap0);
          if (p.prof) cq = clock64();
          mbar_wait(&full[st], rp.ph);
          if (p.prof) c_stage += clock64() - cq;
          tc_fence_after();
          if (p.swap) {  // whole warp, one elected lane issues
            for (int i = 0; i < ntap; ++i) {
              const int tap = tap0 + i;
              const std::uint32_t sa = sbase + sb * strip_bytes + toff[tap] * 16;
              const std::uint32_t sbb = rbase + st * stage_bytes + i * tap_bytes;
#pragma unroll
              for (int k = 0; k < 4; ++k)  // A = filter rows, B = 256 strip positions
                mma_tf32_w(dtm, umma_desc_sw128(sbb + k * 32), umma_desc_sw128(sa + k * 32), idesc, (cc | tap | k) != 0);
            }
          } else {
            // descriptors are the strip / stage bases plus offsets: straight-line issue
            const std::uint64_t ad0 = umma_desc_sw128(sbase + sb * strip_bytes);
            const std::uint64_t bd0 = umma_desc_sw128(rbase + st * stage_bytes);
#pragma unroll
            for (int i = 0; i < kTapsPerStage; ++i) {
              if (i >= ntap) break;
              const int tap = tap0 + i;
              const std::uint64_t ad = ad0 + toff[tap];
              const std::uint64_t bd = bd0 + std::uint32_t(i) * (tap_bytes >> 4);
              for (int m = 0; m < p.msub; ++m) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  mma_tf32_w(dtm + std::uint32_t(m * p.BN), ad + std::uint32_t(m * kBM * 8 + 2 * k), bd + 2 * k, idesc,
                             (cc | tap | k) != 0);
              }
            }
          }
          {
            mma_commit_w(&empty[st]);
            if (ts == tsteps - 1) mma_commit_w(&sempty[sb]);
            if (ts == tsteps - 1 && cc == p.c_chunks - 1) mma_commit_w(&tfull[acc]);
          }
          __syncwarp();
        }
      }
    }
    if (p.prof == 1 && lane == 0 && blockIdx.x < 1024) {
      g_prof[blockIdx.x * 4 + 0] = c_strip + c_stage;
      g_prof[blockIdx.x * 4 + 1] = c_stage;
      g_prof[blockIdx.x * 4 + 2] = c_acc;
      g_prof[blockIdx.x * 4 + 3] = clock64() - t_start;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue
    const int ew = warp - 4;
    int tl = 0;
    long long e_busy = 0, e_last = 0, e_t = 0, e_ld = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++tl) {
      if (p.prof == 2 && tl > 0) {
        e_last = clock64() - e_t;
        e_busy += e_last;
      }
      std::uint32_t nt, mt;
      p.fd_mt.divmod(std::uint32_t(t), nt, mt);
      const int acc = tl & 1;
      mbar_wait(&tfull[acc], (tl >> 1) & 1);
      if (p.prof == 2) e_t = clock64();
      tc_fence_after();
      if (p.swap) {
        // TMEM lane = output channel, column = position: stage 32 x 32
        // blocks through smem so the stores run along positions
        float* tp = xpose + ew * (32 * 33);
        const std::uint32_t tb = tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t(acc * kMaxBN);
        for (int c0 = 0; c0 < 2 * kBM; c0 += 32) {
          float v[32];
          tmem_ld32(tb + std::uint32_t(c0), v);
#pragma unroll
          for (int j = 0; j < 32; ++j) tp[lane * 33 + j] = v[j];
          __syncwarp();
          const int pos = int(mt) * tile_pos + c0 + lane;
          std::uint32_t n, rem, oh, ow;
          p.fd_HWp.divmod(std::uint32_t(pos), n, rem);
          p.fd_Wp.divmod(rem, oh, ow);
          if (int(n) < p.nimg && int(oh) < p.OH && int(ow) < p.OW) {
            if (!p.phase) {
              float* base = p.out + std::int64_t(n) * p.Nout * p.P + int(oh) * p.OW + int(ow);
              for (int r = 0; r < 32; ++r) {
                const int col = ew * 32 + r;
                if (col >= p.Nout) break;
                float* dst = base + std::int64_t(col) * p.P;
                const float val = p.alpha * tp[r * 33 + lane];
                *dst = p.beta == 0.f ? val : val + p.beta * *dst;
              }
            } else {
              const std::int64_t obase = std::int64_t(n) * p.Cr * p.Hr * p.Wr;
              const int hb = int(oh) * p.ssh - p.sph, wb = int(ow) * p.bp * p.ssw - p.spw;
              for (int r = 0; r < 32; ++r) {
                const int col = ew * 32 + r;
                if (col >= p.Nout) break;
                phase_store(p, obase, col, hb, wb, p.alpha * tp[r * 33 + lane]);
              }
            }
          }
          __syncwarp();
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        continue;
      }
      for (int m = 0; m < p.msub; ++m) {
      const int pos = int(mt) * tile_pos + m * kBM + ew * 32 + lane;  // flat (n, hp, wp) position
      std::uint32_t n, rem, oh, ow;
      p.fd_HWp.divmod(std::uint32_t(pos), n, rem);
      p.fd_Wp.divmod(rem, oh, ow);
      const bool ok = int(n) < p.nimg && int(oh) < p.OH && int(ow) < p.OW;
      std::int64_t obase = 0;
      int hb = 0, wb = 0;
      if (ok) {
        if (p.phase) {
          obase = std::int64_t(n) * p.Cr * p.Hr * p.Wr;
          hb = int(oh) * p.ssh - p.sph;
          wb = int(ow) * p.bp * p.ssw - p.spw;
        } else {
          obase = std::int64_t(n) * p.Nout * p.P + int(oh) * p.OW + int(ow);
        }
      }
      const std::uint32_t tbase =
          tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t(acc * kMaxBN + m * p.BN);
      for (int c0 = 0; c0 < p.BN; c0 += 32) {
        float v[32];
        const long long tq = p.prof == 2 ? clock64() : 0;
        tmem_ld32(tbase + std::uint32_t(c0), v);
        if (p.prof == 2) e_ld += clock64() - tq;
        if (!ok) continue;
        if (p.ph32) {
          const int col0 = int(nt) * p.BN + c0;
          phase_store32(p, obase, col0, min(32, min(p.BN - c0, p.Nout - col0)), hb, wb, v);
          continue;
        }
        if (p.phase) {
#pragma unroll 4
          for (int j = 0; j < 32; ++j) {
            const int col = int(nt) * p.BN + c0 + j;
            if (c0 + j >= p.BN || col >= p.Nout) break;
            phase_store(p, obase, col, hb, wb, p.alpha * v[j]);
          }
          continue;
        }
        {
          const int col0 = int(nt) * p.BN + c0;
          store_row32(p, p.out + obase + std::int64_t(col0) * p.P, min(32, min(p.BN - c0, p.Nout - col0)),
                      std::int64_t(p.P), v);
        }
      }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
    if (p.prof == 2 && ew == 0 && lane == 0 && blockIdx.x < 1024) {  // epilogue busy, last epilogue
      if (tl > 0) {
        e_last = clock64() - e_t;
        e_busy += e_last;
      }
      g_prof[blockIdx.x * 4 + 0] = e_busy;
      g_prof[blockIdx.x * 4 + 1] = e_last;
      g_prof[blockIdx.x * 4 + 2] = e_ld;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (p.prof == 2 && threadIdx.x == 0 && blockIdx.x < 1024) {
    g_prof[blockIdx.x * 4 + 3] = clock64() - t_entry;
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// NCHW -> zero-padded channels-last [n][Hp][Wp][Cp] (source pixel (h, w)
// lands at (h + pt, w + pl)); 32 x 33 smem transpose per (n, row, 32-pixel
// block, 32-channel block), 128 threads: eight independent loads per thread in
// flight and 16-byte stores (8 lanes per pixel's 128-byte channel run).
__global__ void __launch_bounds__(128) pad_nhwc_kernel(const float* __restrict__ src, float* __restrict__ dst, int C,
                                                       int H, int W, int Cp, int pt, int pl, int Hp, int Wp) {
  pdl_wait();
  pdl_trigger();
  __shared__ float tile[32][33];
  const int n = blockIdx.z / Hp, hp = blockIdx.z - n * Hp;
  const int w0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = hp - pt, w = w0 + lane - pl;
  const bool row_ok = unsigned(h) < unsigned(H) && unsigned(w) < unsigned(W) && w0 + lane < Wp;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = c0 + warp + 4 * i;
    tile[warp + 4 * i][lane] = (row_ok && c < C) ? __ldg(src + ((std::int64_t(n) * C + c) * H + h) * W + w) : 0.f;
  }
  __syncthreads();
  float* o = dst + (std::int64_t(n) * Hp + hp) * Wp * Cp;
  const int q = threadIdx.x & 7;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int px = (threadIdx.x >> 3) + 16 * k, wp = w0 + px;
    if (wp < Wp)
      *reinterpret_cast<float4*>(o + std::int64_t(wp) * Cp + c0 + 4 * q) =
          make_float4(tile[4 * q][px], tile[4 * q + 1][px], tile[4 * q + 2][px], tile[4 * q + 3][px]);
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
  int ph_hi = -1, pw_hi = -1;  // high-side padding (default: = ph / pw)
  int phase = 0;               // 1: strided BackwardData phase scatter
  int s2d = 0;                 // 1: strided Forward on a space-to-depth copy
  S2D sd{};
  PhaseFilter pf{};
  int Hr = 0, Wr = 0, rph = 0, rpw = 0;  // the real dx extent and conv padding
};

// 1x1 stride-2 unpadded BackwardData over even dx extents: each GEMM pixel
// owns a whole 2x2 dx block (phase_store's float2 path).
int phase_pair(const Geo& g) {
  return g.phase && g.pf.sh == 2 && g.pf.sw == 2 && g.pf.R == 1 && g.pf.S == 1 && g.rph == 0 && g.rpw == 0 &&
         g.Hr % 2 == 0 && g.Wr % 2 == 0 && g.Hout * 2 == g.Hr && g.Wout * 2 == g.Wr && tune("pair", 1);
}

// Strip path (stride-1 after the s2d / phase rewrites, >= 32-channel rows):
// geometry of the padded input and of the per-chunk strip.
struct StripGeo {
  bool ok = false, swap = false;
  int msub = 1, nsb = 2;
  int Hp = 0, Wp = 0, rows = 0, box_rows = 0, nboxes = 0, stages = 0;
  std::size_t strip_bytes = 0;
};
// Few output channels (<= 128): swapped roles -- 256 strip positions as the
// MMA N, output channels (zero-padded to 128) as its M -- so each MMA does
// 4x the work of a 128 x 64 one at about the same issue cost.
// (Measured, AlexNet at 64 images: conv2 BD 191 -> 179 us, conv1 F 148 -> 142
// us; the stride-phase BD of conv1 gets slower, 124 -> 222 us, so phase
// scatters stay on the im2col kernel.)
bool strip_swap(const Geo& g) {
  // Off by default since the implicit GEMM runs two CTAs per SM: that
  // measured faster for these shapes (conv2 BD 157 vs 179 us, conv1 F 132 vs
  // 142 us). UCUDNN_TUNE=sswap=1 turns it back on.
  return g.sh == 1 && g.sw == 1 && cpad(g.Cin) != 4 && g.Nout <= 128 && !g.phase && tune("sswap", 0);
}
int filter_rows(const Geo& g) { return strip_swap(g) ? kBM : pick_bn(g.Nout); }
StripGeo strip_geo(const Geo& g, int BN) {
  StripGeo sg;
  sg.swap = strip_swap(g);
  if (g.sh != 1 || g.sw != 1 || cpad(g.Cin) == 4 || !(sg.swap || tune("strip", 0))) return sg;
  sg.Hp = g.Hin + g.ph + (g.ph_hi < 0 ? g.ph : g.ph_hi);
  sg.Wp = g.Win + g.pw + (g.pw_hi < 0 ? g.pw : g.pw_hi);
  if (sg.Hp - g.R + 1 != g.Hout || sg.Wp - g.S + 1 != g.Wout) return sg;
  sg.msub = sg.swap ? 1 : std::max(1, std::min(std::min(4, tune("strip_msub", 2)), 256 / std::max(BN, 1)));
  sg.rows = (sg.swap ? 2 * kBM : sg.msub * kBM) + (g.R - 1) * sg.Wp + (g.S - 1);
  sg.nboxes = (sg.rows + 255) / 256;  // TMA boxes of <= 256 rows, split evenly (8-row multiples)
  sg.box_rows = ((sg.rows + sg.nboxes - 1) / sg.nboxes + 7) / 8 * 8;
  sg.strip_bytes = std::size_t(sg.nboxes) * sg.box_rows * 128;
  const std::size_t stage = std::size_t(kTapsPerStage) * BN * 128;
  // 227 KB per CTA less the 1 KB alignment slack, the barrier block and the
  // static tap table
  const std::size_t budget = 232448 - 1024 - 256 - 256 - (sg.swap ? 4 * 32 * 33 * 4 : 0);
  // two strip buffers unless that leaves fewer than 3 filter stages
  // (strip_minst): one buffer stalls each chunk change (AlexNet conv2 BD at
  // 64 images, 4 sub-tiles: 553 -> 528 us per 256 images with two buffers and
  // 3 stages; ResNet 3x3 64-channel BD 348 -> 323)
  sg.nsb = 2;
  if ((budget - std::min(budget, 2 * sg.strip_bytes)) / stage < std::size_t(tune("strip_minst", 3)) &&
      tune("strip_nsb", 0) != 2)
    sg.nsb = 1;
  if (sg.nsb * sg.strip_bytes + 2 * stage > budget) return sg;
  sg.stages = int(std::min<std::size_t>(kMaxStages, (budget - sg.nsb * sg.strip_bytes) / stage));
  sg.ok = true;
  return sg;
}

std::size_t geo_ws(const Geo& g, int* ksteps_out = nullptr, int* bn_out = nullptr) {
  const int Cp = cpad(g.Cin), taps = g.R * g.S;
  const bool small = Cp == 4;
  const int ksteps = small ? (taps + 7) / 8 : taps * (Cp / 32);
  const int BN = filter_rows(g), n_tiles = (g.Nout + BN - 1) / BN;
  if (ksteps_out) *ksteps_out = ksteps;
  if (bn_out) *bn_out = BN;
  const StripGeo sg = strip_geo(g, BN);
  const std::size_t act = sg.ok ? std::size_t(g.N) * sg.Hp * sg.Wp * Cp * 4 : std::size_t(g.N) * g.Hin * g.Win * Cp * 4;
  return align256(std::size_t(n_tiles) * ksteps * BN * 128) + align256(act);
}

cudaError_t run_strip(const Geo& g, const StripGeo& sg, const float* act, const float* w, int flip, float* out,
                      void* ws, float alpha, float beta, cudaStream_t st, int flags) {
  const int Cp = cpad(g.Cin), taps = g.R * g.S;
  int ksteps = 0, BN = 0;
  geo_ws(g, &ksteps, &BN);
  const int n_tiles = (g.Nout + BN - 1) / BN;
  float* btiles = static_cast<float*>(ws);
  float* xp = reinterpret_cast<float*>(static_cast<char*>(ws) + align256(std::size_t(n_tiles) * ksteps * BN * 128));
  cudaError_t e;
  if (g.s2d) {
    S2D d = g.sd;
    d.Cp = Cp;
    e = launch_s2d(act, xp, d, g.N, st);
  } else {
    e = launch_pdl(pad_nhwc_kernel, dim3((sg.Wp + 31) / 32, Cp / 32, g.N * sg.Hp), dim3(128), 0, st, act, xp,
                   g.Cin, g.Hin, g.Win, Cp, g.ph, g.pw, sg.Hp, sg.Wp);
  }
  if (e != cudaSuccess) return e;
  if (!(flags & kFilterReady)) {
    e = launch_pdl(pack_filter_kernel, dim3(n_tiles * ksteps, (8 * BN + 255) / 256), dim3(256), 0, st, w, btiles, g.Nout, g.Cin, taps, BN,
                   n_tiles,
                   ksteps, 2, Cp / 32, g.s2d ? 3 : g.phase ? 2 : flip, g.pf, 1, g.Cin);
    if (e != cudaSuccess) return e;
  }

  CUtensorMap xmap;
  const std::uint64_t rows_total = std::uint64_t(g.N) * sg.Hp * sg.Wp;
  const cuuint64_t dims[2] = {cuuint64_t(Cp), cuuint64_t(rows_total)};
  const cuuint64_t strides[1] = {cuuint64_t(Cp) * 4};
  const cuuint32_t box[2] = {32, cuuint32_t(sg.box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  if (encode_tiled()(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, xp, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;

  StripParams p{};
  p.btiles = btiles;
  p.out = out;
  p.alpha = alpha;
  p.beta = beta;
  p.BN = BN;
  p.n_tiles = n_tiles;
  p.Wp = sg.Wp;
  p.HWp = sg.Hp * sg.Wp;
  p.OH = g.Hout;
  p.OW = g.Wout;
  p.swap = sg.swap ? 1 : 0;
  p.msub = sg.msub;
  p.nsb = sg.nsb;
  p.prof = tune("prof", 0);
  const int tile_pos = sg.swap ? 2 * kBM : sg.msub * kBM;
  // the last image needs positions up to (OH-1)*Wp + OW; the padding rows
  // between images are computed and dropped (their strips read zeros)
  p.nimg = g.N;
  p.m_tiles = int(((std::int64_t(g.N) - 1) * p.HWp + (g.Hout - 1) * sg.Wp + g.Wout + tile_pos - 1) / tile_pos);
  p.taps = taps;
  p.S = g.S;
  p.c_chunks = Cp / 32;
  p.Nout = g.Nout;
  p.P = g.Hout * g.Wout;
  p.box_rows = sg.box_rows;
  p.nboxes = sg.nboxes;
  p.stages = sg.stages;
  p.fd_Wp = FastDiv(std::uint32_t(sg.Wp));
  p.fd_HWp = FastDiv(std::uint32_t(p.HWp));
  p.fd_mt = FastDiv(std::uint32_t(p.m_tiles));
  p.phase = g.phase;
  if (g.phase) {
    p.Cr = g.pf.C;
    p.Hr = g.Hr;
    p.Wr = g.Wr;
    p.ssh = g.pf.sh;
    p.ssw = g.pf.sw;
    p.sph = g.rph;
    p.spw = g.rpw;
    p.fd_Cr = FastDiv(std::uint32_t(g.pf.C));
    p.fd_ssw = FastDiv(std::uint32_t(g.pf.bw));
    p.sAh = std::min(g.pf.sh, g.pf.R);
    p.sBw = g.pf.bw;
    p.pair = phase_pair(g);
    p.bp = g.pf.P;
    p.fd_blk = FastDiv(std::uint32_t(p.sAh * g.pf.bw * g.pf.C));
    p.ph32 = g.pf.C % 32 == 0 && !p.pair && p.bp == 1 && p.sAh >= p.ssh && p.sBw >= p.ssw && tune("ph32", 1);
  }
  const int smem = int(sg.nsb * sg.strip_bytes + std::size_t(sg.stages) * kTapsPerStage * BN * 128) + 1024 + 256 +
                   (sg.swap ? 4 * 32 * 33 * 4 : 0);
  // the launch's own size (the kernel also has a small static tap table)
  e = set_smem_attr(reinterpret_cast<const void*>(strip_kernel), std::max(smem, 116 * 1024));
  if (e != cudaSuccess) return e;
  trace_variant("strip swap=%d msub=%d nsb=%d m_tiles=%d n_tiles=%d BN=%d stages=%d boxes=%d", p.swap, p.msub, p.nsb,
                p.m_tiles, p.n_tiles, BN, sg.stages, sg.nboxes);
  return launch_pdl(strip_kernel, dim3(std::min(sm_count(), p.m_tiles * p.n_tiles)), dim3(kThreads),
                    std::size_t(std::max(smem, 116 * 1024)), st, xmap, p);
}

// act_img / w_ldi: image pitch of act and Forward input-channel pitch of w
// when the call covers a slice of the reduction channels (0: dense)
cudaError_t run_geo(const Geo& g, const float* act, const float* w, int flip, float* out, void* ws, float alpha,
                    float beta, cudaStream_t st, int flags, std::int64_t act_img = 0, int w_ldi = 0) {
  if (!act_img) {
    int ks = 0, bn = 0;
    geo_ws(g, &ks, &bn);
    const StripGeo sg = strip_geo(g, bn);
    if (sg.ok) return run_strip(g, sg, act, w, flip, out, ws, alpha, beta, st, flags);
  }
  const int Cp = cpad(g.Cin), taps = g.R * g.S;
  int ksteps = 0, BN = 0;
  geo_ws(g, &ksteps, &BN);
  const int n_tiles = (g.Nout + BN - 1) / BN;
  // 2-SM MMA (precomp2_kernel) for >= 128-wide filter tiles: measured at 64
  // images, conv2 F 95 -> 81 us, conv3 BD 79 -> 65, conv4 F 85 -> 69, conv5
  // 63 -> 52 (conv2 F at 256 images: 489 TFLOP/s); narrower tiles (conv2 BD,
  // conv1) stay on the 1-SM kernel, which won there. A function of the shape
  // only, so all micro-batches of a call agree on the filter layout.
  const bool two_sm = Cp != 4 && BN % 16 == 0 && BN >= tune("two_sm_min_bn", 128) && tune("two_sm", 1);
  // packed filter first: its size does not depend on the micro-batch, so
  // later micro-batches of the same call reuse it (kFilterReady)
  float* btiles = static_cast<float*>(ws);
  float* act_nhwc = reinterpret_cast<float*>(static_cast<char*>(ws) +
                                             align256(std::size_t(n_tiles) * ksteps * BN * 128));
  const int HW = g.Hin * g.Win;
  cudaError_t e;
  if (g.s2d) {
    S2D d = g.sd;
    d.Cp = Cp;
    e = launch_s2d(act, act_nhwc, d, g.N, st);
  } else {
    e = launch_pdl(to_nhwc_kernel, dim3((HW + 63) / 64, (Cp + 31) / 32, g.N), dim3(256), 0, st, act, act_nhwc,
                   g.Cin, HW, Cp, act_img ? act_img : std::int64_t(g.Cin) * HW);
  }
  if (e != cudaSuccess) return e;
  if (!(flags & kFilterReady)) {
    e = launch_pdl(pack_filter_kernel, dim3(n_tiles * ksteps, (8 * BN + 255) / 256), dim3(256), 0, st, w, btiles, g.Nout, g.Cin, taps, BN,
                   n_tiles,
                   ksteps, Cp == 4 ? 1 : 0, Cp / 32, g.s2d ? 3 : g.phase ? 2 : flip, g.pf, two_sm ? 0 : 1,
                   w_ldi ? w_ldi : g.Cin);
    if (e != cudaSuccess) return e;
  }

  CUtensorMap amap;
  const cuuint64_t dims[4] = {cuuint64_t(Cp), cuuint64_t(g.Win), cuuint64_t(g.Hin), cuuint64_t(g.N)};
  const cuuint64_t strides[3] = {cuuint64_t(Cp) * 4, cuuint64_t(Cp) * 4 * g.Win, cuuint64_t(Cp) * 4 * g.Win * g.Hin};
  const int lower[2] = {-g.pw, -g.ph};
  const int upper[2] = {(g.pw_hi < 0 ? g.pw : g.pw_hi) - (g.S - 1), (g.ph_hi < 0 ? g.ph : g.ph_hi) - (g.R - 1)};
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
  p.prof = tune("prof", 0);
  p.phase = g.phase;
  if (g.phase) {
    p.Cr = g.pf.C;
    p.Hr = g.Hr;
    p.Wr = g.Wr;
    p.ssh = g.pf.sh;
    p.ssw = g.pf.sw;
    p.sph = g.rph;
    p.spw = g.rpw;
    p.fd_Cr = FastDiv(std::uint32_t(g.pf.C));
    p.fd_ssw = FastDiv(std::uint32_t(g.pf.bw));
    p.sAh = std::min(g.pf.sh, g.pf.R);
    p.sBw = g.pf.bw;
    p.pair = phase_pair(g);
    p.bp = g.pf.P;
    p.fd_blk = FastDiv(std::uint32_t(p.sAh * g.pf.bw * g.pf.C));
    p.ph32 = g.pf.C % 32 == 0 && !p.pair && p.bp == 1 && p.sAh >= p.ssh && p.sBw >= p.ssw && tune("ph32", 1);
  }
  if (two_sm) {
    CUtensorMap bmap;
    const cuuint64_t bdims[2] = {32, cuuint64_t(n_tiles) * ksteps * BN};
    const cuuint64_t bstr[1] = {128};
    const cuuint32_t bbox[2] = {32, cuuint32_t(BN / 2)};
    const cuuint32_t bes[2] = {1, 1};
    if (encode_tiled()(&bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, btiles, bdims, bstr, bbox, bes,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    // two pair sub-tiles per tile (512 rows) share each filter box:
    // UCUDNN_TUNE=pc2_msub=2 forces it, 0 picks it when every cluster still
    // gets a tile
    const int pc2_msub = tune("pc2_msub", 1);
    p.msub = pc2_msub == 2 || (pc2_msub == 0 && p.M >= 4 * kBM * (sm_count() / 2)) ? 2 : 1;
    p.nacc2 = 2 * p.msub * ((BN + 31) & ~31) <= 512 ? 2 : 1;  // tmem_ld32 reads whole 32-column groups
    p.m_tiles = (p.M + 2 * p.msub * kBM - 1) / (2 * p.msub * kBM);
    p.fd_mt = FastDiv(std::uint32_t(p.m_tiles));
    // one reduction step per stage at BN >= 256 (3 -> 6 stages): AlexNet
    // conv5 F / BD 122 -> 116 / 120 -> 112 us, ResNet l3b1c1 BD 195 -> 182;
    // two at BN <= 192 (ResNet l2 F 199 vs 219 with one; scripts/r02_run107.sh)
    p.ksub = std::max(1, std::min(2, tune("pc2_ksub", p.msub == 2 || BN >= 256 ? 1 : 2)));
    const int stage2 = p.ksub * (p.msub * kBM * 128 + ((BN / 2 * 128 + 1023) & ~1023));
    p.stages = ring_stages(std::min(tune("pc2_stages", 8), (200 * 1024) / stage2));
    const int smem2 = std::max(p.stages * stage2 + 1024 + 256, 116 * 1024);
    e = set_smem_attr(reinterpret_cast<const void*>(precomp2_kernel), 227 * 1024);
    if (e != cudaSuccess) return e;
    const int clusters = std::min(sm_count() / 2, p.m_tiles * p.n_tiles);
    trace_variant("precomp2 flip=%d m_tiles=%d n_tiles=%d clusters=%d BN=%d msub=%d phase=%d s2d=%d", flip,
                  p.m_tiles, p.n_tiles, clusters, BN, p.msub, int(g.phase), int(g.s2d));
    count_launch();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = std::size_t(smem2);
    cfg.stream = st;
    cudaLaunchAttribute cat[1];
    cat[0].id = cudaLaunchAttributeClusterDimension;
    cat[0].val.clusterDim.x = 2;
    cat[0].val.clusterDim.y = 1;
    cat[0].val.clusterDim.z = 1;
    cfg.attrs = cat;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, precomp2_kernel, amap, bmap, p);
  }
  // two 32-deep chunks per stage (8 MMAs per tcgen05.commit): measured
  // 10-25 % faster than one on AlexNet conv2 / conv4 (same box, A/B)
  // Two CTAs per SM (256 TMEM columns each) once there are more tiles than
  // SMs: the second wave's tail disappears and a CTA's epilogue hides behind
  // its neighbour's MMAs. Measured on AlexNet at 64 images: conv2 BD 196 ->
  // 157 us, conv1 F 151 -> 132, conv3 F 71 -> 63, conv4 BD 89 -> 77; with
  // fewer tiles than SMs it packs them onto fewer SMs and loses (conv4 F).
  // Narrow filters (BN <= 64), UCUDNN_TUNE=pc_msub=2: two 128-pixel MMA
  // sub-tiles per tile share each filter chunk, one chunk per stage (still 8
  // MMAs per commit). Off by default: per 256 images, with two CTAs per SM
  // (pc_cps=2) it measured AlexNet conv1 F 438 -> 430 us, conv1 BD 504 ->
  // 496, ResNet l1 F 290 -> 280, but conv2 BD 413 -> 462 and ResNet conv1
  // BD 1085 -> 1102; with one CTA per SM it lost everywhere
  p.msub = tune("pc_msub", 1) == 2 && BN <= 64 && p.M > kBM ? 2 : 1;
  if (p.msub == 2) {
    p.m_tiles = (p.M + 2 * kBM - 1) / (2 * kBM);
    p.fd_mt = FastDiv(std::uint32_t(p.m_tiles));
  }
  p.cps = tune("pc_cps", p.msub == 1 && p.m_tiles * p.n_tiles > sm_count() ? 2 : 1) == 2 ? 2 : 1;
  // one reduction step per stage: twice the stages in the same shared
  // memory (two CTAs per SM with BN = 64 had only two 48 KB stages);
  // measured equal or faster on every planned call (AlexNet conv2 BD 7@256
  // 452 -> 417 us, ResNet l1 F / BD 5@64 340 -> 324, scripts/r02_run105.sh,
  // r02_run106.sh)
  p.ksub = std::max(1, std::min(4, tune("pc_ksub", 1)));
  const int stage_bytes = p.ksub * (p.msub * kBM * 128 + ((BN * 128 + 1023) & ~1023));
  p.stages = ring_stages(std::min(tune("pc_stages", 8), (p.cps == 2 ? 100 * 1024 : 200 * 1024) / stage_bytes));
  // >= 116 KB so the persistent grid lands one CTA per SM (each owns all
  // 512 TMEM columns)
  const int smem = p.cps == 2 ? p.stages * stage_bytes + 1024 + 256
                              : std::max(p.stages * stage_bytes + 1024 + 256, 116 * 1024);
  if (smem > 48 * 1024) {
    // dynamic <= ~202 KB; the cap leaves room for the 5 KB of static tables
    e = set_smem_attr(reinterpret_cast<const void*>(precomp_kernel), 216 * 1024);
    if (e != cudaSuccess) return e;
  }
  const int grid = std::min(p.cps * sm_count(), p.m_tiles * p.n_tiles);
  trace_variant("precomp flip=%d cps=%d msub=%d m_tiles=%d n_tiles=%d grid=%d BN=%d phase=%d s2d=%d", flip,
                p.cps, p.msub, p.m_tiles, p.n_tiles, grid, BN, int(g.phase), int(g.s2d));
  return launch_pdl(precomp_kernel, dim3(grid), dim3(kThreads), std::size_t(smem), st, amap, p);
}

Geo fwd_geo(const ConvShape& s) {
  return Geo{s.N, s.C, s.H, s.W, s.K, s.OH(), s.OW(), s.R, s.S, s.ph, s.pw, s.sh, s.sw};
}
// Strided Forward on a space-to-depth copy: with x_a[i] = x_pad[i*sh + a],
// y[oh] = sum_{t, a} x_a[oh + t] * W[t*sh + a], a stride-1 conv over
// Ah*Bw*C phase-channels with a Th x Tw filter (taps past R / S are zero).
// Used when it shrinks the TMA work: few input channels (AlexNet conv1:
// 3 -> 48 channels, 121 -> 9 taps) or 1x1 strided shortcuts.
Geo fwd_s2d_geo(const ConvShape& s) {
  const int Ah = std::min(s.sh, s.R), Bw = std::min(s.sw, s.S);
  const int Th = (s.R + s.sh - 1) / s.sh, Tw = (s.S + s.sw - 1) / s.sw;
  const int OH = s.OH(), OW = s.OW(), Hq = OH + Th - 1, Wq = OW + Tw - 1;
  Geo g{s.N, Ah * Bw * s.C, Hq, Wq, s.K, OH, OW, Th, Tw, 0, 0, 1, 1};
  g.s2d = 1;
  g.pf = PhaseFilter{s.C, s.R, s.S, Bw, Bw, Tw};
  g.pf.sh = s.sh;  // r = t*sh + a (a < Ah); Bw doubles as the channel-decode stride
  g.sd = S2D{s.C, s.H, s.W, s.sh, s.sw, s.ph, s.pw, Bw, Ah * Bw * s.C, Hq, Wq, 0};
  return g;
}
bool use_s2d(const ConvShape& s) {
  return (s.sh > 1 || s.sw > 1) && (s.C < 32 || (s.R == 1 && s.S == 1)) && tune("s2d", 1);
}
Geo f_geo(const ConvShape& s) { return use_s2d(s) ? fwd_s2d_geo(s) : fwd_geo(s); }
// stride-1 BackwardData as a forward conv of dy with the flipped filter
Geo bwd_data_geo(const ConvShape& s) {
  return Geo{s.N, s.K, s.OH(), s.OW(), s.C, s.H, s.W, s.R, s.S, s.R - 1 - s.ph, s.S - 1 - s.pw, 1, 1};
}
// Strided BackwardData, split by output stride phase. In padded input
// coordinates h' = h + ph = i*sh + a, dx_a[i] = sum_t sum_k dy[k][i - t] *
// W[k][c][a + t*sh] (t < Th = ceil(R/sh)): every phase is a stride-1
// correlation of dy with a Th x Tw sub-filter, so all sh*sw*C phase-channels
// form ONE stride-1 forward conv (padding Th-1 low) whose epilogue scatters
// column (a, b, c) of pixel (i, j) to dx[c][i*sh + a - ph][j*sw + b - pw].
// Taps past the filter edge are zero in the packed filter.
Geo bwd_data_phase_geo(const ConvShape& s) {
  const int Th = (s.R + s.sh - 1) / s.sh, Tw = (s.S + s.sw - 1) / s.sw;
  const int OH = s.OH(), OW = s.OW();
  // cover every dx row: i up to (H - 1 + ph) / sh
  const int Hq = std::max(OH + Th - 1, (s.H - 1 + s.ph) / s.sh + 1);
  const int Wq = std::max(OW + Tw - 1, (s.W - 1 + s.pw) / s.sw + 1);
  // only the phases that own filter taps become GEMM columns
  const int Ah = std::min(s.sh, s.R), Bw = std::min(s.sw, s.S);
  // Few phase-channels (ResNet conv1: 12): block P phase-grid columns into
  // one GEMM row -- a stride-P conv of dy with a Th x (Tw + P - 1) banded
  // filter and P x as many columns -- so each MMA does P x the work and dy
  // is re-read (Tw + P - 1) / P instead of Tw times per output column.
  // P <= 8 (TMA im2col traversal stride); not with tapless phases / pair stores.
  const int nab = Ah * Bw * s.C;
  int P = 1;
  if (Ah == s.sh && Bw == s.sw && !(s.R == 1 && s.S == 1)) {
    P = tune("bd_block", -1);
    if (P < 0) {  // widest block up to 4 keeping the columns in one <= 128-wide tile
      // (ResNet conv1 BD at 256 images: P = 1 / 2 / 4 / 8 -> 1426 / 1074 /
      // 908 / 1211 us; AlexNet conv1, 48 phase-channels: P = 1 is best)
      P = 1;
      while (P < 4 && (P + 1) * nab <= 128) ++P;
      if (nab > 32) P = 1;
    }
    P = std::max(1, std::min(8, P));
  }
  const int Wqb = (Wq + P - 1) / P;
  Geo g{s.N, s.K, OH, OW, P * nab, Hq, Wqb, Th, Tw + P - 1, Th - 1, Tw - 1, 1, P};
  g.ph_hi = Hq - OH;
  g.pw_hi = Wqb * P - OW;
  g.phase = 1;
  g.pf = PhaseFilter{s.C, s.R, s.S, s.sh, s.sw, Tw, Bw};
  g.pf.P = P;
  g.Hr = s.H;
  g.Wr = s.W;
  g.rph = s.ph;
  g.rpw = s.pw;
  return g;
}
Geo bd_geo(const ConvShape& s) { return (s.sh == 1 && s.sw == 1) ? bwd_data_geo(s) : bwd_data_phase_geo(s); }

}  // namespace

// Diagnostic: average MMA-warp cycles (data wait, issue, accumulator wait,
// total) over the CTAs of the last precomp launch run with UCUDNN_TUNE=prof=1.
void precomp_profile(double out[4]) {
  static unsigned long long h[1024 * 4];
  cudaMemcpyFromSymbol(h, g_prof, sizeof(h));
  double s[4] = {0, 0, 0, 0};
  int n = 0;
  for (int b = 0; b < 1024; ++b) {
    if (h[b * 4 + 3] == 0) continue;
    for (int i = 0; i < 4; ++i) s[i] += double(h[b * 4 + i]);
    ++n;
  }
  for (int i = 0; i < 4; ++i) out[i] = n ? s[i] / n : 0;
}

// Space-to-depth copy for the channels-last BackwardFilter (bfnhwc.cu):
// xs[n][i][j][Cp], channel (a*Bw + b)*C + c = x[n][c][i*sh + a - ph][j*sw + b - pw]
cudaError_t space_to_depth_nhwc(const float* x, float* out, int N, int C, int H, int W, int sh, int sw, int ph,
                                int pw, int Ah, int Bw, int Hq, int Wq, int Cp, cudaStream_t st) {
  const S2D d{C, H, W, sh, sw, ph, pw, Bw, Ah * Bw * C, Hq, Wq, Cp};
  return launch_s2d(x, out, d, N, st);
}

// Strided 1x1 Forward (ResNet projections): the taps are a plain subsample
// of x, so copy the sampled pixels into a compact NCHW tensor (one pass) and
// run the 1x1 stride-1 GEMM straight on its planes (z1x1.cu) -- instead of
// the space-to-depth rewrite, which would multiply the reduction by sh*sw
// with all but one phase's weights zero.
namespace {
ConvShape subsampled(const ConvShape& s) {
  ConvShape c = s;
  c.H = s.OH();
  c.W = s.OW();
  c.sh = c.sw = 1;
  return c;
}
bool use_subsample(int op, const ConvShape& s) {
  return op == kFwd && s.R == 1 && s.S == 1 && s.ph == 0 && s.pw == 0 && (s.sh > 1 || s.sw > 1) &&
         tune("pc_subsample", 1) && z1x1_supports(kFwd, subsampled(s));
}
__global__ void subsample_kernel(const float* __restrict__ x, float* __restrict__ xs, int H, int W, int OH, int OW,
                                 int sh, int sw, long long planes) {
  pdl_wait();
  const long long n = planes * OH * OW;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long pl = i / ((long long)OH * OW);
    const int rem = int(i - pl * OH * OW), oh = rem / OW, ow = rem - oh * OW;
    xs[i] = __ldg(x + (pl * H + (long long)oh * sh) * W + (long long)ow * sw);
  }
}
}  // namespace

bool precomp_supports(int op, const ConvShape& s) {
  if (op == kFwd) return s.sh <= 8 && s.sw <= 8 && s.ph <= 127 && s.pw <= 127 && s.R <= 64 && s.S <= 64;
  if (op == kBwdData) {
    if (s.sh == 1 && s.sw == 1) return s.ph <= s.R - 1 && s.pw <= s.S - 1;
    // phase split (any stride): sh*sw*C phase-channels, Th x Tw sub-filters
    return s.sh <= 8 && s.sw <= 8 && s.ph <= s.R - 1 && s.pw <= s.S - 1 && s.R <= 64 && s.S <= 64;
  }
  // BackwardFilter: TMA-tiled phase-split operands (bfilter.cu)
  return bf_supports(s);
}

std::int64_t precomp_workspace(int op, const ConvShape& s) {
  if (use_subsample(op, s)) return (std::int64_t(s.N) * s.C * s.OH() * s.OW() * 4 + 255) / 256 * 256;
  if (op == kFwd) return std::int64_t(geo_ws(f_geo(s)));
  if (op == kBwdData) return std::int64_t(geo_ws(bd_geo(s)));
  return bf_workspace(s);
}

// ---------------------------------------------------------------- channel-sliced
// UCUDNN_ALGO_PRECOMP_SLICED (Forward / BackwardData): the same implicit
// GEMM run over slices of the reduction channels (C for Forward, K for
// BackwardData), each accumulating into the output (beta = 1 after the
// first), so the channels-last operand copy -- the whole of PRECOMP's
// workspace apart from the packed filter -- is per slice, at most
// kSliceCap. Under a 64 MiB limit that lets one call cover 256 images where
// PRECOMP has to be micro-batched (AlexNet conv2 BackwardData: 143 MB copy).
namespace {
// copy cap per slice (UCUDNN_TUNE=slice_cap_kib overrides, for tests)
std::size_t slice_cap() { return std::size_t(tune("slice_cap_kib", 40 * 1024)) << 10; }
struct Sliced {
  Geo g;       // geometry of one slice (Cin = slice channels)
  int flip = 0, ctot = 0, cs = 0, n = 0;  // reduction channels, per slice, slices
  bool ok = false;
};
Sliced sliced_geo(int op, const ConvShape& s) {
  Sliced r;
  if (op == kFwd) {
    if (use_s2d(s)) return r;
    r.g = fwd_geo(s);
  } else if (op == kBwdData) {
    r.g = bd_geo(s);
    r.flip = 1;
  } else {
    return r;
  }
  r.ctot = r.g.Cin;
  const std::size_t act = std::size_t(r.g.N) * r.g.Hin * r.g.Win * cpad(r.ctot) * 4;
  const std::size_t cap = slice_cap();
  r.n = int((act + cap - 1) / cap);
  if (r.n < 2 || r.ctot < 64) return r;  // nothing to gain over PRECOMP
  r.cs = (r.ctot + r.n - 1) / r.n;
  r.cs = (r.cs + 31) / 32 * 32;
  r.n = (r.ctot + r.cs - 1) / r.cs;
  if (r.n < 2) return r;
  r.g.Cin = r.cs;
  int ks = 0, bn = 0;
  geo_ws(r.g, &ks, &bn);
  if (strip_geo(r.g, bn).ok) return r;  // the strip path has no slice support
  r.ok = true;
  return r;
}
}  // namespace

bool precomp_sliced_supports(int op, const ConvShape& s) { return precomp_supports(op, s) && sliced_geo(op, s).ok; }

std::int64_t precomp_sliced_workspace(int op, const ConvShape& s) {
  const Sliced r = sliced_geo(op, s);
  return r.ok ? std::int64_t(geo_ws(r.g)) : 0;
}

cudaError_t precomp_sliced_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws,
                               float alpha, float beta, cudaStream_t st) {
  const Sliced r = sliced_geo(op, s);
  if (!r.ok) return cudaErrorInvalidValue;
  const std::int64_t hw = std::int64_t(r.g.Hin) * r.g.Win;
  const int taps = r.g.R * r.g.S;
  for (int i = 0; i < r.n; ++i) {
    const int c0 = i * r.cs;
    Geo g = r.g;
    g.Cin = std::min(r.cs, r.ctot - c0);
    if (g.Cin <= 0) break;
    // Forward: w[k][c0 + c] (pitch C); BackwardData: w[k0 + k] is contiguous
    // (stride-1: [K][C][R][S] rows; phase: the same rows, decoded by pf)
    const float* w = op == kFwd ? b + std::int64_t(c0) * taps : b + std::int64_t(c0) * s.C * s.R * s.S;
    cudaError_t e = run_geo(g, a + c0 * hw, w, op == kFwd ? 0 : 1, out, ws, alpha,
                            i == 0 ? beta : 1.f, st, 0, std::int64_t(r.ctot) * hw, op == kFwd ? r.ctot : 0);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t precomp_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                        float beta, cudaStream_t st, int flags) {
  if (use_subsample(op, s)) {
    float* xs = static_cast<float*>(ws);
    const long long n = (long long)s.N * s.C * s.OH() * s.OW();
    cudaError_t e = launch_pdl(subsample_kernel, dim3(int(std::min<long long>((n + 255) / 256, 8 * sm_count()))),
                               dim3(256), 0, st, a, xs, s.H, s.W, s.OH(), s.OW(), s.sh, s.sw,
                               (long long)s.N * s.C);
    if (e != cudaSuccess) return e;
    trace_variant("precomp subsample 1x1 s%d -> z1x1", s.sh);
    return z1x1_run(kFwd, subsampled(s), xs, b, out, alpha, beta, st);
  }
  if (op == kFwd) return run_geo(f_geo(s), a, b, 0, out, ws, alpha, beta, st, flags);
  if (op == kBwdData) return run_geo(bd_geo(s), a, b, 1, out, ws, alpha, beta, st, flags);
  return bf_run(s, a, b, out, ws, alpha, beta, st);
}

}  // namespace ucudnn
