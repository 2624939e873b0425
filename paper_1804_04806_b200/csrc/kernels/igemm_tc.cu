// UCUDNN_ALGO_IMPLICIT_GEMM (0 workspace), Forward and BackwardData: a
// persistent tcgen05 implicit GEMM whose operands are gathered straight from
// the caller's NCHW tensors by cp.async -- nothing is staged in global memory.
//
// One GEMM covers both ops ("source" = x for Forward, dy for BackwardData):
//   rows    = positions (n, gi, gj) of a grid over the source, 128 per tile;
//             input coordinates ih = gi*gsh - gph + t, iw = gj*gsw - gpw + u
//   reduce  = (cs, t, u) over source channels x T x U taps
//   columns = output channels (Forward: k) or stride-phase channels
//             (BackwardData: (a, b, c), the adjoint split by output phase)
//   out[n][col][gi*osh + a - oph][gj*osw + b - opw] = alpha * D + beta * out
// Forward (reference_conv.hpp:70-100): grid = OH x OW, taps = R x S at stride
// sh, output column k. BackwardData (reference_conv.hpp:105-135, as the
// gather form of its scatter): with h + ph = i*sh + a, only taps r = a + t*sh
// reach dx row h, from dy row i - t, so
//   dx[c][i*sh + a - ph][j*sw + b - pw] = sum_{k,t,u} dy[k][i-t][j-u] * w[k][c][a+t*sh][b+u*sw]
// -- a stride-1 "forward" conv of dy over a ceil(R/sh) x ceil(S/sw) tap grid
// whose sh*sw*C output columns are scattered to dx; stride 1 is the one-phase
// case. Every dx element belongs to exactly one (position, column).
//
// Operands (zero-workspace implicit GEMM on
// tcgen05/TMEM):
//   A (positions x reduction) is *MN-major*: lane = position, so a warp's 32
//   cp.async of one reduction index read 32 neighbouring source pixels
//   (coalesced) and write one 128 B smem row of the 128B/32B-atom swizzle
//   (Layout_MN_SW128_32B, DESIGN finding 5) -- no bank conflicts;
//   B (columns x reduction) is K-major SW128: Forward with C*R*S % 4 == 0
//   loads it by TMA straight from the KCRS filter (rows k are (c, r, s)
//   contiguous); otherwise lanes gather 32 consecutive reduction indices of a
//   row (Forward: one contiguous 128 B run; BackwardData: the flipped,
//   phase-strided sub-filter, L1/L2-resident).
// Producers never wait for their own copies (cp.async.mbarrier.arrive.noinc,
// finding 11): with an 8-deep ring every producer thread keeps several
// stages of gathers in flight, which is what the round-1 LDG/STS version
// (one stage per thread, 5.5 % tensor pipe) could not.
//
// Warps: 0-3 epilogue (TMEM -> registers -> NCHW stores, alpha/beta), 4 TMEM
// owner + MMA issuer (two 256-column accumulators: a tile's epilogue
// overlaps the next tile's MMAs), 5-20 producers (warp 5 lane 0 also issues
// the TMA B loads).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

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
constexpr int kProd = 16;
constexpr int kThreads = (5 + kProd) * 32;
constexpr std::uint32_t kABytes = kBM * 128;  // 4 MN blocks x 32 K-rows x 128 B

struct ZParams {
  const float* src;
  const float* w;
  float* out;
  float alpha, beta;
  int Cs, Hs, Ws, HWs;
  long long simg;  // Cs*Hs*Ws
  int Hg, Wg, M;
  int gi0, gj0;  // grid origin: position (gi, gj) stands for grid point (gi + gi0, gj + gj0)
  int gsh, gsw, gph, gpw;
  int T, U, Kr, chunks;
  int ncols, BN, m_tiles, n_tiles;
  int bmode;  // 0 TMA, 1 dense rows w[col*Kr + kr], 2 BackwardData phase sub-filter
  int CRS, RS, R, S, fsh, fsw, C;
  int Ho, Wo, osh, osw, oph, opw;
  long long oimg;
  int stages;
  int msub;  // position sub-tiles of 128 per tile, sharing each B stage (halves B traffic at 2)
  int nacc;  // TMEM accumulator sets (2: a tile's epilogue overlaps the next tile's MMAs)
  int bres;  // gathered B (single column tile) resident in smem for every chunk: filled once per CTA
  FastDiv fd_HWg, fd_Wg, fd_TU, fd_U, fd_C, fd_sw;
};

struct ColEnt {
  int ooff;   // output offset of the column within an image, phase offsets excluded
  int woff;   // filter offset of the column's row (bmode 1 / 2)
  short a, b;  // output phase offsets (rows, columns)
  short rl, sl;  // bmode 2: taps valid while t*sh < rl and u*sw < sl
};

__device__ __forceinline__ void cp_async4(std::uint32_t dst, const float* src, std::uint32_t src_size) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_size) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(std::uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_backoff(std::uint64_t* bar, std::uint32_t parity) {
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
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// bits t in [lo, hi) of a width-n mask (n <= 32)
__device__ __forceinline__ std::uint32_t range_mask(int lo, int hi, int n) {
  lo = max(lo, 0);
  hi = min(hi, n);
  if (hi <= lo) return 0u;
  const std::uint32_t h = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
  return h & ~((1u << lo) - 1u);
}
// MN-major SW128 / 32 B-atom descriptor (bfnhwc.cu desc_mn32): LBO = 4096 B
// between 32-position blocks, SBO = 512 B (4 K-rows per atom)
__device__ __forceinline__ std::uint64_t desc_mn32(std::uint32_t saddr) {
  std::uint64_t d = 0;
  d |= std::uint64_t((saddr >> 4) & 0x3FFF);
  d |= std::uint64_t(4096 >> 4) << 16;
  d |= std::uint64_t(512 >> 4) << 32;
  d |= std::uint64_t(1) << 46;
  d |= std::uint64_t(1) << 61;
  return d;
}

__device__ __forceinline__ ColEnt col_entry(const ZParams& p, int col) {
  ColEnt e{};
  if (p.bmode == 2) {  // col = (a*sw + b)*C + c
    std::uint32_t ab, c, a, b;
    p.fd_C.divmod(std::uint32_t(col), ab, c);
    p.fd_sw.divmod(ab, a, b);
    e.ooff = int(c) * p.Ho * p.Wo;
    e.woff = int(c) * p.RS + int(a) * p.S + int(b);
    e.a = short(a);
    e.b = short(b);
    e.rl = short(p.R - int(a));
    e.sl = short(p.S - int(b));
  } else {
    e.ooff = col * p.Ho * p.Wo;
    e.woff = col * p.Kr;
    e.rl = e.sl = 0x7fff;
  }
  return e;
}

template <int MSUB>
__global__ void __launch_bounds__(kThreads, 1)
    zgemm_kernel(const __grid_constant__ CUtensorMap bmap, const ZParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t b_bytes = (std::uint32_t(p.BN) * 128 + 1023) & ~1023u;
  constexpr int msub = MSUB;
  // resident B: [chunk][BN rows][128 B] after the ring; the ring then holds A only
  const std::uint32_t stage_bytes = msub * kABytes + (p.bres ? 0u : b_bytes);
  const int kStages = p.stages;
  const std::uint32_t bres_bytes = p.bres ? std::uint32_t(p.chunks) * std::uint32_t(p.BN) * 128 : 0u;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kStages * stage_bytes + bres_bytes);
  std::uint64_t* empty = full + kMaxStages;
  std::uint64_t* tfull = empty + kMaxStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  __shared__ ColEnt ptab[kMaxBN];  // producers' column table (current n tile)
  __shared__ ColEnt etab[kMaxBN];  // epilogue's

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], kProd * 32 + (p.bmode == 0 ? 1 : 0));
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
  const int units = p.m_tiles * p.n_tiles;

  if (warp >= 5) {
    // ------------------------------------------------ producers
    const int pw = warp - 5;
    const int pb = pw & 3;         // this warp's 32-position block of the tile
    const int js = pw >> 2;        // and its reduction indices k = js, js + 4, ... (k & 3 == js)
    const std::uint32_t sbase = smem_u32(smem);
    const std::uint32_t swz_lane = std::uint32_t(lane & 7) * 4;
    const bool tma_thread = p.bmode == 0 && pw == 0 && lane == 0;
    if (tma_thread) prefetch_tmap(&bmap);
    int st = 0;
    std::uint32_t ph = 0;
    int cur_nt = -1;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int mt = u % p.m_tiles, nt = u / p.m_tiles;
      if (p.bmode != 0 && nt != cur_nt) {
        named_sync(1, kProd * 32);  // every producer is done with the previous table
        for (int j = threadIdx.x - 160; j < p.BN; j += kProd * 32)
          if (nt * p.BN + j < p.ncols) ptab[j] = col_entry(p, nt * p.BN + j);
        named_sync(1, kProd * 32);
        cur_nt = nt;
        if (p.bres) {
          // the whole (single-tile) B once: chunk ch, row r at
          // resB + (ch * BN + r) * 128, SW128 K-major within each chunk
          const std::uint32_t resB = sbase + kStages * stage_bytes;
          const std::uint32_t bsw = std::uint32_t(lane >> 2), bl = std::uint32_t(lane & 3) * 4;
          const int brows = min(p.BN, p.ncols);
          for (int ch = 0; ch < p.chunks; ++ch) {
            const int kr = ch * 32 + lane;
            int boff = 0, brt = 1 << 14, bsu = 1 << 14;
            if (kr < p.Kr) {
              std::uint32_t cs, tu, t, uu;
              p.fd_TU.divmod(std::uint32_t(kr), cs, tu);
              p.fd_U.divmod(tu, t, uu);
              brt = (p.T - 1 - int(t)) * p.fsh;
              bsu = (p.U - 1 - int(uu)) * p.fsw;
              boff = int(cs) * p.CRS + brt * p.S + bsu;
            }
            for (int r = pw; r < p.BN; r += kProd) {
              std::uint32_t ok = 0;
              int off = 0;
              if (r < brows) {
                const ColEnt e = ptab[r];
                ok = (kr < p.Kr && brt < e.rl && bsu < e.sl) ? 1u : 0u;
                off = e.woff + boff;
              }
              const std::uint32_t dst = resB + std::uint32_t(ch * p.BN + r) * 128 +
                                        ((bsw ^ std::uint32_t(r & 7)) << 4) + bl;
              cp_async4(dst, p.w + off, ok * 4u);
            }
          }
          asm volatile("cp.async.wait_all;" ::: "memory");
          named_sync(1, kProd * 32);  // resident B complete before any stage arrives
        }
      }
      // this lane's position in each sub-tile
      std::uint32_t vr[2] = {0, 0}, vs[2] = {0, 0};
      const float* base[2] = {p.src, p.src};
#pragma unroll
      for (int sub = 0; sub < 2; ++sub) {
        const int m = (mt * msub + sub) * kBM + pb * 32 + lane;
        if (sub < msub && m < p.M) {
          std::uint32_t n, g, gi, gj;
          p.fd_HWg.divmod(std::uint32_t(m), n, g);
          p.fd_Wg.divmod(g, gi, gj);
          const int ihb = (int(gi) + p.gi0) * p.gsh - p.gph, iwb = (int(gj) + p.gj0) * p.gsw - p.gpw;
          vr[sub] = range_mask(-ihb, p.Hs - ihb, p.T);
          vs[sub] = range_mask(-iwb, p.Ws - iwb, p.U);
          base[sub] = p.src + std::int64_t(n) * p.simg + std::int64_t(ihb) * p.Ws + iwb;
        }
      }
      const int brows = min(p.BN, p.ncols - nt * p.BN);
      for (int ch = 0; ch < p.chunks; ++ch) {
        mbar_wait(&empty[st], ph ^ 1);
        const std::uint32_t sa = sbase + st * stage_bytes, sb = sa + msub * kABytes;
        if (tma_thread) {
          mbar_expect_tx(&full[st], std::uint32_t(p.BN) * 128);
          tma_2d(smem + st * stage_bytes + msub * kABytes, &bmap, &full[st], ch * 32, nt * p.BN);
        }
        // this lane's reduction entry kr = ch*32 + lane: (cs, t, u)
        const int kr = ch * 32 + lane;
        int eoff = 0, etu = (31 << 8) | 31;
        int boff = 0, brt = 1 << 14, bsu = 1 << 14;
        if (kr < p.Kr) {
          std::uint32_t cs, tu, t, uu;
          p.fd_TU.divmod(std::uint32_t(kr), cs, tu);
          p.fd_U.divmod(tu, t, uu);
          eoff = int(cs) * p.HWs + int(t) * p.Ws + int(uu);
          etu = int(t << 8 | uu);
          if (p.bmode == 2) {
            const int tt = p.T - 1 - int(t), ut = p.U - 1 - int(uu);
            brt = tt * p.fsh;
            bsu = ut * p.fsw;
            boff = int(cs) * p.CRS + brt * p.S + bsu;
          } else {
            boff = kr;
            brt = bsu = 0;
          }
        }
        // A: 8 reduction indices x 32 positions, one 128 B smem row each (the
        // swizzle XOR (k & 3) is this warp's js, so destinations are a
        // per-thread base plus immediates); a skipped copy (src-size 0) never
        // dereferences its address
        const std::uint32_t arow = sa + std::uint32_t(pb) * 4096 + std::uint32_t(js) * 128 +
                                   ((std::uint32_t((lane >> 3) ^ js)) << 5) + swz_lane;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int k = js + 4 * i;
          const int off = __shfl_sync(0xffffffffu, eoff, k);
          const int tu = __shfl_sync(0xffffffffu, etu, k);
          const int t = tu >> 8, uu = tu & 255;
          cp_async4(arow + std::uint32_t(i) * 512, base[0] + off, ((vr[0] >> t) & (vs[0] >> uu) & 1u) * 4u);
          if (msub == 2)
            cp_async4(arow + kABytes + std::uint32_t(i) * 512, base[1] + off,
                      ((vr[1] >> t) & (vs[1] >> uu) & 1u) * 4u);
        }
        // B (gathered): rows of this n tile, lane = reduction index
        if (p.bmode != 0 && !p.bres) {
          const std::uint32_t bsw = std::uint32_t(lane >> 2), bl = std::uint32_t(lane & 3) * 4;
          for (int r = pw; r < p.BN; r += kProd) {
            std::uint32_t ok = 0;
            int off = 0;
            if (r < brows) {
              const ColEnt e = ptab[r];
              ok = (kr < p.Kr && brt < e.rl && bsu < e.sl) ? 1u : 0u;
              off = e.woff + boff;
            }
            const std::uint32_t dst = sb + std::uint32_t(r) * 128 + (((bsw ^ std::uint32_t(r & 7))) << 4) + bl;
            cp_async4(dst, p.w + off, ok * 4u);
          }
        }
        cp_async_arrive(&full[st]);
        if (++st == kStages) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------------ MMA issuer
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN) | (1u << 15);  // A MN-major, B K-major
    const std::uint32_t sbase = smem_u32(smem);
    int it = 0, tl = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
      const int acc = tl % p.nacc, use = tl / p.nacc;
      mbar_wait(&tempty[acc], (use & 1) ^ 1);
      tc_fence_after();
      const std::uint32_t dtm = tmem + std::uint32_t(acc * msub * p.BN);
      for (int ch = 0; ch < p.chunks; ++ch, ++it) {
        const int st = it % kStages;
        mbar_wait(&full[st], (it / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          fence_async_smem();  // cp.async (generic proxy) -> tensor core (async proxy)
          const std::uint32_t sa = sbase + st * stage_bytes;
          const std::uint32_t sb = p.bres ? sbase + kStages * stage_bytes + std::uint32_t(ch * p.BN) * 128
                                          : sa + msub * kABytes;
          for (int sub = 0; sub < msub; ++sub)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              mma_tf32(dtm + std::uint32_t(sub * p.BN), desc_mn32(sa + sub * kABytes + j * 1024),
                       umma_desc_sw128(sb + j * 32), idesc, (ch | j) ? 1u : 0u);
          mma_commit(&empty[st]);
          if (ch + 1 == p.chunks) mma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 0-3)
    const int ew = warp;
    int tl = 0, cur_nt = -1;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
      const int mt = u % p.m_tiles, nt = u / p.m_tiles;
      if (nt != cur_nt) {
        named_sync(2, 128);
        for (int j = threadIdx.x; j < p.BN; j += 128)
          if (nt * p.BN + j < p.ncols) etab[j] = col_entry(p, nt * p.BN + j);
        named_sync(2, 128);
        cur_nt = nt;
      }
      const int acc = tl % p.nacc, use = tl / p.nacc;
      mbar_wait_backoff(&tfull[acc], use & 1);
      tc_fence_after();
      const int ncol = min(p.BN, p.ncols - nt * p.BN);
      for (int sub = 0; sub < msub; ++sub) {
      const int m = (mt * msub + sub) * kBM + ew * 32 + lane;
      bool live = m < p.M;
      int h0 = 0, w0 = 0;
      float* obase = p.out;
      if (live) {
        std::uint32_t n, g, gi, gj;
        p.fd_HWg.divmod(std::uint32_t(m), n, g);
        p.fd_Wg.divmod(g, gi, gj);
        h0 = (int(gi) + p.gi0) * p.osh - p.oph;
        w0 = (int(gj) + p.gj0) * p.osw - p.opw;
        obase = p.out + std::int64_t(n) * p.oimg + std::int64_t(h0) * p.Wo + w0;
      }
      const std::uint32_t tbase =
          tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t((acc * msub + sub) * p.BN);
      for (int c0 = 0; c0 < ncol; c0 += 32) {
        float v[32];
        tmem_ld32(tbase + std::uint32_t(c0), v);
        if (!live) continue;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (c0 + j >= ncol) break;
          const ColEnt e = etab[c0 + j];
          if (unsigned(h0 + e.a) < unsigned(p.Ho) && unsigned(w0 + e.b) < unsigned(p.Wo)) {
            float* dst = obase + e.ooff + int(e.a) * p.Wo + e.b;
            const float val = p.alpha * v[j];
            *dst = p.beta == 0.f ? val : val + p.beta * *dst;
          }
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

int pick_bn(int n) {
  const int tiles = (n + kMaxBN - 1) / kMaxBN;
  return ((n + tiles - 1) / tiles + 15) / 16 * 16;
}

// Fills the op-independent fields and launches.
cudaError_t zlaunch(ZParams p, cudaStream_t st) {
  p.BN = pick_bn(p.ncols);
  p.chunks = (p.Kr + 31) / 32;
  // a gathered B of one column tile that fits next to a >= 3-stage A ring
  // stays resident (filled once per CTA: AlexNet / ResNet conv1
  // BackwardData's phase sub-filters) instead of being re-gathered per tile
  const int bres_bytes = p.chunks * p.BN * 128;
  // Exact but not faster (AlexNet conv1 BD 637 vs 610 us, ResNet conv1 BD
  // 3890 vs 2929: the gathers of A, not of B, bound these), so off by default
  p.bres = p.bmode == 2 && p.ncols <= p.BN && bres_bytes + 3 * int(kABytes) <= 200 * 1024 && tune("z_bres", 0);
  // two position sub-tiles per tile once there are enough positions to keep
  // every SM busy with them: each B stage then feeds 2x the MMA work (not
  // needed when B is resident)
  p.msub = tune("z_msub", !p.bres && p.M >= 2 * kBM * 2 * sm_count() ? 2 : 1) == 2 ? 2 : 1;
  p.nacc = 2 * p.msub * p.BN <= 512 ? 2 : 1;
  p.m_tiles = (p.M + p.msub * kBM - 1) / (p.msub * kBM);
  p.n_tiles = (p.ncols + p.BN - 1) / p.BN;
  p.fd_HWg = FastDiv(std::uint32_t(p.Hg * p.Wg));
  p.fd_Wg = FastDiv(std::uint32_t(p.Wg));
  p.fd_TU = FastDiv(std::uint32_t(p.T * p.U));
  p.fd_U = FastDiv(std::uint32_t(p.U));
  CUtensorMap bmap{};
  if (p.bmode == 0) {
    const cuuint64_t dims[2] = {cuuint64_t(p.Kr), cuuint64_t(p.ncols)};
    const cuuint64_t strides[1] = {cuuint64_t(p.Kr) * 4};
    const cuuint32_t box[2] = {32, cuuint32_t(p.BN)};
    const cuuint32_t es[2] = {1, 1};
    if (encode_tiled()(&bmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(p.w), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  if (p.bres && bres_bytes + 2 * p.msub * int(kABytes) > 200 * 1024) p.bres = 0;
  const int stage_bytes = p.msub * int(kABytes) + (p.bres ? 0 : ((p.BN * 128 + 1023) & ~1023));
  const int ring = 200 * 1024 - (p.bres ? bres_bytes : 0);
  p.stages = std::max(2, std::min({kMaxStages, tune("z_stages", 8), ring / stage_bytes}));
  const int smem = p.stages * stage_bytes + (p.bres ? bres_bytes : 0) + 1024 + 256;
  auto kern = p.msub == 2 ? zgemm_kernel<2> : zgemm_kernel<1>;
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int units = p.m_tiles * p.n_tiles;
  const int grid = std::min(units, sm_count());
  trace_variant("zgemm bmode=%d bres=%d m_tiles=%d n_tiles=%d BN=%d msub=%d nacc=%d chunks=%d stages=%d grid=%d",
                p.bmode, p.bres, p.m_tiles, p.n_tiles, p.BN, p.msub, p.nacc, p.chunks, p.stages, grid);
  return launch_pdl(kern, dim3(grid), dim3(kThreads), std::size_t(smem), st, bmap, p);
}

}  // namespace

bool zgemm_supports(int op, const ConvShape& s) {
  if (op == kFwd) {
    return s.R <= 32 && s.S <= 32 && std::int64_t(s.N) * s.OH() * s.OW() < (1ll << 31) &&
           std::int64_t(s.C) * s.H * s.W < (1ll << 31) && std::int64_t(s.K) * s.C * s.R * s.S < (1ll << 31);
  }
  if (op == kBwdData) {
    const int Th = (s.R + s.sh - 1) / s.sh, Tw = (s.S + s.sw - 1) / s.sw;
    const std::int64_t Hg = (s.H - 1 + s.ph) / s.sh + 1, Wg = (s.W - 1 + s.pw) / s.sw + 1;
    return Th <= 32 && Tw <= 32 && std::int64_t(s.N) * Hg * Wg < (1ll << 31) && s.sh * s.sw * s.C < (1 << 15) &&
           std::int64_t(s.K) * s.OH() * s.OW() < (1ll << 31) && std::int64_t(s.C) * s.H * s.W < (1ll << 31) &&
           std::int64_t(s.K) * s.C * s.R * s.S < (1ll << 31) && s.R < (1 << 14) && s.S < (1 << 14);
  }
  return false;
}

cudaError_t zgemm_forward(const ConvShape& s, const float* x, const float* w, float* y, float alpha, float beta,
                          cudaStream_t st) {
  ZParams p{};
  p.src = x; p.w = w; p.out = y; p.alpha = alpha; p.beta = beta;
  p.Cs = s.C; p.Hs = s.H; p.Ws = s.W; p.HWs = s.H * s.W;
  p.simg = std::int64_t(s.C) * s.H * s.W;
  p.Hg = s.OH(); p.Wg = s.OW();
  p.M = s.N * p.Hg * p.Wg;
  p.gsh = s.sh; p.gsw = s.sw; p.gph = s.ph; p.gpw = s.pw;
  p.T = s.R; p.U = s.S;
  p.Kr = s.C * s.R * s.S;
  p.ncols = s.K;
  p.bmode = (p.Kr % 4 == 0 && (reinterpret_cast<std::uintptr_t>(w) & 15) == 0 && tune("z_tma", 1)) ? 0 : 1;
  p.CRS = p.Kr; p.RS = s.R * s.S; p.R = s.R; p.S = s.S; p.fsh = s.sh; p.fsw = s.sw; p.C = s.C;
  p.Ho = p.Hg; p.Wo = p.Wg; p.osh = 1; p.osw = 1; p.oph = 0; p.opw = 0;
  p.oimg = std::int64_t(s.K) * p.Hg * p.Wg;
  p.fd_C = FastDiv(std::uint32_t(s.C));
  p.fd_sw = FastDiv(1);
  return zlaunch(p, st);
}

cudaError_t zgemm_backward_data(const ConvShape& s, const float* dy, const float* w, float* dx, float alpha,
                                float beta, cudaStream_t st) {
  ZParams p{};
  const int Th = (s.R + s.sh - 1) / s.sh, Tw = (s.S + s.sw - 1) / s.sw;
  p.src = dy; p.w = w; p.out = dx; p.alpha = alpha; p.beta = beta;
  p.Cs = s.K; p.Hs = s.OH(); p.Ws = s.OW(); p.HWs = p.Hs * p.Ws;
  p.simg = std::int64_t(s.K) * p.Hs * p.Ws;
  // grid points i with some phase a landing in [0, H): i*sh + a - ph >= 0 for
  // a <= sh - 1 needs i >= ph / sh (floor); i*sh - ph <= H - 1 needs
  // i <= (H - 1 + ph) / sh
  p.gi0 = s.ph / s.sh;
  p.gj0 = s.pw / s.sw;
  p.Hg = (s.H - 1 + s.ph) / s.sh + 1 - p.gi0;
  p.Wg = (s.W - 1 + s.pw) / s.sw + 1 - p.gj0;
  p.M = s.N * p.Hg * p.Wg;
  p.gsh = 1; p.gsw = 1; p.gph = Th - 1; p.gpw = Tw - 1;
  p.T = Th; p.U = Tw;
  p.Kr = s.K * Th * Tw;
  p.ncols = s.sh * s.sw * s.C;
  p.bmode = 2;
  p.CRS = s.C * s.R * s.S; p.RS = s.R * s.S; p.R = s.R; p.S = s.S; p.fsh = s.sh; p.fsw = s.sw; p.C = s.C;
  p.Ho = s.H; p.Wo = s.W; p.osh = s.sh; p.osw = s.sw; p.oph = s.ph; p.opw = s.pw;
  p.oimg = std::int64_t(s.C) * s.H * s.W;
  p.fd_C = FastDiv(std::uint32_t(s.C));
  p.fd_sw = FastDiv(std::uint32_t(s.sw));
  return zlaunch(p, st);
}

}  // namespace ucudnn
