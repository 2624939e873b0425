// UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM_NHWC (8), BackwardFilter of stride-1
// convolutions: TMA im2col boxes of a channels-last x copy and tiled boxes of
// a channels-last dy copy feed tcgen05.mma with *MN-major* operands.
//
//   dW[k][c][r][s] = beta * dW + alpha * sum_{n,oh,ow} dy[n][k][oh][ow] * x[n][c][oh-ph+r][ow-pw+s]
//   (reference_conv.hpp:141-180)
//
// GEMM view: rows = (tap = r*S+s, c) -- R*S*Cp of them, 32-row atoms of one
// (tap, 32-channel chunk) --, columns = k, reduction = output pixels flattened
// over (n, oh, ow). For a 32-pixel reduction step the rows' operand is, per
// atom, exactly one TMA im2col box of the NHWC x copy (32 pixels x 32
// channels, filter offset (r, s), padding by the box's out-of-bounds fill),
// and the columns' operand one tiled box of the NHWC dy copy (32 pixels x BN
// channels). Both land pixel-row-major with the channels contiguous, i.e. the
// reduction axis is the *strided* one: MN-major UMMA operands. For kind::tf32
// those only exist in the 128B swizzle with 32-byte atomicity (CUTLASS
// Layout_MN_SW128_32B_Atom; descriptor layout type 1, 4 K-rows of 128 B per
// atom; scripts/mn_probe.cu), which TMA writes with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B. Compared with the gather kernel
// (bflsu.cu) the operands arrive by TMA at ~2x the L2 -> SM rate, and no
// shifted replicas are needed (bfilter.cu): im2col boxes start at any pixel.
//
// Persistent kernel, one CTA per SM, units = (column tile, row tile, split of
// the reduction), the row tile fastest so the CTAs running at one moment read
// the same pixel range (dy and x stay L2-resident across row tiles). Warps 0,
// 2, 3: TMA producers owning ring stages s % 3; warp 1: TMEM owner + MMA
// issuer (two 256-column accumulators); warps 4-7: epilogue, fp32 RED of the
// accumulator into a [k][row] scratch (32 lanes = 32 consecutive rows), then a
// finalize kernel applies alpha / beta into dW[k][c][r][s].
#include "bfnhwc.h"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "launch.h"
#include "precomp.h"
#include "sm100.cuh"

namespace ucudnn {

using namespace sm100;

namespace {

constexpr int kBM = 128;
constexpr int kMaxBN = 256;
constexpr int kMaxStages = 8;
constexpr int kThreads = 256;

struct NGeo {
  int N, C, H, W, K, R, S, ph, pw, OH, OW, P;
  int Cp, Kp;        // channel counts padded to 32 (one 128 B swizzle row)
  int M;             // GEMM rows R*S*Cp
  int atoms;         // M / 32
  int two;           // CTA pairs (tcgen05 cta_group::2): M = 256 per MMA, dy box split along N
  int msub;          // MMA sub-tiles per CTA tile (2: the dy box feeds twice the MMA work)
  int m_tiles, n_tiles, BN;
  int steps;         // px-pixel reduction steps (over N*P flattened pixels, or per image with dyd)
  int px;            // pixels per ring stage (32 or 64)
  int dyd;           // dy read in place from NCHW as a K-major operand (OH*OW % 4 == 0: 16 B plane pitch)
  int spi;           // dyd: steps per image (the dy box cannot cross images)
  // strided layers run as the stride-1 BackwardFilter of a space-to-depth
  // copy (the fields above then describe that equivalent convolution)
  int s2d, sh, sw, Ah, Bw, C0, R0, S0, H0, W0, ph0, pw0;
};

int round_up(int a, int b) { return (a + b - 1) / b * b; }

NGeo make_geo(const ConvShape& s) {
  NGeo g{};
  g.N = s.N; g.C = s.C; g.H = s.H; g.W = s.W; g.K = s.K; g.R = s.R; g.S = s.S;
  g.ph = s.ph; g.pw = s.pw; g.OH = s.OH(); g.OW = s.OW();
  g.sh = s.sh; g.sw = s.sw; g.C0 = s.C; g.R0 = s.R; g.S0 = s.S; g.H0 = s.H; g.W0 = s.W; g.ph0 = s.ph; g.pw0 = s.pw;
  g.s2d = s.sh > 1 || s.sw > 1;
  if (g.s2d) {
    // with x_a[i] = x_pad[i*sh + a]: dW[k][c][t*sh + a] is the stride-1
    // BackwardFilter of phase-channel (a, b, c) at tap t over a Hq x Wq copy
    // (AlexNet conv1: 3 -> 48 channels, 11 x 11 -> 3 x 3 taps, 57 x 57)
    g.Ah = std::min(s.sh, s.R); g.Bw = std::min(s.sw, s.S);
    g.R = (s.R + s.sh - 1) / s.sh; g.S = (s.S + s.sw - 1) / s.sw;
    g.C = g.Ah * g.Bw * s.C; g.H = g.OH + g.R - 1; g.W = g.OW + g.S - 1; g.ph = 0; g.pw = 0;
  }
  g.P = g.OH * g.OW;
  g.Cp = round_up(g.C, 32);
  g.Kp = round_up(s.K, 32);
  g.M = g.R * g.S * g.Cp;
  g.atoms = g.M / 32;
  // CTA pairs only with two MMA sub-tiles (512-row pair tiles) and only when
  // those pad no more rows than the 1-SM kernel's 256-row tiles: measured
  // (AlexNet BF at 256 images, 1-SM vs pair) conv4 (M = 3456) 233 -> 206 us,
  // but conv2 / conv3 / conv5 with 256-row pair tiles 378 -> 423, 194 -> 220,
  // 144 -> 153 us
  // Round 2 (warp-wide issue, scripts/r02_run85.sh): pairs now also win for
  // >= 192 output channels with 3x3 / 5x5 filters at 256-row pair tiles --
  // conv2 BF at 64 images 414 -> 373 us per 256, conv3 at 128 215 -> 182,
  // conv5 170 -> 150, ResNet l3 195 -> 178 -- but not at 128 channels
  // (ResNet l2 264 -> 297); 1x1 and space-to-depth layers were not measured
  // and keep the padding rule
  const int knob = tune("bfn2", -1);
  const bool pad_pair = round_up(g.M, 4 * kBM) <= round_up(g.M, 2 * kBM);
  const bool wide_pair = g.Kp >= 192 && g.M >= 2 * kBM && g.R * g.S > 1 && !g.s2d;
  g.two = knob >= 0 ? (knob > 0 && g.M >= 2 * kBM) : (pad_pair || wide_pair);
  const int bq = g.two ? 64 : 32;  // pairs: each CTA holds BN/2 columns, whole 32-column blocks
  g.n_tiles = (g.Kp + kMaxBN - 1) / kMaxBN;
  g.BN = round_up((g.Kp + g.n_tiles - 1) / g.n_tiles, bq);
  g.n_tiles = (g.Kp + g.BN - 1) / g.BN;
  const int pair_rows = (g.two ? 2 : 1) * kBM;
  if (g.M <= pair_rows) {
    g.msub = 1;
  } else if (g.two && knob < 0 && pad_pair) {
    g.msub = 2;
  } else {
    // fewest padded rows, ties to 2 sub-tiles (more MMA work per dy box)
    const int r1 = round_up(g.M, pair_rows), r2 = round_up(g.M, 2 * pair_rows);
    g.msub = r2 <= r1 ? 2 : 1;
    const int forced = tune("bfn_msub", 0);
    if (forced == 1 || forced == 2) g.msub = forced;
  }
  g.m_tiles = (g.M + g.msub * pair_rows - 1) / (g.msub * pair_rows);
  // 64-pixel ring stages (more bytes in flight per stage) win for CTA pairs
  // and for 1-sub-tile, <= 64-column tiles (AlexNet conv4 BF at 128 images
  // 90.6 -> 83.1 us; conv1 through space-to-depth at 32 images 63 -> 45 us)
  // and lose with two 128-row sub-tiles (conv3 80 -> 88, conv5 61 -> 66 us,
  // profiles/r01_bfn_px_sweep.txt); never when two stages would not fit
  const int px_knob = tune("bfn_px", 0);
  g.px = px_knob ? (px_knob == 64 ? 64 : 32) : (g.two || (g.msub == 1 && g.BN <= 64)) ? 64 : 32;
  const int stage64 = ((4 * g.msub + g.BN / (g.two ? 64 : 32)) * 64 * 128 + 1023) & ~1023;
  if (g.px == 64 && 2 * stage64 + 1280 > 220 * 1024) g.px = 32;
  // dy's NCHW planes are 16 B aligned when OH*OW % 4 == 0: a {32 px, BN k}
  // tiled box of dy then lands as the standard SWIZZLE_128B K-major operand
  // (pixels contiguous), so dy needs no channels-last copy and the
  // workspace holds only x's copy (ResNet l1-l3: 3136 / 784 / 196 pixels)
  // (dy in place keeps 32-pixel stages: it saves the dy copy, which the
  // default prefers over 64-pixel stages; UCUDNN_TUNE=bfn_px=64 forces the copy)
  g.dyd = g.P % 4 == 0 && px_knob != 64 && tune("bfn_dyd", 1);
  if (g.dyd) g.px = 32;
  g.spi = (g.P + g.px - 1) / g.px;
  g.steps = g.dyd ? g.N * g.spi : int((std::int64_t(g.N) * g.P + g.px - 1) / g.px);
  return g;
}

std::size_t a256(std::size_t b) { return (b + 255) / 256 * 256; }
std::size_t x_bytes(const NGeo& g) { return a256(std::size_t(g.N) * g.H * g.W * g.Cp * 4); }
std::size_t dy_bytes(const NGeo& g) { return g.dyd ? 0 : a256(std::size_t(g.N) * g.P * g.Kp * 4); }
int rows_pad(const NGeo& g) { return g.m_tiles * g.msub * (g.two ? 2 : 1) * kBM; }
std::size_t acc_bytes(const NGeo& g) { return a256(std::size_t(g.K) * rows_pad(g) * 4); }

struct NParams {
  float* acc;  // [K][rpad] fp32 partial sums
  int C, Cp, K, S, RS, M, atoms, cch, BN, rpad, ph, pw;
  int m_tiles, tiles, splits, steps, steps_per_unit, stages, px, msub, nacc, dyd, P;
  FastDiv fd_spi;
  FastDiv fd_P, fd_OW;
};

__device__ __forceinline__ void tma_3d(void* dst, const void* tmap, std::uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// MN-major descriptor, 128B swizzle with 32 B atoms: `lbo` = byte stride
// between 32-element MN blocks, SBO = 512 (4 K-rows of 128 B per atom).
__device__ __forceinline__ std::uint64_t desc_mn32(std::uint32_t saddr, std::uint32_t lbo) {
  std::uint64_t d = 0;
  d |= std::uint64_t((saddr >> 4) & 0x3FFF);
  d |= std::uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= std::uint64_t(512 >> 4) << 32;
  d |= std::uint64_t(1) << 46;
  d |= std::uint64_t(1) << 61;
  return d;
}

__global__ void __launch_bounds__(kThreads, 1)
    bfn_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap dmap, const NParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t blk = std::uint32_t(p.px) * 128;  // one 32-channel block of px pixel rows
  const std::uint32_t a_bytes = 4 * p.msub * blk;
  const std::uint32_t b_bytes = std::uint32_t(p.BN / 32) * blk;
  const std::uint32_t stage_bytes = (a_bytes + b_bytes + 1023) & ~1023u;
  const int kStages = p.stages;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kStages * stage_bytes);
  std::uint64_t* empty = full + kMaxStages;
  std::uint64_t* tfull = empty + kMaxStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);

  if (threadIdx.x == 0) {
    prefetch_tmap(&xmap);
    prefetch_tmap(&dmap);
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
  const std::uint32_t tmem = tmem_base_uniform(tmem_slot);
  pdl_wait();
  pdl_trigger();
  const int units = p.tiles * p.splits;

  if (warp == 0 || warp == 2 || warp == 3) {
    const int pq = warp == 0 ? 0 : warp - 1;
    const int nprod = kStages < 3 ? kStages : 3;
    if (lane == 0) {
      // ------------------------------------------------ TMA producers
      int it = 0;
      RingOwner ro;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int tile = u % p.tiles, split = u / p.tiles;
        const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
        const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
        for (int g = g0; g < g1; ++g, ++it, ro.step(kStages, nprod)) {
          if (ro.own != pq) continue;
          const int st = ro.slot;
          mbar_wait(&empty[st], ro.ph ^ 1);
          mbar_expect_tx(&full[st], a_bytes + b_bytes);
          unsigned char* sa = smem + st * stage_bytes;
          // first output pixel of the step -> im2col start (its window corner)
          std::uint32_t n, pix, oh, ow, q0;
          if (p.dyd) {
            std::uint32_t j;
            p.fd_spi.divmod(std::uint32_t(g), n, j);
            pix = j * std::uint32_t(p.px);
            q0 = n * std::uint32_t(p.P) + pix;
          } else {
            q0 = std::uint32_t(g) * std::uint32_t(p.px);
            p.fd_P.divmod(q0, n, pix);
          }
          p.fd_OW.divmod(pix, oh, ow);
          const int cw = int(ow) - p.pw, ch = int(oh) - p.ph;
#pragma unroll 1
          for (int i = 0; i < 4 * p.msub; ++i) {
            // atoms past the last (tap, chunk) re-load the last one: their
            // rows are dropped by the epilogue
            const int a = min(mt * 4 * p.msub + i, p.atoms - 1);
            const int tap = a / p.cch, cc = a - tap * p.cch;
            const int r = tap / p.S, s = tap - r * p.S;
            tma_im2col_4d(sa + i * blk, &xmap, &full[st], cc * 32, cw, ch, int(n), (unsigned short)s,
                          (unsigned short)r);
          }
          if (p.dyd) tma_3d(sa + a_bytes, &dmap, &full[st], int(pix), nt * p.BN, int(n));
          else tma_3d(sa + a_bytes, &dmap, &full[st], 0, int(q0), nt * (p.BN / 32));
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN) | (1u << 15) | (p.dyd ? 0u : (1u << 16));
    const std::uint32_t sbase = smem_u32(smem);
    const int ksub = p.px / 8;
    int it = 0, tl = 0;
    RingPos rp;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
      const int split = u / p.tiles;
      const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
      const int acc = tl % p.nacc, use = tl / p.nacc;
      mbar_wait(&tempty[acc], (use & 1) ^ 1);
      tc_fence_after();
      const std::uint32_t dtm = tmem + std::uint32_t(acc * p.msub * p.BN);
      for (int g = g0; g < g1; ++g, ++it, rp.step(kStages)) {
        const int st = rp.slot;
        mbar_wait(&full[st], rp.ph);
        tc_fence_after();
        if (lane == 0) {
          const std::uint32_t sa = sbase + st * stage_bytes, sb = sa + a_bytes;
          for (int m = 0; m < p.msub; ++m)
            for (int j = 0; j < ksub; ++j)
              mma_tf32(dtm + std::uint32_t(m * p.BN), desc_mn32(sa + m * 4 * blk + j * 1024, blk),
                       p.dyd ? umma_desc_sw128(sb + j * 32) : desc_mn32(sb + j * 1024, blk), idesc,
                       (g != g0 || j != 0) ? 1u : 0u);
          mma_commit(&empty[st]);
          if (g + 1 >= g1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
      if (g1 <= g0 && lane == 0) mma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue: RED into acc[k][row]
    const int ew = warp - 4;
    int tl = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
      const int tile = u % p.tiles, split = u / p.tiles;
      const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
      const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
      const int acc = tl % p.nacc, use = tl / p.nacc;
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      for (int m = 0; m < p.msub; ++m) {
        const std::uint32_t tbase =
            tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t((acc * p.msub + m) * p.BN);
        const int row = (mt * p.msub + m) * kBM + ew * 32 + lane;
        const bool live = g1 > g0 && row < p.M && (row % p.Cp) < p.C;
        for (int c0 = 0; c0 < p.BN; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + std::uint32_t(c0), v);
          if (!live) continue;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int k = nt * p.BN + c0 + j;
            if (k >= p.K) break;
            red_add(p.acc + std::int64_t(k) * p.rpad + row, v[j]);
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

__device__ __forceinline__ void tma_3d_2sm(void* dst, const void* tmap, std::uint32_t bar_cluster, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(bar_cluster), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// CTA-pair version (tcgen05.mma.cta_group::2): per MMA sub-tile 256 rows,
// 128 from each CTA's own im2col boxes; each CTA loads half of the dy box
// (BN/2 columns), so per SM a step moves (4 * msub + BN/64) blocks instead of
// (4 * msub + BN/32). Rank 0 issues the MMAs; both CTAs' TMA bytes count on
// its full barriers; commits multicast to both CTAs; both epilogues release
// rank 0's accumulator barrier (as bf2_kernel in bfilter.cu).
__global__ void __launch_bounds__(kThreads, 1)
    bfn2_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap dmap, const NParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t rank = cluster_rank();
  const std::uint32_t blk = std::uint32_t(p.px) * 128;
  const std::uint32_t a_bytes = 4 * p.msub * blk;
  const std::uint32_t b_bytes = std::uint32_t(p.BN / 64) * blk;
  const std::uint32_t stage_bytes = (a_bytes + b_bytes + 1023) & ~1023u;
  const int kStages = p.stages;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kStages * stage_bytes);
  std::uint64_t* empty = full + kMaxStages;
  std::uint64_t* tfull = empty + kMaxStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  if (threadIdx.x == 0) {
    prefetch_tmap(&xmap);
    prefetch_tmap(&dmap);
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
  cluster_sync();
  tc_fence_after();
  const std::uint32_t tmem = tmem_base_uniform(tmem_slot);
  const int units = p.tiles * p.splits;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0 || warp == 2 || warp == 3) {
    const int pq = warp == 0 ? 0 : warp - 1;
    const int nprod = kStages < 3 ? kStages : 3;
    if (lane == 0) {
      int it = 0;
      RingOwner ro;
      for (int u = cid; u < units; u += ncl) {
        const int tile = u % p.tiles, split = u / p.tiles;
        const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
        const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
        for (int g = g0; g < g1; ++g, ++it, ro.step(kStages, nprod)) {
          if (ro.own != pq) continue;
          const int st = ro.slot;
          mbar_wait(&empty[st], ro.ph ^ 1);
          if (rank == 0) mbar_expect_tx(&full[st], 2u * (a_bytes + b_bytes));
          const std::uint32_t bar = mapa(smem_u32(&full[st]), 0);
          unsigned char* sa = smem + st * stage_bytes;
          std::uint32_t n, pix, oh, ow, q0;
          if (p.dyd) {
            std::uint32_t j;
            p.fd_spi.divmod(std::uint32_t(g), n, j);
            pix = j * std::uint32_t(p.px);
            q0 = n * std::uint32_t(p.P) + pix;
          } else {
            q0 = std::uint32_t(g) * std::uint32_t(p.px);
            p.fd_P.divmod(q0, n, pix);
          }
          p.fd_OW.divmod(pix, oh, ow);
          const int cw = int(ow) - p.pw, ch = int(oh) - p.ph;
#pragma unroll 1
          for (int m = 0; m < p.msub; ++m) {
            const int a0 = (((mt * p.msub + m) * 2 + int(rank)) * kBM) / 32;
#pragma unroll 1
            for (int i = 0; i < 4; ++i) {
              const int a = min(a0 + i, p.atoms - 1);
              const int tap = a / p.cch, cc = a - tap * p.cch;
              const int r = tap / p.S, s = tap - r * p.S;
              tma_im2col_4d_2sm(sa + (m * 4 + i) * blk, &xmap, bar, cc * 32, cw, ch, int(n), (unsigned short)s,
                                (unsigned short)r);
            }
          }
          if (p.dyd) tma_3d_2sm(sa + a_bytes, &dmap, bar, int(pix), nt * p.BN + int(rank) * (p.BN / 2), int(n));
          else tma_3d_2sm(sa + a_bytes, &dmap, bar, 0, int(q0), nt * (p.BN / 32) + int(rank) * (p.BN / 64));
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (rank == 0) {
      const std::uint32_t idesc = idesc_tf32(2 * kBM, p.BN) | (1u << 15) | (p.dyd ? 0u : (1u << 16));
      const std::uint32_t sbase = smem_u32(smem);
      const int ksub = p.px / 8;
      int it = 0, tl = 0;
    RingPos rp;
      for (int u = cid; u < units; u += ncl, ++tl) {
        const int split = u / p.tiles;
        const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
        const int acc = tl % p.nacc, use = tl / p.nacc;
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const std::uint32_t dtm = tmem + std::uint32_t(acc * p.msub * p.BN);
        for (int g = g0; g < g1; ++g, ++it, rp.step(kStages)) {
          const int st = rp.slot;
          mbar_wait(&full[st], rp.ph);
          tc_fence_after();
          if (lane == 0) {
            const std::uint32_t sa = sbase + st * stage_bytes, sb = sa + a_bytes;
            for (int m = 0; m < p.msub; ++m)
              for (int j = 0; j < ksub; ++j)
                mma_tf32_2sm(dtm + std::uint32_t(m * p.BN), desc_mn32(sa + m * 4 * blk + j * 1024, blk),
                             p.dyd ? umma_desc_sw128(sb + j * 32) : desc_mn32(sb + j * 1024, blk), idesc,
                             (g != g0 || j != 0) ? 1u : 0u);
            mma_commit_2sm(&empty[st], 3);
            if (g + 1 >= g1) mma_commit_2sm(&tfull[acc], 3);
          }
          __syncwarp();
        }
        if (g1 <= g0 && lane == 0) mma_commit_2sm(&tfull[acc], 3);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const std::uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), 0);
    int tl = 0;
    for (int u = cid; u < units; u += ncl, ++tl) {
      const int tile = u % p.tiles, split = u / p.tiles;
      const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
      const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
      const int acc = tl % p.nacc, use = tl / p.nacc;
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      for (int m = 0; m < p.msub; ++m) {
        const std::uint32_t tbase =
            tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t((acc * p.msub + m) * p.BN);
        const int row = ((mt * p.msub + m) * 2 + int(rank)) * kBM + ew * 32 + lane;
        const bool live = g1 > g0 && row < p.M && (row % p.Cp) < p.C;
        for (int c0 = 0; c0 < p.BN; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + std::uint32_t(c0), v);
          if (!live) continue;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int k = nt * p.BN + c0 + j;
            if (k >= p.K) break;
            red_add(p.acc + std::int64_t(k) * p.rpad + row, v[j]);
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
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_free_2sm<512>(tmem);
  }
}

// NCHW -> N(HW)Cp with zero channels C..Cp-1: 64 pixels x 32 channels per
// block, coalesced reads along pixels, float4 stores along channels.
__global__ void __launch_bounds__(256) nhwc_kernel(const float* __restrict__ src, float* __restrict__ dst, int C,
                                                   int HW, int Cp) {
  pdl_wait();
  pdl_trigger();
  __shared__ float tile[32][65];
  const int n = blockIdx.z;
  const int p0 = blockIdx.x * 64, c0 = blockIdx.y * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* s = src + std::int64_t(n) * C * HW;
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
    if (pp < HW)
      *reinterpret_cast<float4*>(d + std::int64_t(pp) * Cp + c0 + 4 * q) =
          make_float4(tile[4 * q][pl], tile[4 * q + 1][pl], tile[4 * q + 2][pl], tile[4 * q + 3][pl]);
  }
}

struct NFinal {
  const float* acc;
  float* dw;
  float alpha, beta;
  int C, Cp, RS, rpad;
  std::int64_t n;
  int s2d, S, sh, sw, Bw, Tw;  // s2d: dW[k][c][r][s] from phase-channel (r % sh, s % sw, c) at tap (r / sh, s / sw)
  FastDiv fd_RS, fd_C;        // 32-bit index math (dW has < 2^31 elements): the 64-bit % and / made this an
                              // instruction-bound kernel
};

// dW[k][c][r][s] = beta * dW + alpha * acc[k][(r*S+s)*Cp + c]
__global__ void __launch_bounds__(256) bfn_finalize_kernel(const NFinal f) {
  pdl_wait();
  pdl_trigger();
  const std::uint32_t n = std::uint32_t(f.n);
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    std::uint32_t t, tap_, k_, c_;
    f.fd_RS.divmod(i, t, tap_);
    f.fd_C.divmod(t, k_, c_);
    const int tap = int(tap_), c = int(c_), k = int(k_);
    int row = tap * f.Cp + c;
    if (f.s2d) {
      const int r = tap / f.S, s = tap - r * f.S;
      const int tr = r / f.sh, a = r - tr * f.sh, ts = s / f.sw, b = s - ts * f.sw;
      row = (tr * f.Tw + ts) * f.Cp + (a * f.Bw + b) * f.C + c;
    }
    const float v = f.acc[std::int64_t(k) * f.rpad + row];
    f.dw[i] = f.beta == 0.f ? f.alpha * v : f.alpha * v + f.beta * f.dw[i];
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

}  // namespace

bool bfn_supports(const ConvShape& s) {
  // stride 1 (the im2col walk would need traversal strides), whole 32-channel
  // chunks of x (a padded copy of 3-channel inputs would be 90 % zeros),
  // 32-bit flattened pixel coordinates. Strided layers go through a
  // space-to-depth copy when that shrinks the work: few input channels
  // (AlexNet / ResNet conv1) or 1x1 filters (ResNet strided shortcuts)
  const bool base = s.R <= 16 && s.S <= 16 && s.ph < s.R && s.pw < s.S &&
                    std::int64_t(s.N) * s.OH() * s.OW() + 64 < (std::int64_t(1) << 31) && tune("bfn", 1);
  if (!base) return false;
  if (s.sh == 1 && s.sw == 1) return s.C % 32 == 0;
  const NGeo g = make_geo(s);
  // the s2d row copy keeps Wq * sw columns of each input row
  return (s.C < 32 || (s.R == 1 && s.S == 1 && s.C % 32 == 0)) && s.sh <= 8 && s.sw <= 8 &&
         g.W * s.sw >= s.pw + s.W && g.R <= 16 && g.S <= 16 && tune("bfn_s2d", 1);
}

std::int64_t bfn_workspace(const ConvShape& s) {
  const NGeo g = make_geo(s);
  return std::int64_t(acc_bytes(g) + x_bytes(g) + dy_bytes(g));
}

cudaError_t bfn_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha,
                    float beta, cudaStream_t st, int flags) {
  const NGeo g = make_geo(s);
  float* acc = static_cast<float*>(ws);
  float* xn = reinterpret_cast<float*>(static_cast<char*>(ws) + acc_bytes(g));
  float* dyn = reinterpret_cast<float*>(static_cast<char*>(ws) + acc_bytes(g) + x_bytes(g));
  // the [k][row] scratch depends only on the filter shape, so a run of
  // micro-batches keeps accumulating into it and finalizes once
  cudaError_t e = cudaSuccess;
  if (!(flags & kAccumulate)) e = cudaMemsetAsync(acc, 0, std::size_t(g.K) * rows_pad(g) * 4, st);
  if (e != cudaSuccess) return e;
  const int HW = g.H * g.W;
  if (g.s2d)
    e = space_to_depth_nhwc(x, xn, g.N, g.C0, g.H0, g.W0, g.sh, g.sw, g.ph0, g.pw0, g.Ah, g.Bw, g.H, g.W, g.Cp, st);
  else
    e = launch_pdl(nhwc_kernel, dim3((HW + 63) / 64, g.Cp / 32, g.N), dim3(256), 0, st, x, xn, g.C, HW, g.Cp);
  if (e != cudaSuccess) return e;
  if (!g.dyd) {
    e = launch_pdl(nhwc_kernel, dim3((g.P + 63) / 64, g.Kp / 32, g.N), dim3(256), 0, st, dy, dyn, g.K, g.P, g.Kp);
    if (e != cudaSuccess) return e;
  }

  CUtensorMap xmap, dmap;
  {
    const cuuint64_t dims[4] = {cuuint64_t(g.Cp), cuuint64_t(g.W), cuuint64_t(g.H), cuuint64_t(g.N)};
    const cuuint64_t strides[3] = {cuuint64_t(g.Cp) * 4, cuuint64_t(g.Cp) * 4 * g.W,
                                   cuuint64_t(g.Cp) * 4 * g.W * g.H};
    const int lower[2] = {-g.pw, -g.ph};
    const int upper[2] = {g.pw - (g.S - 1), g.ph - (g.R - 1)};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode_im2col()(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, xn, dims, strides, lower, upper, 32,
                                 cuuint32_t(g.px), estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    int drv = 0;
    cudaDriverGetVersion(&drv);
    if (drv <= 13010 && std::size_t(g.N) * HW * g.Cp * 4 < 131072)  // encoder quirk (as in precomp.cu)
      reinterpret_cast<std::uint64_t*>(&xmap)[1] &= ~(1ull << 21);
  }
  if (g.dyd) {
    if (reinterpret_cast<std::uintptr_t>(dy) & 15) return cudaErrorMisalignedAddress;  // TMA base alignment
    // dy in place: (pixel, k, n), a {32 px, BN(/2) k, 1} box = K-major rows
    const cuuint64_t dims[3] = {cuuint64_t(g.P), cuuint64_t(g.K), cuuint64_t(g.N)};
    const cuuint64_t strides[2] = {cuuint64_t(g.P) * 4, cuuint64_t(g.P) * g.K * 4};
    const cuuint32_t box[3] = {32, cuuint32_t(g.two ? g.BN / 2 : g.BN), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_tiled()(&dmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(dy), dims, strides, box,
                                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  } else {
    // dy_nhwc as (k in chunk, pixel, chunk): a {32, px, BN/32} box lands as
    // BN/32 blocks of [px rows][32 channels] -- the MN-major B operand
    const cuuint64_t dims[3] = {32, cuuint64_t(std::int64_t(g.N) * g.P), cuuint64_t(g.Kp / 32)};
    const cuuint64_t strides[2] = {cuuint64_t(g.Kp) * 4, 128};
    const cuuint32_t box[3] = {32, cuuint32_t(g.px), cuuint32_t(g.BN / (g.two ? 64 : 32))};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_tiled()(&dmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dyn, dims, strides, box, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }

  const int sms = sm_count();
  NParams p{};
  p.acc = acc;
  p.C = g.C; p.Cp = g.Cp; p.K = g.K; p.S = g.S; p.RS = g.R * g.S; p.M = g.M; p.atoms = g.atoms;
  p.cch = g.Cp / 32; p.BN = g.BN; p.rpad = rows_pad(g); p.ph = g.ph; p.pw = g.pw;
  p.m_tiles = g.m_tiles;
  p.tiles = g.m_tiles * g.n_tiles;
  p.steps = g.steps;
  p.px = g.px;
  p.msub = g.msub;
  p.nacc = 2 * g.msub * g.BN <= 512 ? 2 : 1;
  p.fd_P = FastDiv(std::uint32_t(g.P));
  p.dyd = g.dyd;
  p.P = g.P;
  p.fd_spi = FastDiv(std::uint32_t(g.spi));
  p.fd_OW = FastDiv(std::uint32_t(g.OW));
  // split the reduction so the tiles fill the SMs (or SM pairs) once, >= 8 steps per unit
  const int slots = g.two ? sms / 2 : sms;
  const int splits =
      deterministic() ? 1 : std::max(1, std::min(p.steps / 8, tune("bfn_waves", 1) * slots / p.tiles));
  p.steps_per_unit = (p.steps + splits - 1) / splits;
  p.splits = (p.steps + p.steps_per_unit - 1) / p.steps_per_unit;
  const int stage_bytes = ((4 * g.msub + g.BN / (g.two ? 64 : 32)) * g.px * 128 + 1023) & ~1023;
  p.stages = std::max(2, std::min({kMaxStages, tune("bfn_stages", 8), (200 * 1024) / stage_bytes}));
  const int smem = p.stages * stage_bytes + 1024 + 256;
  e = set_smem_attr(reinterpret_cast<const void*>(bfn_kernel), 220 * 1024);
  if (e == cudaSuccess) e = set_smem_attr(reinterpret_cast<const void*>(bfn2_kernel), 220 * 1024);
  if (e != cudaSuccess) return e;
  const int units = p.tiles * p.splits;
  trace_variant("%s tiles=%d splits=%d units=%d msub=%d px=%d dyd=%d s2d=%d acc=%d defer=%d", g.two ? "bfn2" : "bfn",
                p.tiles, p.splits, units, p.msub, p.px, int(g.dyd), int(g.s2d), (flags & kAccumulate) ? 1 : 0,
                (flags & kDeferFinal) ? 1 : 0);
  if (g.two) {
    count_launch();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * std::min(slots, units));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = std::size_t(smem);
    cfg.stream = st;
    cudaLaunchAttribute cat[1];
    cat[0].id = cudaLaunchAttributeClusterDimension;
    cat[0].val.clusterDim.x = 2;
    cat[0].val.clusterDim.y = 1;
    cat[0].val.clusterDim.z = 1;
    cfg.attrs = cat;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, bfn2_kernel, xmap, dmap, p);
  } else {
    e = launch_pdl(bfn_kernel, dim3(std::min(units, sms)), dim3(kThreads), std::size_t(smem), st, xmap, dmap, p);
  }
  if (e != cudaSuccess) return e;
  if (flags & kDeferFinal) return cudaSuccess;

  NFinal f{};
  f.acc = acc;
  f.dw = dw;
  f.alpha = alpha;
  f.beta = beta;
  f.C = g.C0; f.Cp = g.Cp; f.RS = g.R0 * g.S0; f.rpad = rows_pad(g);
  f.n = std::int64_t(g.K) * g.C0 * g.R0 * g.S0;
  f.s2d = g.s2d; f.S = g.S0; f.sh = g.sh; f.sw = g.sw; f.Bw = g.Bw; f.Tw = g.S;
  f.fd_RS = FastDiv(std::uint32_t(f.RS));
  f.fd_C = FastDiv(std::uint32_t(f.C));
  return launch_pdl(bfn_finalize_kernel, dim3(int(std::min<std::int64_t>((f.n + 255) / 256, 8 * sms))), dim3(256),
                    0, st, f);
}

}  // namespace ucudnn
