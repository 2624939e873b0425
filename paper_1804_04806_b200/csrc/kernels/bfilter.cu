// UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM, BackwardFilter: a tcgen05 GEMM whose
// operands are fetched by plain TMA *tiled* loads -- no im2col buffer.
//
//   dW[k][c][r][s] += alpha * sum_{n,oh,ow} dy[n][k][oh][ow] * x[n][c][oh*sh-ph+r][ow*sw-pw+s]
//   (reference_conv.hpp:141-171; beta applied once up front, :173-180)
//
// tcgen05 kind::tf32 only executes K-major operands,
// so the reduction axis -- output pixels -- must be the contiguous one in
// shared memory. NCHW already has pixels contiguous; what stops TMA is the
// 16-byte stride rule (rows of 27 / 13 / 55 floats) and the conv geometry.
// Two cheap, HBM-bound re-layouts in the workspace fix both:
//
//   x_ph[n][cc][Hq*Wq]  cc = (a, b, c): the zero-padded input split into
//                       its (sh x sw) stride phases (only phases a < R,
//                       b < S are kept), plane i*Wq + j = x_pad[i*sh+a][j*sw+b]
//   dy_p[n][k][OH*Wq]   dy with rows re-pitched from OW to Wq, zero in
//                       columns ow >= OW
//
// In these layouts output pixel (oh, ow) sits at flat position
// j = oh*Wq + ow of dy_p, and its tap (r, s) = (qh*sh + a, qw*sw + b) reads
// x_ph plane (a, b, c) at j + qh*Wq + qw. So for a fixed (qh, qw) the A
// operand of a 32-pixel reduction step is a dense [channels x 32] box of
// x_ph at a shifted flat coordinate, and the B operand a dense [k x 32] box
// of dy_p: each lands in shared memory as the SWIZZLE_128B K-major UMMA
// layout directly. The padded columns of dy_p are zero, so whatever x_ph
// holds under them contributes nothing; TMA's out-of-bounds zero fill
// covers every other edge. GEMM rows are (qh, qw, cc) -- for strided convs
// all phases of one shifted window share one box (AlexNet conv1: 48 rows).
// TMA requires the innermost start coordinate to be 16-byte aligned (a
// misaligned one is an illegal instruction on this part), so x_ph is stored
// as T <= 4 replicas shifted by 0..T-1 elements and a tap offset o reads
// replica (o mod 4) at o rounded down; with Qw < 4 the pitch Wq is rounded
// to a multiple of 4 so only T = Qw replicas exist.
//
// Persistent kernel, one CTA per SM, split-K over (image, 32-pixel step)
// units, 256 threads: warp 0 = TMA producer over a 4-stage mbarrier ring,
// warp 1 = TMEM owner + MMA issuer (two 256-column accumulators), warps 4-7
// = epilogue (TMEM -> fp32 RED into dW), overlapping the next unit.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "bfilter.h"
#include "bflsu.h"
#include "conv_common.h"
#include "launch.h"
#include "sm100.cuh"

namespace ucudnn {
using namespace sm100;

namespace {

constexpr int kBM = 128;
// ring depth that splits evenly over 3 or 2 producer threads
inline int ring_stages(int fit) { return fit > 8 ? 8 : fit < 2 ? 2 : fit; }
constexpr int kMaxStages = 8;
constexpr int kMaxSub = 2;  // 32-pixel reduction chunks per stage
constexpr int kThreads = 256;
constexpr int kMaxBN = 256;

struct BfGeo {
  int N, C, H, W, K, R, S, ph, pw, sh, sw, OH, OW;
  int Ah, Bw, Qh, Qw;  // phases kept, tap offsets per phase
  int CC, CCp, Gb;     // phase-channels, padded to a multiple of Gb, rows per box
  int Hq, Wq, Lq, Lp;  // phase plane: rows, pitch, length, padded length (x 4 floats)
  int T;               // shifted replicas of x_ph (TMA start coordinates are 16 B aligned)
  int Ld, Ldp;         // dy_p plane: OH*Wq and its padded length
  int Lc;              // 32-pixel reduction steps per image
  int M, BN, m_tiles, n_tiles;
  int swap;            // 1: MMA rows = output channels k (K <= 128), columns = (q, cc) rows
  int Kb;              // swap: dy box rows (K rounded to 8; MMA rows past it are never read)
  int x_direct, dy_direct;  // the re-layout would be an identity copy (1x1 stride-1 convs): TMA reads x / dy
};

int round_up(int a, int b) { return (a + b - 1) / b * b; }

BfGeo make_geo(const ConvShape& s) {
  BfGeo g{};
  g.N = s.N; g.C = s.C; g.H = s.H; g.W = s.W; g.K = s.K; g.R = s.R; g.S = s.S;
  g.ph = s.ph; g.pw = s.pw; g.sh = s.sh; g.sw = s.sw; g.OH = s.OH(); g.OW = s.OW();
  g.Ah = std::min(s.sh, s.R);
  g.Bw = std::min(s.sw, s.S);
  g.Qh = (s.R + s.sh - 1) / s.sh;
  g.Qw = (s.S + s.sw - 1) / s.sw;
  g.CC = g.Ah * g.Bw * s.C;
  // rows per TMA box = largest power of two <= 128 dividing CCp: pad small
  // channel counts to a power of two (MMA rows are cheaper than TMA boxes)
  if (g.CC < 128) {
    g.CCp = 8;
    while (g.CCp < g.CC) g.CCp <<= 1;
  } else {
    g.CCp = round_up(g.CC, 32);
  }
  g.Gb = 128;
  while (g.CCp % g.Gb) g.Gb >>= 1;
  g.Hq = (s.H + 2 * s.ph + s.sh - 1) / s.sh;
  g.Wq = (s.W + 2 * s.pw + s.sw - 1) / s.sw;
  // A tap offset qh*Wq + qw needs replica (offset mod 4). With a pitch that
  // is a multiple of 4 only qw mod 4 matters (Qw replicas); with >= 4 column
  // offsets all four are needed anyway, so keep the tight pitch.
  if (g.Qw < 4 && g.Qh * g.Qw > 1) {
    g.Wq = round_up(g.Wq, 4);
    g.T = g.Qw;
  } else {
    g.T = g.Qh * g.Qw > 1 ? 4 : 1;
  }
  g.Lq = g.Hq * g.Wq;
  g.Lp = round_up(g.Lq, 4);
  g.Ld = g.OH * g.Wq;
  g.Ldp = round_up(g.Ld, 4);
  g.Lc = (g.Ld + 31) / 32;
  g.M = g.Qh * g.Qw * g.CCp;
  g.x_direct = s.sh == 1 && s.sw == 1 && s.ph == 0 && s.pw == 0 && g.T == 1 && g.Wq == s.W && g.Hq == s.H &&
               g.Lp == g.Lq;
  g.dy_direct = g.Wq == g.OW && g.Ldp == g.Ld;
  // Few output channels (AlexNet conv1, ResNet stage 1: K = 64): an N = 64
  // MMA is issue-bound, so swap roles -- MMA rows are the K channels (one
  // 128-row tile, zero-filled past K) and the (q, cc) rows become N <= 256.
  g.swap = s.K <= 128 && g.M > 128;
  if (g.swap) {
    g.n_tiles = (g.M + kMaxBN - 1) / kMaxBN;
    g.BN = round_up((g.M + g.n_tiles - 1) / g.n_tiles, std::max(g.Gb, 16));
    g.n_tiles = (g.M + g.BN - 1) / g.BN;
    g.m_tiles = 1;
    g.Kb = round_up(s.K, 8);
    return g;
  }
  const int nt = (s.K + kMaxBN - 1) / kMaxBN;
  g.BN = round_up((s.K + nt - 1) / nt, 16);
  g.n_tiles = (s.K + g.BN - 1) / g.BN;
  g.m_tiles = (g.M + kBM - 1) / kBM;
  return g;
}

std::size_t a256(std::size_t b) { return (b + 255) / 256 * 256; }
std::size_t x_bytes(const BfGeo& g) { return g.x_direct ? 0 : a256(std::size_t(g.T) * g.N * g.CC * g.Lp * 4); }
std::size_t dy_bytes(const BfGeo& g) { return g.dy_direct ? 0 : a256(std::size_t(g.N) * g.K * g.Ldp * 4); }
// RED scratch in the GEMM's own layout ([k][x row], or [x row][k] when the
// roles are swapped), so a warp's 32 lanes reduce into 32 consecutive floats
// -- one L2 transaction instead of 32 scattered ones into dW[k][c][r][s].
int rows_pad(const BfGeo& g) { return g.swap ? g.n_tiles * g.BN : (g.m_tiles + 1) / 2 * 2 * kBM; }
int cols_pad(const BfGeo& g) { return g.swap ? kBM : g.n_tiles * g.BN; }
std::size_t acc_bytes(const BfGeo& g) { return a256(std::size_t(rows_pad(g)) * cols_pad(g) * 4); }

struct BfParams {
  float* dw;
  float alpha;
  int K, CRS, RS, S, R, C, Bw, Ah, sh, sw, Qw, CCp, CC, Gb, Wq, M, BN;
  int m_tiles, tiles, splits, steps, steps_per_unit, Lc, T, stages, swap, Kb, ksub, prof;
  float* acc;  // RED scratch: non-swap [k][row] (pitch rpad), swap [row][k] (pitch 128)
  int rpad;
};

// GEMM row (qh, qw, cc) of the x operand -> dW offset (c, r, s), or -1
__device__ __forceinline__ int x_row_off(const BfParams& p, int row) {
  if (row >= p.M) return -1;
  const int q = row / p.CCp, cc = row - q * p.CCp;
  const int qh = q / p.Qw, qw = q - qh * p.Qw;
  if (cc >= p.CC) return -1;
  const int ab = cc / p.C, c = cc - ab * p.C;
  const int a = ab / p.Bw, b = ab - a * p.Bw;
  const int r = qh * p.sh + a, s = qw * p.sw + b;
  return (r < p.R && s < p.S) ? c * p.RS + r * p.S + s : -1;
}

__device__ __forceinline__ void tma_4d(void* dst, const void* tmap, std::uint64_t* bar, int x, int y, int z, int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "r"(w)
      : "memory");
}

__device__ unsigned long long g_bfprof[1024 * 4];

__global__ void __launch_bounds__(kThreads, 1)
    bf_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap dmap, const BfParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t a_bytes = kBM * 128;
  const std::uint32_t b_bytes = std::uint32_t(p.BN) * 128;
  const std::uint32_t sub_bytes = a_bytes + ((b_bytes + 1023) & ~1023u);
  const int kSub = p.ksub;
  const std::uint32_t stage_bytes = kSub * sub_bytes;
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
  pdl_wait();  // everything above touched only smem / TMEM / the param-space tensor maps
  pdl_trigger();
  const int units = p.tiles * p.splits;

  if (warp == 0 || warp == 2 || warp == 3) {
    // up to three producer threads, stage s owned by thread s % 3 (one
    // thread's TMA issue stream keeps only about one stage in flight:
    // scripts/tma_probe.cu). Fixed ownership keeps every stage's parity
    // waits in order, so no producer can run two rounds ahead on a stage.
    const int pq = warp == 0 ? 0 : warp - 1;
    const int nprod = kStages < 3 ? kStages : 3;
    if (lane == 0) {
      // ------------------------------------------------ TMA producer
      const int boxes = kBM / p.Gb;
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int tile = u % p.tiles, split = u / p.tiles;
        const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
        const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
        for (int g = g0; g < g1; g += kSub, ++it) {
          if ((it % kStages) % nprod != pq) continue;
          const int st = it % kStages, nsub = min(kSub, g1 - g);
          mbar_wait(&empty[st], ((it / kStages) & 1) ^ 1);
          mbar_expect_tx(&full[st], nsub * ((p.swap ? std::uint32_t(p.Kb) * 128 : a_bytes) + b_bytes));
          for (int sub = 0; sub < nsub; ++sub) {
            unsigned char* sa = smem + st * stage_bytes + sub * sub_bytes;
            const int n = (g + sub) / p.Lc, j0 = ((g + sub) - n * p.Lc) * 32;
            // swap: A = the dy box (K rows), B = the x boxes of column tile nt
            unsigned char* xa = p.swap ? sa + a_bytes : sa;
            const int xrow0 = p.swap ? nt * p.BN : mt * kBM;
            const int nbox = p.swap ? p.BN / p.Gb : boxes;
#pragma unroll 1
            for (int bx = 0; bx < nbox; ++bx) {
              const int row0 = xrow0 + bx * p.Gb;
              const int q = row0 / p.CCp, cc0 = row0 - q * p.CCp;
              const int qh = q / p.Qw, qw = q - qh * p.Qw;
              // rows past M: an out-of-range channel coordinate makes TMA
              // zero-fill the box. TMA wants the innermost start coordinate
              // 16-byte aligned: the misaligned part of the tap offset
              // selects a pre-shifted replica.
              const int o = j0 + qh * p.Wq + qw;
              tma_4d(xa + bx * (p.Gb * 128), &xmap, &full[st], o & ~3, row0 < p.M ? cc0 : p.CC, n, (o & 3) % p.T);
            }
            if (p.swap) tma_4d(sa, &dmap, &full[st], j0, 0, n, 0);
            else tma_4d(sa + a_bytes, &dmap, &full[st], j0, nt * p.BN, n, 0);
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
    long long c_data = 0, c_issue = 0, c_acc = 0, t_start = clock64();
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
      const int split = u / p.tiles;
      const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
      const int acc = tl & 1;
      long long c0 = p.prof ? clock64() : 0;
      mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
      tc_fence_after();
      if (p.prof) c_acc += clock64() - c0;
      const std::uint32_t dtm = tmem + std::uint32_t(acc * kMaxBN);
      for (int g = g0; g < g1; g += kSub, ++it) {
        const int st = it % kStages, nsub = min(kSub, g1 - g);
        long long c1 = p.prof ? clock64() : 0;
        mbar_wait(&full[st], (it / kStages) & 1);
        tc_fence_after();
        long long c2 = p.prof ? clock64() : 0;
        if (p.prof) c_data += c2 - c1;
        if (lane == 0) {
          for (int sub = 0; sub < nsub; ++sub) {
            const std::uint32_t sa = sbase + st * stage_bytes + sub * sub_bytes, sb = sa + a_bytes;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              mma_tf32(dtm, umma_desc_sw128(sa + q * 32), umma_desc_sw128(sb + q * 32), idesc,
                       (g + sub != g0 || q != 0) ? 1u : 0u);
          }
          mma_commit(&empty[st]);
          if (g + kSub >= g1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (p.prof) c_issue += clock64() - c2;
      }
      if (g1 <= g0 && lane == 0) mma_commit(&tfull[acc]);
      __syncwarp();
    }
    if (p.prof && lane == 0 && blockIdx.x < 1024) {
      g_bfprof[blockIdx.x * 4 + 0] = c_data;
      g_bfprof[blockIdx.x * 4 + 1] = c_issue;
      g_bfprof[blockIdx.x * 4 + 2] = c_acc;
      g_bfprof[blockIdx.x * 4 + 3] = clock64() - t_start;
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ epilogue: RED into dW
    __shared__ int offtab[kMaxBN];
    const int ew = warp - 4;
    int tl = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
      const int tile = u % p.tiles, split = u / p.tiles;
      const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
      const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
      const int acc = tl & 1;
      mbar_wait(&tfull[acc], (tl >> 1) & 1);
      tc_fence_after();
      const std::uint32_t tbase = tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t(acc * kMaxBN);
      if (p.swap) {
        // TMEM lane = output channel k, column = x row of tile nt
        asm volatile("bar.sync 1, 128;" ::: "memory");  // previous unit done with offtab
        for (int j = ew * 32 + lane; j < p.BN; j += 128) offtab[j] = x_row_off(p, nt * p.BN + j);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int k = ew * 32 + lane;
        const bool live = k < p.K && g1 > g0;
        for (int c0 = 0; c0 < p.BN; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + std::uint32_t(c0), v);
          if (!live) continue;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (c0 + j >= p.BN) break;
            if (offtab[c0 + j] >= 0) red_add(p.acc + std::int64_t(nt * p.BN + c0 + j) * kBM + k, v[j]);
          }
        }
      } else {
        // this thread's GEMM row -> dW offset (c, r, s), or invalid
        const int row = mt * kBM + ew * 32 + lane;
        const int off = g1 > g0 ? x_row_off(p, row) : -1;
        for (int c0 = 0; c0 < p.BN; c0 += 32) {
          float v[32];
          tmem_ld32(tbase + std::uint32_t(c0), v);
          if (off < 0) continue;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int k = nt * p.BN + c0 + j;
            if (c0 + j >= p.BN || k >= p.K) break;
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


// 2-SM BackwardFilter (K >= 128, roles not swapped): CTA pairs with
// tcgen05.mma cta_group::2 -- 256 x rows (128 per CTA, each CTA's own x
// boxes) x BN output channels, the dy box split along N (BN/2 rows per CTA).
// Same split-K units over (image, 32-pixel step), same RED-into-scratch
// epilogue per CTA; rank 0 issues the MMAs, both CTAs' TMA bytes count on
// its barriers, commits multicast to both, both epilogues release rank 0's
// accumulator barrier.
__global__ void __launch_bounds__(kThreads, 1)
    bf2_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap dmap, const BfParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t rank = cluster_rank();
  const int bh = p.BN / 2;
  const std::uint32_t a_bytes = kBM * 128;
  const std::uint32_t b_bytes = std::uint32_t(bh) * 128;
  const std::uint32_t stage_bytes = a_bytes + ((b_bytes + 1023) & ~1023u);
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
  const int units = p.tiles * p.splits;  // tiles = pair tiles x n tiles
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0 || warp == 2 || warp == 3) {
    const int pq = warp == 0 ? 0 : warp - 1;
    const int nprod = kStages < 3 ? kStages : 3;
    if (lane == 0) {
      const int boxes = kBM / p.Gb;
      int it = 0;
      for (int u = cid; u < units; u += ncl) {
        const int tile = u % p.tiles, split = u / p.tiles;
        const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;  // m_tiles counts 256-row pair tiles
        const int g0 = split * p.steps_per_unit, g1 = min(p.steps, g0 + p.steps_per_unit);
        const int xrow0 = mt * 2 * kBM + int(rank) * kBM;
        for (int g = g0; g < g1; ++g, ++it) {
          if ((it % kStages) % nprod != pq) continue;
          const int st = it % kStages;
          mbar_wait(&empty[st], ((it / kStages) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(&full[st], 2u * (a_bytes + b_bytes));
          const std::uint32_t bar = mapa(smem_u32(&full[st]), 0);
          unsigned char* sa = smem + st * stage_bytes;
          const int n = g / p.Lc, j0 = (g - n * p.Lc) * 32;
#pragma unroll 1
          for (int bx = 0; bx < boxes; ++bx) {
            const int row0 = xrow0 + bx * p.Gb;
            const int q = row0 / p.CCp, cc0 = row0 - q * p.CCp;
            const int qh = q / p.Qw, qw = q - qh * p.Qw;
            const int o = j0 + qh * p.Wq + qw;
            tma_4d_2sm(sa + bx * (p.Gb * 128), &xmap, bar, o & ~3, row0 < p.M ? cc0 : p.CC, n, (o & 3) % p.T);
          }
          tma_4d_2sm(sa + a_bytes, &dmap, bar, j0, nt * p.BN + int(rank) * bh, n, 0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (rank == 0) {
      const std::uint32_t idesc = idesc_tf32(2 * kBM, p.BN);
      const std::uint32_t sbase = smem_u32(smem);
      const std::uint64_t da0 = umma_desc_sw128(sbase), db0 = umma_desc_sw128(sbase + a_bytes);
      int it = 0, tl = 0;
      for (int u = cid; u < units; u += ncl, ++tl) {
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
            const std::uint32_t o = (std::uint32_t(st) * stage_bytes) >> 4;
            mma_tf32_2sm(dtm, da0 + o, db0 + o, idesc, g != g0);
            mma_tf32_2sm(dtm, da0 + o + 2, db0 + o + 2, idesc, 1u);
            mma_tf32_2sm(dtm, da0 + o + 4, db0 + o + 4, idesc, 1u);
            mma_tf32_2sm(dtm, da0 + o + 6, db0 + o + 6, idesc, 1u);
            mma_commit_2sm(&empty[st], 3);
            if (g == g1 - 1) mma_commit_2sm(&tfull[acc], 3);
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
      const int acc = tl & 1;
      mbar_wait(&tfull[acc], (tl >> 1) & 1);
      tc_fence_after();
      const std::uint32_t tbase = tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t(acc * kMaxBN);
      const int row = mt * 2 * kBM + int(rank) * kBM + ew * 32 + lane;
      const int off = g1 > g0 ? x_row_off(p, row) : -1;
      for (int c0 = 0; c0 < p.BN; c0 += 32) {
        float v[32];
        tmem_ld32(tbase + std::uint32_t(c0), v);
        if (off < 0) continue;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int k = nt * p.BN + c0 + j;
          if (c0 + j >= p.BN || k >= p.K) break;
          red_add(p.acc + std::int64_t(k) * p.rpad + row, v[j]);
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

// x (NCHW) -> x_ph[t][n][(a,b,c)][Lp]: zero padding + stride-phase split,
// replica t shifted left by t elements. One thread = 4 consecutive plane
// positions of every replica (float4 stores; HBM-bound).
struct XPhaseArgs {
  const float* x;
  float* out;
  int C, H, W, ph, pw, sh, sw, Bw, CC, T;
  std::int64_t units, rep;  // float4 units per replica, floats per replica
  FastDiv fd_u, fd_wq, fd_c, fd_bw;  // units per plane, plane pitch, C, Bw
};
__device__ __forceinline__ void x_phase_unit(const XPhaseArgs& a, std::int64_t u) {
  std::uint32_t plane, q;
  a.fd_u.divmod(std::uint32_t(u), plane, q);
  std::uint32_t n, cc, ab, c, pa, pb;
  n = plane / std::uint32_t(a.CC);
  cc = plane - n * std::uint32_t(a.CC);
  a.fd_c.divmod(cc, ab, c);
  a.fd_bw.divmod(ab, pa, pb);
  const float* src = a.x + (std::int64_t(n) * a.C + c) * a.H * a.W;
  const int p0 = int(q) * 4;
  float v[7];
  std::uint32_t i, j;
  a.fd_wq.divmod(std::uint32_t(p0), i, j);
#pragma unroll
  for (int e = 0; e < 7; ++e) {
    const int h = int(i) * a.sh + int(pa) - a.ph, w = int(j) * a.sw + int(pb) - a.pw;
    v[e] = (e < a.T + 3 && unsigned(h) < unsigned(a.H) && unsigned(w) < unsigned(a.W)) ? __ldg(src + h * a.W + w)
                                                                                      : 0.f;
    if (++j == a.fd_wq.d) {
      j = 0;
      ++i;
    }
  }
  float4* dst = reinterpret_cast<float4*>(a.out) + u;
#pragma unroll
  for (int t = 0; t < 4; ++t)
    if (t < a.T) dst[t * (a.rep / 4)] = make_float4(v[t], v[t + 1], v[t + 2], v[t + 3]);
}

// dy (NCHW) -> dy_p[n][k][Ldp]: rows re-pitched to Wq, zero beyond OW.
struct DyPitchArgs {
  const float* dy;
  float* out;
  int OH, OW;
  std::int64_t units;
  FastDiv fd_u, fd_wq;
};
__device__ __forceinline__ void dy_pitch_unit(const DyPitchArgs& a, std::int64_t u) {
  std::uint32_t plane, q, i, j;
  a.fd_u.divmod(std::uint32_t(u), plane, q);
  const float* src = a.dy + std::int64_t(plane) * a.OH * a.OW;
  a.fd_wq.divmod(q * 4, i, j);
  float v[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    v[e] = (int(i) < a.OH && int(j) < a.OW) ? __ldg(src + int(i) * a.OW + int(j)) : 0.f;
    if (++j == a.fd_wq.d) {
      j = 0;
      ++i;
    }
  }
  reinterpret_cast<float4*>(a.out)[u] = make_float4(v[0], v[1], v[2], v[3]);
}

// One launch for everything BackwardFilter does before its GEMM: the two
// re-layouts (either may be skipped) and dW *= beta (beta != 1).
__global__ void __launch_bounds__(256) bf_prep_kernel(const XPhaseArgs xa, const DyPitchArgs da, float4* acc,
                                                       std::int64_t an) {
  pdl_wait();
  pdl_trigger();
  const std::int64_t nx = xa.units, nd = da.units, total = nx + nd + an;
  for (std::int64_t u = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; u < total;
       u += std::int64_t(gridDim.x) * blockDim.x) {
    if (u < nx) x_phase_unit(xa, u);
    else if (u < nx + nd) dy_pitch_unit(da, u - nx);
    else acc[u - nx - nd] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// dW[k][c][r][s] = beta * dW + alpha * scratch[k][row(c, r, s)]: every dW
// element owns exactly one GEMM row, so this is a plain gather-update.
struct FinalizeArgs {
  const float* acc;
  float* dw;
  float alpha, beta;
  int K, C, R, S, sh, sw, Bw, Qw, CCp, rpad, swap;
  std::int64_t n;  // K * C * R * S
};
__global__ void __launch_bounds__(256) bf_finalize_kernel(const FinalizeArgs f) {
  pdl_wait();
  pdl_trigger();
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < f.n;
       i += std::int64_t(gridDim.x) * blockDim.x) {
    const int s = int(i % f.S);
    std::int64_t t = i / f.S;
    const int r = int(t % f.R);
    t /= f.R;
    const int c = int(t % f.C), k = int(t / f.C);
    const int qh = r / f.sh, a = r - qh * f.sh, qw = s / f.sw, b = s - qw * f.sw;
    const int row = (qh * f.Qw + qw) * f.CCp + (a * f.Bw + b) * f.C + c;
    const float v = f.swap ? f.acc[std::int64_t(row) * kBM + k] : f.acc[std::int64_t(k) * f.rpad + row];
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

int sm_count() {
  static int v = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return v;
}

// dims (d0, d1, d2, d3) with element pitches of dims 1..3; box (box0, box1, 1, 1)
bool encode_4d(CUtensorMap* m, const float* base, int d0, int d1, int d2, int d3, std::int64_t pitch1,
               std::int64_t pitch2, std::int64_t pitch3, int box0, int box1) {
  const cuuint64_t dims[4] = {cuuint64_t(d0), cuuint64_t(d1), cuuint64_t(d2), cuuint64_t(d3)};
  const cuuint64_t strides[3] = {cuuint64_t(pitch1) * 4, cuuint64_t(pitch2) * 4, cuuint64_t(pitch3) * 4};
  const cuuint32_t box[4] = {cuuint32_t(box0), cuuint32_t(box1), 1, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return encode_tiled()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

void bf_profile(double out[4]) {
  static unsigned long long h[1024 * 4];
  cudaMemcpyFromSymbol(h, g_bfprof, sizeof(h));
  double s[4] = {0, 0, 0, 0};
  int n = 0;
  for (int b = 0; b < 1024; ++b) {
    if (h[b * 4 + 3] == 0) continue;
    for (int i = 0; i < 4; ++i) s[i] += double(h[b * 4 + i]);
    ++n;
  }
  for (int i = 0; i < 4; ++i) out[i] = n ? s[i] / n : 0;
}

// UCUDNN_TUNE=bfl=1 routes PRECOMP BackwardFilter to the gather kernel (bflsu.cu; algo 6)
bool use_lsu(const ConvShape& s) { return tune("bfl", 0) && bfl_supports(s); }

bool bf_supports(const ConvShape& s) {
  if (use_lsu(s)) return true;
  const BfGeo g = make_geo(s);
  // TMA coordinates are int32 and box dims <= 256; flat offsets must fit
  return std::int64_t(g.Lq) + 64 < (std::int64_t(1) << 30) && g.CC < (1 << 20) && s.K < (1 << 20) &&
         std::int64_t(g.N) * g.CC * g.Lp / 4 < (std::int64_t(1) << 31) &&
         std::int64_t(g.N) * g.K * g.Ldp / 4 < (std::int64_t(1) << 31);
}

std::int64_t bf_workspace(const ConvShape& s) {
  if (use_lsu(s)) return bfl_workspace(s);
  const BfGeo g = make_geo(s);
  return std::int64_t(x_bytes(g) + dy_bytes(g) + acc_bytes(g));
}

cudaError_t bf_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha, float beta,
                   cudaStream_t st) {
  if (use_lsu(s)) return bfl_run(s, x, dy, dw, ws, alpha, beta, st);
  const BfGeo g = make_geo(s);
  const float* xph = g.x_direct ? x : static_cast<const float*>(ws);
  const float* dyp = g.dy_direct ? dy : reinterpret_cast<const float*>(static_cast<char*>(ws) + x_bytes(g));
  const FastDiv fd_wq(std::uint32_t(g.Wq));
  const int sms = sm_count();
  XPhaseArgs xa{x, const_cast<float*>(xph), g.C, g.H, g.W, g.ph, g.pw, g.sh, g.sw, g.Bw, g.CC, g.T,
                g.x_direct ? 0 : std::int64_t(g.N) * g.CC * (g.Lp / 4), std::int64_t(g.N) * g.CC * g.Lp,
                FastDiv(std::uint32_t(g.Lp / 4)), fd_wq, FastDiv(std::uint32_t(g.C)), FastDiv(std::uint32_t(g.Bw))};
  DyPitchArgs da{dy, const_cast<float*>(dyp), g.OH, g.OW, g.dy_direct ? 0 : std::int64_t(g.N) * g.K * (g.Ldp / 4),
                 FastDiv(std::uint32_t(g.Ldp / 4)), fd_wq};
  float* accbuf = reinterpret_cast<float*>(static_cast<char*>(ws) + x_bytes(g) + dy_bytes(g));
  const std::int64_t an = std::int64_t(rows_pad(g)) * cols_pad(g) / 4;
  const std::int64_t prep = xa.units + da.units + an;
  cudaError_t e = launch_pdl(bf_prep_kernel, dim3(int(std::min<std::int64_t>((prep + 255) / 256, 16 * sms))), dim3(256),
                             0, st, xa, da, reinterpret_cast<float4*>(accbuf), an);
  if (e != cudaSuccess) return e;

  CUtensorMap xmap, dmap;
  const std::int64_t rep = std::int64_t(g.N) * g.CC * g.Lp;
  if (!encode_4d(&xmap, xph, g.Lq, g.CC, g.N, g.T, g.Lp, std::int64_t(g.CC) * g.Lp, rep, 32, g.Gb))
    return cudaErrorInvalidValue;
  // 2-SM kernel (the MMA pairs 256 x rows; each CTA loads half of the dy
  // rows) where it measured faster: 256-wide or multi-tile K (AlexNet
  // conv3-5, 32-64 images: 3-10 %); K = 192 in one tile (conv2) lost 2-3 %.
  const bool two = !g.swap && g.BN % 16 == 0 && (g.BN >= 256 || (g.BN >= 128 && g.n_tiles >= 2)) && tune("bf2", 1);
  if (!encode_4d(&dmap, dyp, g.Ld, g.K, g.N, 1, g.Ldp, std::int64_t(g.K) * g.Ldp, std::int64_t(g.N) * g.K * g.Ldp, 32,
                 g.swap ? g.Kb : two ? g.BN / 2 : g.BN))
    return cudaErrorInvalidValue;

  BfParams p{};
  p.dw = dw;
  p.alpha = alpha;
  p.K = g.K; p.C = g.C; p.R = g.R; p.S = g.S;
  p.RS = g.R * g.S;
  p.CRS = g.C * p.RS;
  p.Bw = g.Bw; p.Ah = g.Ah; p.sh = g.sh; p.sw = g.sw; p.Qw = g.Qw;
  p.CCp = g.CCp; p.CC = g.CC; p.Gb = g.Gb; p.Wq = g.Wq; p.M = g.M; p.BN = g.BN;
  p.m_tiles = g.m_tiles;
  p.tiles = g.m_tiles * g.n_tiles;
  p.Lc = g.Lc;
  p.T = g.T;
  p.swap = g.swap;
  p.acc = accbuf;
  p.rpad = rows_pad(g);
  p.prof = tune("prof", 0);
  p.Kb = g.Kb;
  p.steps = g.N * g.Lc;
  // split the reduction so the tiles fill the SMs once, >= 8 steps per unit
  if (two) {
    p.m_tiles = (g.m_tiles + 1) / 2;
    p.tiles = p.m_tiles * g.n_tiles;
    int sp = deterministic() ? 1 : std::max(1, std::min(p.steps / 8, (sms / 2) / p.tiles));
    p.ksub = 1;
    p.steps_per_unit = (p.steps + sp - 1) / sp;
    p.splits = (p.steps + p.steps_per_unit - 1) / p.steps_per_unit;
    const int stage2 = kBM * 128 + ((g.BN / 2 * 128 + 1023) & ~1023);
    p.stages = ring_stages(std::min(tune("bf2_stages", 8), (200 * 1024) / stage2));
    const int smem2 = std::max(p.stages * stage2 + 1024 + 256, 116 * 1024);
    e = set_smem_attr(reinterpret_cast<const void*>(bf2_kernel), 227 * 1024);
    if (e != cudaSuccess) return e;
    count_launch();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * std::min(sms / 2, p.tiles * p.splits));
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
    e = cudaLaunchKernelEx(&cfg, bf2_kernel, xmap, dmap, p);
    if (e != cudaSuccess) return e;
    FinalizeArgs f2{accbuf, dw, alpha, beta, g.K, g.C, g.R, g.S, g.sh, g.sw, g.Bw, g.Qw, g.CCp, rows_pad(g), g.swap,
                    s.w_elems()};
    return launch_pdl(bf_finalize_kernel, dim3(int(std::min<std::int64_t>((f2.n + 255) / 256, 8 * sms))), dim3(256), 0,
                      st, f2);
  }
  int splits = deterministic() ? 1 : std::max(1, std::min(p.steps / 8, tune("bf_waves", 1) * sms / p.tiles));
  p.ksub = std::max(1, std::min(kMaxSub, tune("bf_ksub", 1)));
  const int kSub = p.ksub;
  p.steps_per_unit = ((p.steps + splits - 1) / splits + kSub - 1) / kSub * kSub;
  p.splits = (p.steps + p.steps_per_unit - 1) / p.steps_per_unit;
  const int stage_bytes = kSub * (kBM * 128 + ((g.BN * 128 + 1023) & ~1023));
  p.stages = ring_stages(std::min(tune("bf_stages", 8), (200 * 1024) / stage_bytes));
  const int smem = std::max(p.stages * stage_bytes + 1024 + 256, 116 * 1024);
  e = set_smem_attr(reinterpret_cast<const void*>(bf_kernel), 220 * 1024);  // + 1 KB static offtab
  if (e != cudaSuccess) return e;
  e = launch_pdl(bf_kernel, dim3(std::min(sms, p.tiles * p.splits)), dim3(kThreads), std::size_t(smem), st, xmap, dmap,
                 p);
  if (e != cudaSuccess) return e;
  FinalizeArgs f{accbuf, dw, alpha, beta, g.K, g.C, g.R, g.S, g.sh, g.sw, g.Bw, g.Qw, g.CCp, rows_pad(g), g.swap,
                 s.w_elems()};
  return launch_pdl(bf_finalize_kernel, dim3(int(std::min<std::int64_t>((f.n + 255) / 256, 8 * sms))), dim3(256), 0, st,
                    f);
}

}  // namespace ucudnn
