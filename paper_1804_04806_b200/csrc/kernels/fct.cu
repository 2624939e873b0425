// Few-channel strided layers (AlexNet conv1: 3 channels, 11x11, stride 4;
// ResNet conv1: 3 channels, 7x7, stride 2) with the im2col operand built
// straight into tensor memory: no space-to-depth copy, no workspace for
// Forward, and no operand tile ever stored to shared memory.
//
//   Forward: y[n][k][oh][ow] = alpha * sum_{c,r,s} x[n][c][oh*sh-ph+r][ow*sw-pw+s] * w[k][c][r][s] + beta * y
//   (reference_conv.hpp:70-100)
//
// The im2col expansion of these layers is large (AlexNet conv1: 363 taps per
// output pixel from 3 input channels, ~7.6x the input) and the earlier paths
// either stream it from L2 through TMA im2col boxes of a space-to-depth copy
// (algorithm 5: L2 -> SM bound) or rebuild it in shared memory (fps.cu:
// bound by the LDS + STS of every element). Here:
//
// * a tile is TR whole output rows of one image (TR * OW <= 128 pixels, one
//   per TMEM lane); a CTA owns a contiguous run of tiles, so consecutive
//   tiles share R - TR*sh of their input rows;
// * loader warps keep the input rows in a ring in shared memory (C rows per
//   virtual row index, RR rows deep): per tile they load only the rows the
//   previous tile did not (TR*sh of them; all PH at an image change), with
//   coalesced loads, up to several tiles ahead of the consumers;
// * A-operand producers -- one thread per output pixel, i.e. per TMEM lane --
//   read their taps from the ring with vector loads (sw consecutive taps are
//   sw consecutive floats: LDS.128 for stride 4, LDS.64 for stride 2,
//   conflict-free across a warp) and write them to TMEM with tcgen05.st;
// * tcgen05.mma takes A from TMEM and the filter (B, K-major SWIZZLE_128B)
//   from shared memory, where it stays resident for the whole persistent
//   kernel; two TMEM accumulator sets overlap a tile's NCHW epilogue with
//   the next tile's MMAs.
//
// Reduction order: (c, r, s') with s' padded to SP = round_up(S, 4) taps (the
// padded taps have zero filter weights); an A ring slot holds KG (c, r)
// groups = KG * SP / 32 whole 32-float filter chunks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>



#include "conv_common.h"
#include "fct.h"
#include "launch.h"
#include "sm100.cuh"

namespace ucudnn {
using namespace sm100;

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled_fct();  // (defined with the stride-1 host code)

constexpr int kBM = 128;
constexpr int kMaxSlots = 8;
constexpr int kNB = 8;        // tile barriers (ring of tiles in flight between loaders and producers)
constexpr int kHist = 8;      // loader's history of tile row origins (>= the lookahead)
// Forward: 20 warps (5 per SM sub-partition: 96 registers; 21 would get 80)
constexpr int kFwdWarps = 20;
constexpr int kRB = 4;        // ring rows per loader batch (8 x 32 columns each)
constexpr int kMaxGroups = 64;
// warps: 0-7 A producers, 8 MMA issuer, 9 .. 8+nepi epilogue, the rest row loaders
constexpr int kThreads = kFwdWarps * 32;

struct TGeo {
  int OH, OW, TR, np, tiles_per_img, units, grid;
  int SP, groups, gpad, kslots, kred, nchunk, BN;
  int PH, pitch, slot_cols, nslots, RR;
  std::size_t b_bytes, r_bytes, smem;
};

struct TParams {
  const float* x;
  const float* w;
  float* y;
  float alpha, beta;
  int C, H, W, K, R, S, ph, pw, sh, sw, OH, OW;
  int TR, np, tiles_per_img, units;
  int groups, kslots, nchunk, BN, PH, pitch, nslots, RR;
  int nepi;  // epilogue warps (4 or 8); the loaders get the other 11 - nepi
  int dbg;  // UCUDNN_TUNE=fct_dbg=1: per-role wait cycles of CTAs 0-1 (printf)
  long long CHW, KOHW;
};

// Waits of the warps off the critical path (epilogue, row loaders): back off
// with nanosleep so the spinning does not take issue slots from the A
// producers sharing their SM sub-partitions.
__device__ __forceinline__ void mbar_wait_sleep(std::uint64_t* bar, std::uint32_t parity) {
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

// 32 lanes x 8 columns of 32-bit from registers into TMEM
__device__ __forceinline__ void tmem_st8(std::uint32_t taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]^T, M = 128 x N x 8, executed by the whole
// (converged) warp with one elected lane issuing: operands computed by every
// lane from uniform values stay in uniform registers (inside `if (lane == 0)`
// ptxas re-broadcast every operand per MMA: ~120 instead of ~50 cycles per
// MMA, scripts/mma_ts_probe.cu).
__device__ __forceinline__ void mma_tf32_ts_warp(std::uint32_t d_tmem, std::uint32_t a_tmem, std::uint64_t bdesc,
                                                 std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_ts_2sm_warp(std::uint32_t d_tmem, std::uint32_t a_tmem, std::uint64_t bdesc,
                                                     std::uint32_t idesc, std::uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_warp(std::uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
      : "memory");
}

// the SP taps of group (c, r) at this thread's pixel, vector loads of SW floats
template <int SW, int SP>
__device__ __forceinline__ void load_group(std::uint32_t addr, float* v) {
  if constexpr (SW == 4) {
#pragma unroll
    for (int i = 0; i < SP / 4; ++i)
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(v[4 * i]), "=f"(v[4 * i + 1]), "=f"(v[4 * i + 2]), "=f"(v[4 * i + 3])
                   : "r"(addr + 16 * i));
  } else {
#pragma unroll
    for (int i = 0; i < SP / 2; ++i)
      asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v[2 * i]), "=f"(v[2 * i + 1]) : "r"(addr + 8 * i));
  }
}

// This CTA's contiguous tile range [t0, t1).
__device__ __forceinline__ void tile_range(const TParams& p, int& t0, int& t1) {
  t0 = int((long long)blockIdx.x * p.units / gridDim.x);
  t1 = int((long long)(blockIdx.x + 1) * p.units / gridDim.x);
}

// Virtual ring row of the first input row of the CTA's next tile, the same
// recurrence in loaders and producers: consecutive tiles of one image
// advance by TR*sh rows; a new image starts after the last row loaded.
struct RowWalk {
  int vstart = 0, vend = 0, n = -1;
  __device__ __forceinline__ bool next(const TParams& p, int u) {
    const int nn = u / p.tiles_per_img;
    const bool fresh = nn != n;
    vstart = fresh ? vend : vstart + p.TR * p.sh;
    vend = vstart + p.PH;
    n = nn;
    return fresh;
  }
};

// The BackwardFilter kernel's walk: units are single output rows (n, oh).
struct BParams;
struct RowWalkB {
  int vstart = 0, vend = 0, n = -1;
  int oh = 0, vmod = 0;  // step(): row within the image, vstart % RR
  template <typename P>
  __device__ __forceinline__ bool next(const P& p, int u) {
    const int nn = u / p.OH;
    const bool fresh = nn != n;
    vstart = fresh ? vend : vstart + p.sh;
    vend = vstart + p.R;
    n = nn;
    return fresh;
  }
  // next() for consecutive units u, u + 1, ...: the image / row and the ring
  // row of vstart are stepped (one division on the first call only)
  template <typename P>
  __device__ __forceinline__ bool step(const P& p, int u) {
    bool fresh;
    if (n < 0) {
      n = u / p.OH;
      oh = u - n * p.OH;
      fresh = true;
    } else if (++oh == p.OH) {
      oh = 0;
      ++n;
      fresh = true;
    } else {
      fresh = false;
    }
    vmod += fresh ? vend - vstart : p.sh;
    while (vmod >= p.RR) vmod -= p.RR;
    vstart = fresh ? vend : vstart + p.sh;
    vend = vstart + p.R;
    return fresh;
  }
};

// Wait-time instrumentation (build with -DFCT_PROFILE, run with
// UCUDNN_TUNE=fct_dbg=1): cycles each role spent waiting, CTAs 0-1, printf.
#ifdef FCT_PROFILE
#define FCT_T0 long long t_beg = clock64(), t_w1 = 0, t_w2 = 0, t_w3 = 0, t_q = 0
#define FCT_W(acc, stmt)    \
  do {                      \
    t_q = clock64();        \
    stmt;                   \
    acc += clock64() - t_q; \
  } while (0)
#define FCT_PRINT(name)                                                                          \
  if ((threadIdx.x & 31) == 0 && blockIdx.x < 1 && (warp % 4) == 0 || (threadIdx.x == 13 * 32 || threadIdx.x == 15 * 32) && blockIdx.x < 1)                     \
  printf("blk %d %s: total %lld wait1 %lld wait2 %lld w3 %lld\n", blockIdx.x, name, clock64() - t_beg, t_w1, \
         t_w2, t_w3)
#else
#define FCT_T0
#define FCT_W(acc, stmt) stmt
#define FCT_PRINT(name)
#endif

template <int SW, int SP, int KG>
__global__ void __launch_bounds__(kThreads, 1) fct_fwd_kernel(const TParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t b_bytes = std::uint32_t(p.nchunk) * p.BN * 128;
  float* ring = reinterpret_cast<float*>(smem + b_bytes);  // [C][RR][pitch]
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(ring + p.C * p.RR * p.pitch);
  std::uint64_t* afull = bars;
  std::uint64_t* aempty = afull + kMaxSlots;
  std::uint64_t* loaded = aempty + kMaxSlots;
  std::uint64_t* consumed = loaded + kNB;
  std::uint64_t* tfull = consumed + kNB;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  __shared__ int gc[kMaxGroups], gr[kMaxGroups];  // group -> ring offset of channel c (floats), tap row r (-1: padding)

  // the filter, K-major SWIZZLE_128B, resident: row k, reduction index
  // kk = (c * R + r) * SP + s' in 32-float chunks of BN rows
  {
    const int per_chunk = p.BN * 32;
    const int total = p.nchunk * per_chunk;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int chunk = i / per_chunk, rem = i - chunk * per_chunk;
      const int k = rem >> 5, j = rem & 31;
      const int kk = chunk * 32 + j;
      const int g = kk / SP, s = kk - g * SP;
      float v = 0.f;
      if (k < p.K && g < p.groups && s < p.S) {
        const int c = g / p.R, r = g - c * p.R;
        v = p.w[((long long)(k * p.C + c) * p.R + r) * p.S + s];
      }
      *reinterpret_cast<float*>(smem + chunk * p.BN * 128 + k * 128 + (((j >> 2) ^ (k & 7)) << 4) + (j & 3) * 4) = v;
    }
  }
  for (int g = threadIdx.x; g < kMaxGroups; g += blockDim.x) {
    const int c = g / p.R, r = g - c * p.R;
    gc[g] = c * p.RR * p.pitch;
    gr[g] = g < p.groups ? r : -1;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxSlots; ++s) {
      mbar_init(&afull[s], 256);
      mbar_init(&aempty[s], 1);
    }
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&loaded[b], (11 - p.nepi) * 32);
      mbar_init(&consumed[b], 256);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], p.nepi * 32);
    }
    mbar_fence_init();
  }
  if (warp == 8) tmem_alloc<512>(tmem_slot);
  fence_async_smem();  // the filter stores are read by the tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // warp-uniform by construction (a shuffle from lane 0), so the tcgen05
  // operands derived from it live in uniform registers
  const std::uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  int t0, t1;
  tile_range(p, t0, t1);
  const int my_units = t1 - t0;
  const std::uint32_t a_col0 = 2u * std::uint32_t(p.BN);  // A ring after the two accumulator sets

  if (warp < 8) {
    // ------------------------------------------------ A producers: one output pixel per thread;
    // warps w and w + 4 share TMEM lane quarter w % 4 and take the two
    // halves of every slot's (c, r) groups
    const int quarter = warp & 3, half = warp >> 2;
    const int px = quarter * 32 + lane;
    const int pe = px < p.np ? px : 0;
    const int rl = pe / p.OW, ow = pe - rl * p.OW;
    const std::uint32_t rbase = smem_u32(ring) + std::uint32_t(ow * SW * 4);
    const std::uint32_t tlane = tmem + (std::uint32_t(quarter * 32) << 16);
    constexpr int KH = KG / 2;
    RowWalk walk;
    RingPos rs;  // A ring slot over the whole kernel
    FCT_T0;
    for (int i = 0; i < my_units; ++i) {
      walk.next(p, t0 + i);
      FCT_W(t_w1, mbar_wait_sleep(&loaded[i % kNB], (i / kNB) & 1));
      const int row0 = (walk.vstart + rl * p.sh) % p.RR;  // ring row of tap row 0 at this pixel
      for (int ks = 0; ks < p.kslots; ++ks, rs.step(p.nslots)) {
        const int slot = rs.slot;
        FCT_W(t_w2, mbar_wait(&aempty[slot], rs.ph ^ 1));
        tc_fence_after();
        const int g0 = ks * KG + half * KH;
        float v[KH * SP];
#pragma unroll
        for (int q = 0; q < KH; ++q) {
          const int r = gr[g0 + q];
          if (r >= 0) {
            int row = row0 + r;
            if (row >= p.RR) row -= p.RR;
            load_group<SW, SP>(rbase + std::uint32_t(gc[g0 + q] + row * p.pitch) * 4, v + q * SP);
          } else {
#pragma unroll
            for (int j = 0; j < SP; ++j) v[q * SP + j] = 0.f;
          }
        }
        const std::uint32_t ta = tlane + a_col0 + std::uint32_t(slot * KG * SP + half * KH * SP);
#pragma unroll
        for (int j = 0; j < KH * SP; j += 8) tmem_st8(ta + std::uint32_t(j), v + j);
        FCT_W(t_w3, tmem_st_wait());
        tc_fence_before();
        mbar_arrive(&afull[slot]);
      }
      mbar_arrive(&consumed[i % kNB]);  // this thread's ring reads are done (their values went to TMEM)
    }
    FCT_PRINT("prod (loaded, slot)");
  } else if (warp >= 9 && warp < 9 + p.nepi) {
    // ------------------------------------------------ epilogue (NCHW stores, lane = pixel); with 8
    // warps (store-heavy layers: few input rows per tile) two take each lane quarter
    const int quarter = warp & 3, half = (warp - 9) >> 2, nh = p.nepi >> 2;
    const int px = quarter * 32 + lane;
    const int rl = px / p.OW, ow = px - rl * p.OW;
    const long long ks = (long long)p.OH * p.OW;
    FCT_T0;
    for (int i = 0; i < my_units; ++i) {
      const int u = t0 + i;
      const int n = u / p.tiles_per_img, oh0 = (u - n * p.tiles_per_img) * p.TR;
      const int acc = i & 1;
      FCT_W(t_w1, mbar_wait_sleep(&tfull[acc], (i >> 1) & 1));
      tc_fence_after();
      const bool live = px < p.np && oh0 + rl < p.OH;
      float* yb = p.y + (long long)n * p.KOHW + (long long)(oh0 + rl) * p.OW + ow;
      for (int c0 = half * 32; c0 < p.BN; c0 += 32 * nh) {
        float v[32];
        tmem_ld32(tmem + (std::uint32_t(quarter * 32) << 16) + std::uint32_t(acc * p.BN + c0), v);
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
    FCT_PRINT("epi (tfull, -)");
  } else if (warp == 8) {
    // ------------------------------------------------ MMA issuer (whole warp, one elected lane)
    // A slot spans KG * SP / 32 whole filter chunks, so every descriptor is
    // the slot's base plus a compile-time step: straight-line issue code
    constexpr int kMmas = KG * SP / 8;
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN);
    const std::uint64_t bdesc0 = umma_desc_sw128(smem_u32(smem));
    const std::uint32_t chunk_desc = std::uint32_t(p.BN * 128) >> 4;
    RingPos rs;
    FCT_T0;
    for (int i = 0; i < my_units; ++i) {
      const int acc = i & 1;
      FCT_W(t_w1, mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1));
      tc_fence_after();
      const std::uint32_t d = tmem + std::uint32_t(acc * p.BN);
      std::uint64_t bd = bdesc0;
      for (int ks = 0; ks < p.kslots; ++ks, rs.step(p.nslots)) {
        const int slot = rs.slot;
        FCT_W(t_w2, mbar_wait(&afull[slot], rs.ph));
        tc_fence_after();
        const std::uint32_t ta = tmem + a_col0 + std::uint32_t(slot * KG * SP);
#pragma unroll
        for (int j = 0; j < kMmas; ++j)
          mma_tf32_ts_warp(d, ta + std::uint32_t(8 * j), bd + (j >> 2) * chunk_desc + 2 * (j & 3), idesc,
                           (ks | j) ? 1u : 0u);
        mma_commit_warp(&aempty[slot]);
        if (ks + 1 == p.kslots) mma_commit_warp(&tfull[acc]);
        __syncwarp();
        bd += (kMmas >> 2) * chunk_desc;
      }
    }
    FCT_PRINT("mma (tempty, afull)");
  } else if (warp >= 9 + p.nepi) {
    // ------------------------------------------------ row loaders (zero off the image)
    const int lw = warp - 9 - p.nepi, nl = 11 - p.nepi;
    RowWalk walk;
    __shared__ int hist[kHist];  // vstart of the last kHist tiles (shared: a local array spilled to L2-latency local memory)
    int waited = -1;  // every tile <= waited has been consumed
    FCT_T0;
    for (int i = 0; i < my_units; ++i) {
      const int u = t0 + i;
      const bool fresh = walk.next(p, u);
      const int n = u / p.tiles_per_img, oh0 = (u - n * p.tiles_per_img) * p.TR;
      const int lo = fresh ? walk.vstart : walk.vend - p.TR * p.sh;  // virtual rows [lo, vend) are new
      const int cnt = walk.vend - lo;
      // they overwrite virtual rows [lo - RR, vend - RR): wait until every
      // tile that may still read one of those has been consumed
      const int ov = walk.vend - 1 - p.RR;
      int need = -1;
      for (int j = i - 1; j >= 0 && j >= i - kHist; --j)
        if (hist[j % kHist] <= ov) {
          need = j;
          break;
        }
      if (need > waited) {
        FCT_W(t_w1, mbar_wait_sleep(&consumed[need % kNB], (need / kNB) & 1));
        waited = need;
      }
      __syncwarp();
      if (lane == 0) hist[i % kHist] = walk.vstart;
      __syncwarp();
      const float* xn = p.x + (long long)n * p.CHW;
      const int nrows = p.C * cnt;
      for (int cb = 0; cb < p.pitch; cb += 256) {
        for (int q0 = lw; q0 < nrows; q0 += nl * kRB) {
          float v[kRB][8];
#pragma unroll
          for (int rb = 0; rb < kRB; ++rb) {
            const int q = q0 + rb * nl;
            const int c = q / cnt, vr = lo + q - c * cnt;
            const int ih = oh0 * p.sh - p.ph + (vr - walk.vstart);
            const bool rok = q < nrows && unsigned(ih) < unsigned(p.H);
            const float* src = xn + ((long long)c * p.H + (rok ? ih : 0)) * p.W;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int col = cb + lane + 32 * j;
              const int iw = col - p.pw;
              v[rb][j] = rok && col < p.pitch && unsigned(iw) < unsigned(p.W) ? __ldg(src + iw) : 0.f;
            }
          }
#pragma unroll
          for (int rb = 0; rb < kRB; ++rb) {
            const int q = q0 + rb * nl;
            if (q >= nrows) break;
            const int c = q / cnt, vr = lo + q - c * cnt;
            float* dst = ring + (c * p.RR + vr % p.RR) * p.pitch + cb + lane;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (cb + lane + 32 * j < p.pitch) dst[32 * j] = v[rb][j];
          }
        }
      }
      mbar_arrive(&loaded[i % kNB]);  // release: this thread's ring stores
    }
    FCT_PRINT("load (consumed, loading)");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// ============================================================== BackwardFilter
//
//   dW[k][c][r][s] = beta * dW + alpha * sum_{n,oh,ow} dy[n][k][oh][ow] * x[n][c][oh*sh-ph+r][ow*sw-pw+s]
//   (reference_conv.hpp:141-180)
//
// D[q][k] = sum_px A[q][px] * B[k][px] with q = (c, r, s) on the TMEM lanes
// (QT tiles of 128), the reduction over output pixels in 32-pixel blocks of
// one output row, and N = the K output channels. A (the x taps) is built in
// TMEM: producer thread q reads x[c][oh*sh-ph+r][ow*sw-pw+s] for the block's
// 32 pixels from the input-row ring (the ring pitch is = S mod 32, so the 32
// lanes of a warp -- consecutive (r, s) -- hit 32 different banks) and
// stores them with one tcgen05.st. B (dy rows, 32 pixels x K) arrives by
// coalesced loads into a K-major SWIZZLE_128B ring. A CTA owns a contiguous
// run of output rows and accumulates all of them in TMEM; at the end its
// partial sums go to its own workspace slice and a finalize adds the slices
// in a fixed order: deterministic, no atomics.
constexpr int kBfMaxQT = 3;
constexpr int kBfDSlots = 12;  // dy ring (8 KB per 64-channel block)
constexpr int kBfXLoaders = 1;  // x-row loader warp (bulk copies)
constexpr int kBfDLoaders = 4;  // dy loader warps, each owning whole 32-pixel blocks (64 loads in flight per lane)
// warps: 0 .. 4*QT-1 A producers (+ the final slice store), 12 MMA issuer,
// 13 x-row loader, 14-17 dy loaders (18 warps: 96 registers)
constexpr int kBfThreads = (4 * kBfMaxQT + 1 + kBfXLoaders + kBfDLoaders) * 32;

struct BParams {
  const float* x;
  const float* dy;
  float* slices;
  int C, H, W, K, R, S, ph, pw, sh, sw, OH, OW;
  int rows, BN, nblk, units, RR, pitch, nslots;
  int dtma;  // dy blocks by TMA (16 B aligned dy rows, BN == K): one box per block instead of loader warps
  long long CHW, KOHW;
};

__device__ __forceinline__ void tma_3d_b(std::uint32_t dst, const void* tmap, std::uint64_t* bar, int x, int y,
                                         int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_u32(std::uint32_t dst, const void* src, std::uint32_t bytes,
                                             std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_st32(std::uint32_t taddr, const float (&v)[32]) {
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
}

__device__ __forceinline__ void bf_range(const BParams& p, int& u0, int& u1) {
  u0 = int((long long)blockIdx.x * p.units / gridDim.x);
  u1 = int((long long)(blockIdx.x + 1) * p.units / gridDim.x);
}

template <int SW, int QT>
__global__ void __launch_bounds__(kBfThreads, 1)
    fct_bwdf_kernel(const __grid_constant__ CUtensorMap dmap, const BParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t dslot_bytes = std::uint32_t(p.BN) * 128;
  unsigned char* dring = smem;  // kBfDSlots x [BN rows x 128 B], SWIZZLE_128B K-major
  float* ring = reinterpret_cast<float*>(dring + kBfDSlots * dslot_bytes);  // [C][RR][pitch]
  // the pitch is odd in general: round the barrier block up to 16 B
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(
      (reinterpret_cast<std::uintptr_t>(ring + p.C * p.RR * p.pitch) + 15) & ~std::uintptr_t(15));
  std::uint64_t* afull = bars;
  std::uint64_t* aempty = afull + kMaxSlots;
  std::uint64_t* dfull = aempty + kMaxSlots;
  std::uint64_t* dempty = dfull + kBfDSlots;
  std::uint64_t* loaded = dempty + kBfDSlots;
  std::uint64_t* consumed = loaded + kNB;
  std::uint64_t* tdone = consumed + kNB;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tdone + 1);
  int* eshift = reinterpret_cast<int*>(tmem_slot + 4);  // [C][RR]: data offset of each ring row (-1: zero row)

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxSlots; ++s) {
      mbar_init(&afull[s], QT * 128);
      mbar_init(&aempty[s], 1);
    }
    if (p.dtma) prefetch_tmap(&dmap);
    for (int s = 0; s < kBfDSlots; ++s) {
      mbar_init(&dfull[s], p.dtma ? 1 : 32);
      mbar_init(&dempty[s], 1);
    }
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&loaded[b], 1);
      mbar_init(&consumed[b], QT * 128);
    }
    mbar_init(tdone, 1);
    mbar_fence_init();
  }
  if (warp == 12) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  int u0, u1;
  bf_range(p, u0, u1);
  const int my_units = u1 - u0;
  const std::uint32_t a_col0 = std::uint32_t(QT * p.BN);  // A ring after the QT accumulators

  if (warp < 4 * QT) {
    // ------------------------------------------------ A producers: lane = x row q = (c, r, s)
    const int qt = warp >> 2, quarter = warp & 3;
    const int q = qt * 128 + quarter * 32 + lane;
    const bool qok = q < p.rows;
    const int qe = qok ? q : 0;
    const int c = qe / (p.R * p.S), rs = qe - c * p.R * p.S, r = rs / p.S, s = rs - r * p.S;
    const std::uint32_t tq = tmem + (std::uint32_t(quarter * 32) << 16) + a_col0 + std::uint32_t(qt * 32);
    RowWalkB walk;
    RingPos ra;
    FCT_T0;
    for (int i = 0; i < my_units; ++i) {
      walk.step(p, u0 + i);
      FCT_W(t_w1, mbar_wait(&loaded[i % kNB], (i / kNB) & 1));
      int prow = walk.vmod + r;
      if (prow >= p.RR) prow -= p.RR;
      // the ring row's data offset (bulk copies land 16 B aligned), -1: off the image
      const int e = eshift[c * p.RR + prow];
      const std::uint32_t xb = smem_u32(ring) + std::uint32_t(((c * p.RR + prow) * p.pitch + max(e, 0) + s) * 4);
      const bool live = qok && e >= 0;
      for (int b = 0; b < p.nblk; ++b, ra.step(p.nslots)) {
        const int slot = ra.slot;
        FCT_W(t_w2, mbar_wait(&aempty[slot], ra.ph ^ 1));
        tc_fence_after();
        const int ow0 = b * 32;
        const std::uint32_t a0 = xb + std::uint32_t(ow0 * SW * 4);
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[j]) : "r"(a0 + j * SW * 4));
        // only taps on the image count: the ring around the copied row data
        // (padding columns, rows off the image, pixels past the row end) may
        // hold anything
        const int iw0 = ow0 * SW + s - p.pw;
        // (skipping this test for interior blocks measured slower: ResNet
        // conv1 BF 392 -> 466 us -- the branch splits the warp's lanes)
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (!live || ow0 + j >= p.OW || unsigned(iw0 + j * SW) >= unsigned(p.W)) v[j] = 0.f;
        tmem_st32(tq + std::uint32_t(slot * QT * 32), v);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&afull[slot]);
      }
      mbar_arrive(&consumed[i % kNB]);
    }
    FCT_PRINT("bf prod (loaded, aempty)");
    // ------------------------------------------------ this CTA's partial sums -> its slice
    if (my_units > 0) {
      mbar_wait_sleep(tdone, 0);
      tc_fence_after();
    }
    float* slice = p.slices + (long long)blockIdx.x * p.rows * p.K + (long long)q * p.K;
    for (int k0 = 0; k0 < p.BN; k0 += 32) {
      float v[32];
      if (my_units > 0) {
        tmem_ld32(tmem + (std::uint32_t(quarter * 32) << 16) + std::uint32_t(qt * p.BN + k0), v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
      if (!qok) continue;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (k0 + j < p.K) slice[k0 + j] = v[j];
    }
  } else if (warp == 12) {
    // ------------------------------------------------ MMA issuer (whole warp, one elected lane)
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN);
    const std::uint64_t dd0 = umma_desc_sw128(smem_u32(dring));
    const std::uint32_t dslot_desc = dslot_bytes >> 4;
    int g = 0;
    const int total = my_units * p.nblk;
    FCT_T0;
    RingPos rs;
    for (; g < total; ++g, rs.step(p.nslots)) {
      const int slot = rs.slot, ds = g % kBfDSlots;
      FCT_W(t_w1, mbar_wait(&afull[slot], rs.ph));
      FCT_W(t_w2, mbar_wait(&dfull[ds], (g / kBfDSlots) & 1));
      tc_fence_after();
      const std::uint32_t ta = tmem + a_col0 + std::uint32_t(slot * QT * 32);
      const std::uint64_t bd = dd0 + std::uint64_t(ds) * dslot_desc;
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int t = 0; t < QT; ++t)
          mma_tf32_ts_warp(tmem + std::uint32_t(t * p.BN), ta + std::uint32_t(t * 32 + 8 * k), bd + 2 * k, idesc,
                           (g | k) ? 1u : 0u);
      mma_commit_warp(&aempty[slot]);
      mma_commit_warp(&dempty[ds]);
      __syncwarp();
    }
    FCT_PRINT("bf mma (afull, dfull)");
    if (total > 0) mma_commit_warp(tdone);
    __syncwarp();
  } else if (warp == 13) {
    // ------------------------------------------------ x-row loader: one bulk copy per new ring row
    // (issued by one lane each, all rows of a unit in flight at once), landed
    // 16 B aligned with the row's shift recorded in eshift
    RowWalkB walk;
    __shared__ int hist[kHist];  // (shared: a local array spilled to L2-latency local memory)
    int waited = -1;
    FCT_T0;
    for (int i = 0; i < my_units; ++i) {
      const int u = u0 + i;
      const bool fresh = walk.next(p, u);
      const int n = u / p.OH, oh = u - n * p.OH;
      const int lo = fresh ? walk.vstart : walk.vend - p.sh;
      const int cnt = walk.vend - lo;
      const int ov = walk.vend - 1 - p.RR;
      int need = -1;
      for (int j = i - 1; j >= 0 && j >= i - kHist; --j)
        if (hist[j % kHist] <= ov) {
          need = j;
          break;
        }
      if (need > waited) {
        FCT_W(t_w1, mbar_wait_sleep(&consumed[need % kNB], (need / kNB) & 1));
        waited = need;
      }
      __syncwarp();
      if (lane == 0) hist[i % kHist] = walk.vstart;
      __syncwarp();
      const int nrows = p.C * cnt;  // <= 4 * 11: at most two rows per lane
      std::uint32_t bytes[2] = {0, 0}, dst[2] = {0, 0};
      const float* src[2] = {nullptr, nullptr};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = lane + 32 * h;
        if (row >= nrows) continue;
        const int c = row / cnt, vr = lo + row - c * cnt;
        const int ih = oh * p.sh - p.ph + (vr - walk.vstart);
        const int prow = vr % p.RR;
        int e = -1;
        if (unsigned(ih) < unsigned(p.H)) {
          const float* rp = p.x + ((long long)(n * p.C + c) * p.H + ih) * p.W;
          const std::uintptr_t af = reinterpret_cast<std::uintptr_t>(rp) >> 2;  // float address
          e = int((af - std::uintptr_t(p.pw)) & 3);
          const std::uintptr_t a0 = af & ~std::uintptr_t(3), a1 = (af + p.W + 3) & ~std::uintptr_t(3);
          src[h] = reinterpret_cast<const float*>(a0 << 2);
          bytes[h] = std::uint32_t(a1 - a0) * 4;
          dst[h] = smem_u32(ring) + std::uint32_t(((c * p.RR + prow) * p.pitch + e + p.pw - int(af & 3)) * 4);
        }
        eshift[c * p.RR + prow] = e;
      }
      std::uint32_t total = bytes[0] + bytes[1];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
      __syncwarp();
      FCT_W(t_w2, if (lane == 0) mbar_expect_tx(&loaded[i % kNB], total));  // arrive (releases eshift) + the bytes to come
      __syncwarp();
      FCT_W(t_w3,
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (bytes[h]) bulk_g2s_u32(dst[h], src[h], bytes[h], &loaded[i % kNB]));
    }
    FCT_PRINT("bf xload (consumed, -)");
  } else if (warp >= 13 + kBfXLoaders && p.dtma) {
    // ------------------------------------------------ dy blocks by TMA: one 3-D box (32 pixels x K) each,
    // landing as the SWIZZLE_128B K-major operand, zero past the row end
    if (warp == 13 + kBfXLoaders && lane == 0) {
      const int total = my_units * p.nblk;
      for (int g = 0; g < total; ++g) {
        const int u = u0 + g / p.nblk, b = g % p.nblk;
        const int n = u / p.OH, oh = u - n * p.OH;
        const int ds = g % kBfDSlots;
        mbar_wait_sleep(&dempty[ds], ((g / kBfDSlots) & 1) ^ 1);
        mbar_expect_tx(&dfull[ds], dslot_bytes);
        tma_3d_b(smem_u32(dring) + std::uint32_t(ds) * dslot_bytes, &dmap, &dfull[ds], b * 32, oh, n * p.K);
      }
    }
    __syncwarp();
  } else if (warp >= 13 + kBfXLoaders) {
    // ------------------------------------------------ dy loaders: warp g % 4 owns block g
    // ([K rows x 32 pixels], zero past the row end), all its rows in flight at once
    const int dw = warp - 13 - kBfXLoaders;
    const long long ks = (long long)p.OH * p.OW;
    const int total = my_units * p.nblk;
    FCT_T0;
    for (int g = dw; g < total; g += kBfDLoaders) {
      const int u = u0 + g / p.nblk, b = g % p.nblk;
      const int n = u / p.OH, oh = u - n * p.OH;
      const int ds = g % kBfDSlots;
      const int ow = b * 32 + lane;
      const bool pok = ow < p.OW;
      const float* src = p.dy + (long long)n * p.KOHW + (long long)oh * p.OW + (pok ? ow : 0);
      float v[64];
#pragma unroll
      for (int k = 0; k < 64; ++k) v[k] = pok && k < p.K ? __ldg(src + k * ks) : 0.f;
      FCT_W(t_w1, mbar_wait_sleep(&dempty[ds], ((g / kBfDSlots) & 1) ^ 1));
      unsigned char* slotp = dring + ds * dslot_bytes + (lane & 3) * 4;
#pragma unroll
      for (int k = 0; k < 64; ++k)
        if (k < p.BN) *reinterpret_cast<float*>(slotp + k * 128 + (((lane >> 2) ^ (k & 7)) << 4)) = v[k];
      fence_async_smem();  // generic stores -> the tensor core's async-proxy reads
      mbar_arrive(&dfull[ds]);
    }
    FCT_PRINT("bf dyload (dempty, -)");
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 12) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// ---------------------------------------------------------- stride-1 variant
// The same D[q][k] = sum_px x-tap[q][px] * dy[k][px] for stride-1 layers with
// many channels (ResNet 3x3 layers: C*R*S = 576 .. 2304 x rows). The x rows q
// are split into groups of QT*128 (QT = 3 for K <= 64, 2 for K <= 128) and the
// grid into one set of CTAs per group, each CTA accumulating its group's
// rows over a contiguous run of output rows. Operands come by TMA straight
// from the caller's NCHW tensors (16 B aligned rows: W % 4 == 0): per output
// row one 4-D box of x (XW columns from w = -4, the group's CR channels,
// zero-filled off the image) into a row ring [RR][CR][XW] (ring rows padded
// so a warp's (c, r, s) lanes spread over the banks), and per 32-pixel block
// one 3-D box of dy (32 pixels x K channels) that lands as the SWIZZLE_128B
// K-major B operand. No loader threads touch the data. (Ring rows start 128 B
// aligned, as TMA destinations must.)
constexpr int kB1Threads = 15 * 32;  // 0 .. 4*QT-1 producers, 12 MMA, 13 x TMA, 14 dy TMA
constexpr int kB1MaxDS = 8;

struct B1Params {
  float* slices;
  int C, H, W, K, R, S, ph, pw, OH, OW;
  int rows, BN, nblk, units, RR, XW, RS, CR, QG, cpg, nslots, nds;
};

__device__ __forceinline__ void tma_4d(std::uint32_t dst, const void* tmap, std::uint64_t* bar, int x, int y, int z,
                                       int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "r"(w)
      : "memory");
}
__device__ __forceinline__ void tma_3d(std::uint32_t dst, const void* tmap, std::uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

struct RowWalk1 {
  int vstart = 0, vend = 0, n = -1;
  int oh = 0, vmod = 0;  // step(): row within the image, vstart % RR
  __device__ __forceinline__ bool next(const B1Params& p, int u) {
    const int nn = u / p.OH;
    const bool fresh = nn != n;
    vstart = fresh ? vend : vstart + 1;
    vend = vstart + p.R;
    n = nn;
    return fresh;
  }
  // next() for consecutive units (RowWalkB::step)
  __device__ __forceinline__ bool step(const B1Params& p, int u) {
    bool fresh;
    if (n < 0) {
      n = u / p.OH;
      oh = u - n * p.OH;
      fresh = true;
    } else if (++oh == p.OH) {
      oh = 0;
      ++n;
      fresh = true;
    } else {
      fresh = false;
    }
    vmod += fresh ? vend - vstart : 1;
    while (vmod >= p.RR) vmod -= p.RR;
    vstart = fresh ? vend : vstart + 1;
    vend = vstart + p.R;
    return fresh;
  }
};

template <int QT>
__global__ void __launch_bounds__(kB1Threads, 1)
    fct_bwdf1_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap dmap,
                     const B1Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t dslot_bytes = std::uint32_t(p.BN) * 128;
  unsigned char* dring = smem;  // nds x [BN rows x 128 B], SWIZZLE_128B K-major
  float* ring = reinterpret_cast<float*>(dring + p.nds * dslot_bytes);  // [RR] x (RS floats: [CR][XW], 128 B rows)
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(ring + p.RR * p.RS);
  std::uint64_t* afull = bars;
  std::uint64_t* aempty = afull + kMaxSlots;
  std::uint64_t* dfull = aempty + kMaxSlots;
  std::uint64_t* dempty = dfull + kB1MaxDS;
  std::uint64_t* loaded = dempty + kB1MaxDS;
  std::uint64_t* consumed = loaded + kNB;
  std::uint64_t* tdone = consumed + kNB;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tdone + 1);
  if (threadIdx.x == 0) {
    prefetch_tmap(&xmap);
    prefetch_tmap(&dmap);
    for (int s = 0; s < kMaxSlots; ++s) {
      mbar_init(&afull[s], QT * 128);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < kB1MaxDS; ++s) {
      mbar_init(&dfull[s], 1);
      mbar_init(&dempty[s], 1);
    }
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&loaded[b], 1);
      mbar_init(&consumed[b], QT * 128);
    }
    mbar_init(tdone, 1);
    mbar_fence_init();
  }
  if (warp == 12) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_wait();
  const std::uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const int grp = blockIdx.x / p.cpg, bi = blockIdx.x - grp * p.cpg;
  const int u0 = int((long long)bi * p.units / p.cpg), u1 = int((long long)(bi + 1) * p.units / p.cpg);
  const int my_units = u1 - u0;
  const int c_lo = grp * p.CR;  // the group's whole channels [c_lo, c_lo + CR)
  const std::uint32_t a_col0 = std::uint32_t(QT * p.BN);

  if (warp < 4 * QT) {
    // ------------------------------------------------ A producers: lane = x row q = (c, r, s) of the group
    // lane ql = (r * CR + cl) * S + s: a warp's lanes share r (mostly) and
    // span ~10 channels x S taps, which the channel stride XW = 12 (mod 32)
    // spreads over the banks (c-major order put lanes differing only in r,
    // 3 x 3 = 9 rows apart, on one bank: 2.8 wavefronts per load)
    const int qt = warp >> 2, quarter = warp & 3;
    const int ql = qt * 128 + quarter * 32 + lane;
    const int rcl = ql / p.S, s = ql - rcl * p.S, r = rcl / p.CR, cl = rcl - r * p.CR;
    const bool qok = r < p.R && c_lo + cl < p.C;
    const int xoff = (qok ? cl * p.XW + s : 0) + 4 - p.pw;  // ring column 0 is w = -4
    const std::uint32_t tq = tmem + (std::uint32_t(quarter * 32) << 16) + a_col0 + std::uint32_t(qt * 32);
    RowWalk1 walk;
    RingPos rs;
    for (int i = 0; i < my_units; ++i) {
      walk.step(p, u0 + i);
      mbar_wait(&loaded[i % kNB], (i / kNB) & 1);
      int prow = walk.vmod + (qok ? r : 0);
      if (prow >= p.RR) prow -= p.RR;
      const std::uint32_t xb = smem_u32(ring) + std::uint32_t((prow * p.RS + xoff) * 4);
      for (int b = 0; b < p.nblk; ++b, rs.step(p.nslots)) {
        const int slot = rs.slot;
        mbar_wait(&aempty[slot], rs.ph ^ 1);
        tc_fence_after();
        const int ow0 = b * 32;
        const std::uint32_t a0 = xb + std::uint32_t(ow0 * 4);
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[j]) : "r"(a0 + j * 4));
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (!qok || ow0 + j >= p.OW) v[j] = 0.f;
        tmem_st32(tq + std::uint32_t(slot * QT * 32), v);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&afull[slot]);
      }
      mbar_arrive(&consumed[i % kNB]);
    }
    if (my_units > 0) {
      mbar_wait_sleep(tdone, 0);
      tc_fence_after();
    }
    float* slice = p.slices + ((long long)blockIdx.x * p.QG + ql) * p.K;
    for (int k0 = 0; k0 < p.BN; k0 += 32) {
      float v[32];
      if (my_units > 0) {
        tmem_ld32(tmem + (std::uint32_t(quarter * 32) << 16) + std::uint32_t(qt * p.BN + k0), v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
      if (!qok) continue;
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        if (k0 + j + 4 <= p.K)
          *reinterpret_cast<float4*>(slice + k0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
  } else if (warp == 12) {
    // ------------------------------------------------ MMA issuer (whole warp, one elected lane)
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN);
    const std::uint64_t dd0 = umma_desc_sw128(smem_u32(dring));
    const std::uint32_t dslot_desc = dslot_bytes >> 4;
    const int total = my_units * p.nblk;
    RingPos rs, rd;
    for (int g = 0; g < total; ++g, rs.step(p.nslots), rd.step(p.nds)) {
      const int slot = rs.slot, ds = rd.slot;
      mbar_wait(&afull[slot], rs.ph);
      mbar_wait(&dfull[ds], rd.ph);
      tc_fence_after();
      const std::uint32_t ta = tmem + a_col0 + std::uint32_t(slot * QT * 32);
      const std::uint64_t bd = dd0 + std::uint64_t(ds) * dslot_desc;
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int t = 0; t < QT; ++t)
          mma_tf32_ts_warp(tmem + std::uint32_t(t * p.BN), ta + std::uint32_t(t * 32 + 8 * k), bd + 2 * k, idesc,
                           (g | k) ? 1u : 0u);
      mma_commit_warp(&aempty[slot]);
      mma_commit_warp(&dempty[ds]);
      __syncwarp();
    }
    if (total > 0) mma_commit_warp(tdone);
    __syncwarp();
  } else if (warp == 13) {
    // ------------------------------------------------ x rows: one TMA box per new output row
    RowWalk1 walk;
    __shared__ int hist[kHist];
    int waited = -1;
    for (int i = 0; i < my_units; ++i) {
      const int u = u0 + i;
      const bool fresh = walk.next(p, u);
      const int n = u / p.OH, oh = u - n * p.OH;
      const int lo = fresh ? walk.vstart : walk.vend - 1;
      const int ov = walk.vend - 1 - p.RR;
      int need = -1;
      for (int j = i - 1; j >= 0 && j >= i - kHist; --j)
        if (hist[j % kHist] <= ov) {
          need = j;
          break;
        }
      if (need > waited) {
        mbar_wait_sleep(&consumed[need % kNB], (need / kNB) & 1);
        waited = need;
      }
      __syncwarp();
      if (lane == 0) {
        hist[i % kHist] = walk.vstart;
        const int cnt = walk.vend - lo;
        mbar_expect_tx(&loaded[i % kNB], std::uint32_t(cnt * p.CR * p.XW * 4));
        for (int vr = lo; vr < walk.vend; ++vr)
          tma_4d(smem_u32(ring) + std::uint32_t((vr % p.RR) * p.RS * 4), &xmap, &loaded[i % kNB], -4,
                 oh - p.ph + (vr - walk.vstart), c_lo, n);
      }
      __syncwarp();
    }
  } else if (warp == 14) {
    // ------------------------------------------------ dy blocks: one TMA box (32 pixels x K channels) each
    if (lane == 0) {
      const int total = my_units * p.nblk;
      for (int g = 0; g < total; ++g) {
        const int u = u0 + g / p.nblk, b = g - (g / p.nblk) * p.nblk;
        const int n = u / p.OH, oh = u - n * p.OH;
        const int ds = g % p.nds;
        mbar_wait_sleep(&dempty[ds], ((g / p.nds) & 1) ^ 1);
        mbar_expect_tx(&dfull[ds], dslot_bytes);
        tma_3d(smem_u32(dring) + std::uint32_t(ds) * dslot_bytes, &dmap, &dfull[ds], b * 32, oh, n * p.K);
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 12) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

// dW[k][q] = beta * dW + alpha * sum over the group's CTAs of slice[cta][q - group * QG][k], in order
struct B1Final {
  const float* slices;
  float* dw;
  float alpha, beta;
  int rows, K, QG, cpg, CR, R, S;
  FastDiv fd_K;  // 32-bit index math (dW has < 2^31 elements)
};
__global__ void __launch_bounds__(256) fct_bwdf1_finalize_kernel(const B1Final f) {
  pdl_wait();
  const std::uint32_t n = std::uint32_t(f.rows) * std::uint32_t(f.K);
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    std::uint32_t q_, k_;
    f.fd_K.divmod(i, q_, k_);
    const int q = int(q_), k = int(k_);
    const int RS = f.R * f.S, c = q / RS, rs = q - c * RS, r = rs / f.S, s = rs - r * f.S;
    const int grp = c / f.CR, ql = (r * f.CR + (c - grp * f.CR)) * f.S + s;  // the kernel's lane order
    const float* sl = f.slices + ((long long)grp * f.cpg * f.QG + ql) * f.K + k;
    const long long cstride = (long long)f.QG * f.K;
    float part[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int b = 0;
    for (; b + 8 <= f.cpg; b += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) part[j] += sl[(b + j) * cstride];
    }
    for (int j = 0; b < f.cpg; ++b, ++j) part[j] += sl[b * cstride];
    const float acc = ((part[0] + part[1]) + (part[2] + part[3])) + ((part[4] + part[5]) + (part[6] + part[7]));
    float* d = f.dw + (long long)k * f.rows + q;
    *d = f.beta == 0.f ? f.alpha * acc : f.alpha * acc + f.beta * *d;
  }
}

// dW[k][q] = beta * dW + alpha * sum_g slice_g[q][k], slices added in order
struct BFinal {
  const float* slices;
  float* dw;
  float alpha, beta;
  int rows, K, nslices;
  FastDiv fd_K;  // 32-bit index math (dW has < 2^31 elements)
};
__global__ void __launch_bounds__(256) fct_bwdf_finalize_kernel(const BFinal f) {
  pdl_wait();
  const long long n = (long long)f.rows * f.K;
  for (std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < std::uint32_t(n); i += gridDim.x * blockDim.x) {
    std::uint32_t q_, k_;
    f.fd_K.divmod(i, q_, k_);
    const int q = int(q_), k = int(k_);
    // eight interleaved partial sums (loads in flight instead of one
    // dependent chain of ~148), combined in a fixed order: deterministic
    float part[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int g = 0;
    for (; g + 8 <= f.nslices; g += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) part[j] += f.slices[(g + j) * n + i];
    }
    for (int j = 0; g < f.nslices; ++g, ++j) part[j] += f.slices[g * n + i];
    const float acc = ((part[0] + part[1]) + (part[2] + part[3])) + ((part[4] + part[5]) + (part[6] + part[7]));
    float* d = f.dw + (long long)k * f.rows + q;
    *d = f.beta == 0.f ? f.alpha * acc : f.alpha * acc + f.beta * *d;
  }
}

// ============================================================== BackwardData
//
//   dx[n][c][h][w] = beta * dx + alpha * sum_{k,r,s} dy[n][k][(h+ph-r)/sh][(w+pw-s)/sw] * w[k][c][r][s]
//   (terms with (h+ph-r) % sh == 0 and (w+pw-s) % sw == 0; reference_conv.hpp:104-138)
//
// Stride-phase form: with h + ph = i*sh + a, w + pw = j*sw + b (a, b < sh),
//   dx[c][i*sh+a-ph][j*sw+b-pw] = sum_{k,t,u} dy[k][i-t][j-u] * w[k][c][a+sh*t][b+sw*u]
// so one "phase pixel" (i, j) -- a TMEM lane -- owns the sh*sw dx pixels of
// every channel: N = C*sh*sw columns (AlexNet conv1: 48), reduction
// (t, u, k) over the T x U taps of each phase and the K dy channels. The
// filter, rearranged into that (c, a, b) x (t, u, k) matrix, stays resident
// in shared memory; the dy rows a tile of phase rows needs sit in a ring
// (bulk copies, one per channel row, landed 16 B aligned -- each row's float
// shift follows from its address, so producers compute it instead of
// looking it up); producer thread (i, j) reads dy[k][i-t][j-u] for 32
// channels per slot (lanes = consecutive j: conflict-free) and writes them
// to TMEM; one ring slot = one (t, u) tap = 64 reduction columns. The
// epilogue scatters each lane's 48 columns to its sh x sw dx block of every
// channel.
constexpr int kBdKp = 64;  // reduction columns per (t, u) tap: K <= 64, zero-padded
constexpr int kBdKS = 68;  // ring floats per position: 64 channels + 4 (16 B rows 17 chunks apart: conflict-free)
constexpr int kBdLoaders = 4;
// warps: 0-7 A producers, 8-11 epilogue, 12 MMA issuer, 13-16 dy-row loaders
constexpr int kBdThreads = (13 + kBdLoaders) * 32;

struct DParams {
  const float* dy;
  const float* w;
  float* dx;
  float alpha, beta;
  int C, H, W, K, R, S, ph, pw, sh, OH, OW;
  int T, U, Hq, Wq, TR, np, tps, SW, nstrip, units, BN, AS, nslots, RR, XP, PH;
  long long OHW, KOHW, CHW;
};

struct RowWalkD {
  int vstart = 0, vend = 0, n = -1;
  __device__ __forceinline__ bool next(const DParams& p, int u) {
    const int nn = u / p.tps;  // (image, column strip)
    const bool fresh = nn != n;
    vstart = fresh ? vend : vstart + p.TR;
    vend = vstart + p.PH;
    n = nn;
    return fresh;
  }
};

template <int SH, int TU, bool PAIR>
__global__ void __launch_bounds__(kBdThreads, 1) fct_bwdd_kernel(const DParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kChunks = TU * kBdKp / 32;
  // CTA pair: each CTA holds half of the filter's N rows and its own 128
  // lanes of A and D; rank 0 issues M = 256 MMAs for both
  const std::uint32_t rank = PAIR ? cluster_rank() : 0;
  const int BH = PAIR ? p.BN / 2 : p.BN;  // filter rows held here
  const std::uint32_t b_bytes = std::uint32_t(kChunks) * BH * 128;
  float* ring = reinterpret_cast<float*>(smem + b_bytes);  // [RR][XP][kBdKS]
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(ring + p.RR * p.XP * kBdKS);
  std::uint64_t* afull = bars;
  std::uint64_t* aempty = afull + kMaxSlots;
  std::uint64_t* loaded = aempty + kMaxSlots;
  std::uint64_t* consumed = loaded + kNB;
  std::uint64_t* tfull = consumed + kNB;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);

  // the filter as B[(c, a, b)][(t, u, k)] = w[k][c][a + sh t][b + sh u] (0 off the filter),
  // K-major SWIZZLE_128B, BN rows per 32-column chunk
  {
    const int per_chunk = BH * 32;
    const int total = kChunks * per_chunk;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int chunk = i / per_chunk, rem = i - chunk * per_chunk;
      const int lrow = rem >> 5, j = rem & 31, row = int(rank) * BH + lrow;
      const int kk = chunk * 32 + j;
      const int tu = kk / kBdKp, k = kk - tu * kBdKp;
      const int t = tu / p.U, u = tu - t * p.U;
      const int c = row / (p.sh * p.sh), ab = row - c * p.sh * p.sh, a = ab / p.sh, b = ab - a * p.sh;
      const int r = a + p.sh * t, q = b + p.sh * u;
      float v = 0.f;
      if (c < p.C && k < p.K && r < p.R && q < p.S) v = p.w[((long long)(k * p.C + c) * p.R + r) * p.S + q];
      *reinterpret_cast<float*>(smem + chunk * BH * 128 + lrow * 128 + (((j >> 2) ^ (lrow & 7)) << 4) + (j & 3) * 4) =
          v;
    }
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxSlots; ++s) {
      mbar_init(&afull[s], PAIR ? 512 : 256);  // PAIR: both CTAs' producers, on rank 0's barrier
      mbar_init(&aempty[s], 1);
    }
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&loaded[b], kBdLoaders * 32);
      mbar_init(&consumed[b], 256);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 256 : 128);
    }
    mbar_fence_init();
  }
  if (warp == 12) {
    if constexpr (PAIR) tmem_alloc_2sm<512>(tmem_slot);
    else tmem_alloc<512>(tmem_slot);
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // both CTAs' barriers initialised before any remote arrive
  tc_fence_after();
  const std::uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  // units: contiguous runs; a pair splits its run in two halves, the second
  // CTA padding its half with a dummy tile when the run is odd (both CTAs
  // must feed every pair MMA)
  int t0, my_units, real_units;
  if constexpr (PAIR) {
    const int pairs = gridDim.x >> 1, pid = blockIdx.x >> 1;
    const int pa0 = int((long long)pid * p.units / pairs), pa1 = int((long long)(pid + 1) * p.units / pairs);
    const int h = (pa1 - pa0 + 1) >> 1;
    t0 = rank == 0 ? pa0 : pa0 + h;
    my_units = h;
    real_units = rank == 0 ? h : pa1 - pa0 - h;
  } else {
    t0 = int((long long)blockIdx.x * p.units / gridDim.x);
    my_units = real_units = int((long long)(blockIdx.x + 1) * p.units / gridDim.x) - t0;
  }
  const std::uint32_t afull0 = PAIR ? mapa(smem_u32(&afull[0]), 0) : 0;
  const std::uint32_t tempty0 = PAIR ? mapa(smem_u32(&tempty[0]), 0) : 0;
  const std::uint32_t a_col0 = 2u * std::uint32_t(p.AS);

  if (warp < 8) {
    // ------------------------------------------------ A producers: lane = phase pixel (i, j);
    // warps w and w + 4 share lane quarter w % 4 and take channels [0, 32) / [32, 64)
    const int quarter = warp & 3, half = warp >> 2;
    const int px = quarter * 32 + lane;
    const bool pok = px < p.np;
    const int pe = pok ? px : 0;
    const int rl = pe / p.SW, jl = pe - rl * p.SW;  // strip-local phase column
    const std::uint32_t tlane = tmem + (std::uint32_t(quarter * 32) << 16);
    const int k0 = half * 32;
    RowWalkD walk;
    // slot / parity and tap (t, u) are stepped, not divided: the runtime
    // divisions were most of this loop's instructions (ResNet conv1 BD, ncu)
    int slot = 0, sph = 0;
    FCT_T0;
    for (int i = 0; i < my_units; ++i) {
      const int u_ = t0 + i;
      walk.next(p, u_);
      FCT_W(t_w1, mbar_wait(&loaded[i % kNB], (i / kNB) & 1));
      const int row0 = (walk.vstart + rl + p.T - 1) % p.RR;
      const std::uint32_t col0 = smem_u32(ring) + std::uint32_t(((jl + p.U - 1) * kBdKS + k0) * 4);
      int t = 0, u = 0;
      for (int tu = 0; tu < TU; ++tu) {
        // ring row of dy row i - t, position j - u (+ U - 1): its 32 channels are contiguous
        const int prow = row0 - t < 0 ? row0 - t + p.RR : row0 - t;
        const std::uint32_t addr = col0 + std::uint32_t((prow * p.XP - u) * kBdKS * 4);
        FCT_W(t_w2, mbar_wait(&aempty[slot], sph ^ 1));
        tc_fence_after();
        float v[32];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(v[4 * q]), "=f"(v[4 * q + 1]), "=f"(v[4 * q + 2]), "=f"(v[4 * q + 3])
                       : "r"(addr + 16 * q));
        tmem_st32(tlane + a_col0 + std::uint32_t(slot * kBdKp + half * 32), v);
        tmem_st_wait();
        tc_fence_before();
        if constexpr (PAIR) mbar_arrive_remote(afull0 + std::uint32_t(slot) * 8);
        else mbar_arrive(&afull[slot]);
        if (++u == p.U) {
          u = 0;
          ++t;
        }
        if (++slot == p.nslots) {
          slot = 0;
          sph ^= 1;
        }
      }
      mbar_arrive(&consumed[i % kNB]);
    }
    FCT_PRINT("bd prod (loaded, aempty)");
  } else if (warp < 12) {
    // ------------------------------------------------ epilogue: lane (i, j) -> its SH x SH dx blocks;
    // columns are (c, a, b) with b fastest, so a lane's SH values of one
    // (c, a) are SH consecutive dx floats: one vector store when the row's
    // alignment (uniform across the warp) allows
    const int quarter = warp & 3;
    const int px = quarter * 32 + lane;
    const int rl = px / p.SW, jl = px - rl * p.SW;
    const long long HW = (long long)p.H * p.W;
    FCT_T0;
    for (int i = 0; i < my_units; ++i) {
      const int u_ = t0 + i;
      const int key = u_ / p.tps, n = key / p.nstrip;
      const int j = (key - n * p.nstrip) * p.SW + jl, ii = (u_ - key * p.tps) * p.TR + rl;
      const int w0 = j * SH - p.pw;
      const bool wall = w0 >= 0 && w0 + SH <= p.W;  // all SH columns on the image
      const int acc = i & 1;
      FCT_W(t_w1, mbar_wait_sleep(&tfull[acc], (i >> 1) & 1));
      tc_fence_after();
      const bool live = px < p.np && ii < p.Hq && j < p.Wq && i < real_units;
      const int h0 = ii * SH - p.ph;
      float* dxn = p.dx + (long long)n * p.CHW;
      for (int c0 = 0; c0 < p.BN; c0 += 32) {
        float v[32];
        tmem_ld32(tmem + (std::uint32_t(quarter * 32) << 16) + std::uint32_t(acc * p.AS + c0), v);
        if (!live) continue;
#pragma unroll
        for (int rr = 0; rr < 32 / SH; ++rr) {  // one (c, a) row of SH values per step
          const int ca = c0 / SH + rr, c = ca / SH, a = ca - c * SH;
          const int h = h0 + a;
          if (c >= p.C || unsigned(h) >= unsigned(p.H)) continue;
          float* d = dxn + c * HW + (long long)h * p.W + w0;
          if (p.beta == 0.f && wall) {
            float o[SH];
#pragma unroll
            for (int b = 0; b < SH; ++b) o[b] = p.alpha * v[rr * SH + b];
            const unsigned mis = unsigned(reinterpret_cast<std::uintptr_t>(d) >> 2) & 3;
            if constexpr (SH == 4) {
              if (mis == 0) {
                *reinterpret_cast<float4*>(d) = make_float4(o[0], o[1], o[2], o[3]);
              } else if (mis == 2) {
                *reinterpret_cast<float2*>(d) = make_float2(o[0], o[1]);
                *reinterpret_cast<float2*>(d + 2) = make_float2(o[2], o[3]);
              } else {
                d[0] = o[0];
                *reinterpret_cast<float2*>(d + 1 + (mis == 1 ? 0 : 0)) = make_float2(o[1], o[2]);
                d[3] = o[3];
              }
            } else {
              if ((mis & 1) == 0) {
                *reinterpret_cast<float2*>(d) = make_float2(o[0], o[1]);
              } else {
                d[0] = o[0];
                d[1] = o[1];
              }
            }
          } else {
#pragma unroll
            for (int b = 0; b < SH; ++b) {
              if (unsigned(w0 + b) >= unsigned(p.W)) continue;
              const float val = p.alpha * v[rr * SH + b];
              d[b] = p.beta == 0.f ? val : val + p.beta * d[b];
            }
          }
        }
      }
      tc_fence_before();
      if constexpr (PAIR) mbar_arrive_remote(tempty0 + std::uint32_t(acc) * 8);
      else mbar_arrive(&tempty[acc]);
    }
    FCT_PRINT("bd epi (tfull, -)");
  } else if (warp == 12) {
    // ------------------------------------------------ MMA issuer (whole warp, one elected lane;
    // PAIR: rank 0 only, M = 256 over both CTAs' lanes, commits multicast to both)
    if (PAIR && rank != 0) goto mma_done;
    {
    const std::uint32_t idesc = idesc_tf32(PAIR ? 2 * kBM : kBM, p.BN);
    const std::uint64_t bdesc0 = umma_desc_sw128(smem_u32(smem));
    const std::uint32_t chunk_desc = std::uint32_t(BH * 128) >> 4;
    int slot = 0, sph = 0;
    FCT_T0;
    for (int i = 0; i < my_units; ++i) {
      const int acc = i & 1;
      FCT_W(t_w1, mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1));
      tc_fence_after();
      const std::uint32_t d = tmem + std::uint32_t(acc * p.AS);
      std::uint64_t bd = bdesc0;
      for (int tu = 0; tu < TU; ++tu) {
        FCT_W(t_w2, mbar_wait(&afull[slot], sph));
        tc_fence_after();
        const std::uint32_t ta = tmem + a_col0 + std::uint32_t(slot * kBdKp);
#pragma unroll
        for (int m = 0; m < kBdKp / 8; ++m) {
          if constexpr (PAIR)
            mma_tf32_ts_2sm_warp(d, ta + std::uint32_t(8 * m), bd + (m >> 2) * chunk_desc + 2 * (m & 3), idesc,
                                 (tu | m) ? 1u : 0u);
          else
            mma_tf32_ts_warp(d, ta + std::uint32_t(8 * m), bd + (m >> 2) * chunk_desc + 2 * (m & 3), idesc,
                             (tu | m) ? 1u : 0u);
        }
        if constexpr (PAIR) {
          mma_commit_2sm_w(&aempty[slot], 3);
          if (tu + 1 == TU) mma_commit_2sm_w(&tfull[acc], 3);
        } else {
          mma_commit_warp(&aempty[slot]);
          if (tu + 1 == TU) mma_commit_warp(&tfull[acc]);
        }
        __syncwarp();
        bd += (kBdKp / 32) * chunk_desc;
        if (++slot == p.nslots) {
          slot = 0;
          sph ^= 1;
        }
      }
    }
    FCT_PRINT("bd mma (tempty, afull)");
    }
  mma_done:;
  } else {
    // ------------------------------------------------ dy-row loaders: the dy rows each tile adds,
    // transposed to [position][channel] (4 channels per lane: 4 coalesced
    // loads, one 16 B store), zero off the tensor
    const int lw = warp - 13;
    RowWalkD walk;
    __shared__ int hist[kHist];
    int waited = -1;
    const int nxb = (p.XP + 31) / 32;
    FCT_T0;
    for (int i = 0; i < my_units; ++i) {
      const int u_ = t0 + i;
      const bool fresh = walk.next(p, u_);
      const int key = u_ / p.tps, n = key / p.nstrip, j0 = (key - n * p.nstrip) * p.SW;
      const int i0 = (u_ - key * p.tps) * p.TR;
      const int lo = fresh ? walk.vstart : walk.vend - p.TR;
      const int cnt = walk.vend - lo;
      const int ov = walk.vend - 1 - p.RR;
      int need = -1;
      for (int jj = i - 1; jj >= 0 && jj >= i - kHist; --jj)
        if (hist[jj % kHist] <= ov) {
          need = jj;
          break;
        }
      if (need > waited) {
        FCT_W(t_w1, mbar_wait_sleep(&consumed[need % kNB], (need / kNB) & 1));
        waited = need;
      }
      if (lw == 0) {
        __syncwarp();
        if (lane == 0) hist[i % kHist] = walk.vstart;
        __syncwarp();
      }
      const float* dyn = p.dy + (long long)(i < real_units ? n : 0) * p.KOHW;
      // warp lw owns channel quads lw, lw + 4, .. (16 channels); per new row,
      // every (position block, quad) of the warp is in flight at once (a
      // pair's dummy tile loads nothing: its rows are never stored)
      for (int rr = 0; rr < (i < real_units ? cnt : 0); ++rr) {
        const int y = i0 - (p.T - 1) + (lo + rr - walk.vstart);
        const bool yok = unsigned(y) < unsigned(p.OH);
        const float* rowp = dyn + (long long)(lw * 4) * p.OHW + (long long)(yok ? y : 0) * p.OW;
        float* dstrow = ring + ((lo + rr) % p.RR) * p.XP * kBdKS + lw * 4;
        float v[2][kBdKp / 16][4];
#pragma unroll
        for (int xb = 0; xb < 2; ++xb) {
          const int ow = j0 + xb * 32 + lane - (p.U - 1);
          const bool ok = yok && xb < nxb && xb * 32 + lane < p.XP && unsigned(ow) < unsigned(p.OW);
#pragma unroll
          for (int qq = 0; qq < kBdKp / 16; ++qq)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int k = lw * 4 + qq * 16 + e;
              v[xb][qq][e] = ok && k < p.K ? __ldg(rowp + (long long)(qq * 16 + e) * p.OHW + ow) : 0.f;
            }
        }
#pragma unroll
        for (int xb = 0; xb < 2; ++xb) {
          const int x = xb * 32 + lane;
          if (xb < nxb && x < p.XP) {
#pragma unroll
            for (int qq = 0; qq < kBdKp / 16; ++qq)
              *reinterpret_cast<float4*>(dstrow + x * kBdKS + qq * 16) =
                  make_float4(v[xb][qq][0], v[xb][qq][1], v[xb][qq][2], v[xb][qq][3]);
          }
        }
      }
      mbar_arrive(&loaded[i % kNB]);  // release: this thread's ring stores
    }
    FCT_PRINT("bd load (consumed, -)");
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync();  // no CTA leaves while its peer may still signal its barriers
  if (warp == 12) {
    tc_fence_after();
    if constexpr (PAIR) tmem_free_2sm<512>(tmem);
    else tmem_free<512>(tmem);
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

TGeo make_tgeo(const ConvShape& s) {
  TGeo g{};
  g.OH = s.OH();
  g.OW = s.OW();
  g.TR = std::max(1, kBM / std::max(1, g.OW));
  g.TR = std::min(g.TR, std::max(1, tune("fct_rows", g.TR)));
  g.np = g.TR * g.OW;
  g.tiles_per_img = (g.OH + g.TR - 1) / g.TR;
  g.units = s.N * g.tiles_per_img;
  g.grid = std::min(sm_count(), g.units);
  g.SP = (s.S + 3) / 4 * 4;
  g.groups = s.C * s.R;
  const int KG = g.SP == 12 ? 8 : 4;  // a slot = whole 32-float filter chunks
  g.gpad = (g.groups + KG - 1) / KG * KG;
  g.kslots = g.gpad / KG;
  g.kred = g.gpad * g.SP;
  g.nchunk = (g.kred + 31) / 32;
  g.BN = (s.K + 15) / 16 * 16;
  g.PH = (g.TR - 1) * s.sh + s.R;
  g.pitch = ((g.OW - 1) * s.sw + g.SP + 3) / 4 * 4;
  g.slot_cols = KG * g.SP;
  g.nslots = std::min(kMaxSlots, (512 - 2 * g.BN) / std::max(1, g.slot_cols));
  g.b_bytes = std::size_t(g.nchunk) * g.BN * 128;
  // ring depth: as many rows as fit, at most what the loaders' tile history
  // can track
  const std::size_t fixed = g.b_bytes + 1024 + 512;
  const std::size_t row_bytes = std::size_t(s.C) * g.pitch * 4;
  const int step = g.TR * s.sh;
  int rr = int((220 * 1024 - std::min<std::size_t>(fixed, 220 * 1024)) / row_bytes);
  rr = std::min(rr, g.PH + (kHist - 2) * step);
  // one output row per tile: the shallowest ring is fastest (ResNet conv1 F
  // 451 -> 426 us); AlexNet's two-row tiles are indifferent
  // (scripts/r02_run102.sh)
  if (g.TR == 1) rr = std::min(rr, g.PH + step);
  rr = std::min(rr, tune("fct_ring", rr));
  g.RR = std::max(rr, 1);
  g.r_bytes = row_bytes * g.RR;
  g.smem = fixed + g.r_bytes;
  return g;
}

}  // namespace

bool fct_fwd_supports(const ConvShape& s) {
  if (s.sh != s.sw || (s.sw != 2 && s.sw != 4) || s.C > 4 || s.K > 128 || !tune("fct", 1)) return false;
  const int SP = (s.S + 3) / 4 * 4;
  if (!((s.sw == 4 && SP == 12) || (s.sw == 2 && SP == 8))) return false;
  const TGeo g = make_tgeo(s);
  // the ring must hold two tiles' rows so loading overlaps consuming
  return g.OW <= kBM && g.gpad <= kMaxGroups && g.nslots >= 2 && g.RR >= g.PH + g.TR * s.sh &&
         g.smem <= 220 * 1024 && std::int64_t(s.N) * s.K * g.OH * g.OW < (1ll << 40);
}

cudaError_t fct_fwd_run(const ConvShape& s, const float* x, const float* w, float* y, float alpha, float beta,
                        cudaStream_t st) {
  const TGeo g = make_tgeo(s);
  TParams p{};
  p.x = x; p.w = w; p.y = y; p.alpha = alpha; p.beta = beta;
  p.C = s.C; p.H = s.H; p.W = s.W; p.K = s.K; p.R = s.R; p.S = s.S; p.ph = s.ph; p.pw = s.pw;
  p.sh = s.sh; p.sw = s.sw; p.OH = g.OH; p.OW = g.OW;
  p.TR = g.TR; p.np = g.np; p.tiles_per_img = g.tiles_per_img; p.units = g.units;
  p.groups = g.groups; p.kslots = g.kslots; p.nchunk = g.nchunk; p.BN = g.BN; p.PH = g.PH; p.pitch = g.pitch;
  p.nslots = g.nslots; p.RR = g.RR;
  // few new input rows per tile (ResNet conv1: 2 x 3) -> store-bound: 8 epilogue warps
  p.nepi = tune("fct_epi", s.C * g.TR * s.sh <= 8 ? 8 : 4) == 8 ? 8 : 4;
  p.dbg = tune("fct_dbg", 0);
  p.CHW = std::int64_t(s.C) * s.H * s.W;
  p.KOHW = std::int64_t(s.K) * g.OH * g.OW;
  void (*kern)(const TParams) = s.sw == 4 ? fct_fwd_kernel<4, 12, 8> : fct_fwd_kernel<2, 8, 4>;
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), int(g.smem));
  if (e != cudaSuccess) return e;
  trace_variant("fct fwd units=%d grid=%d TR=%d np=%d kslots=%d BN=%d pitch=%d slots=%d ring=%d", g.units, g.grid,
                g.TR, g.np, g.kslots, g.BN, g.pitch, g.nslots, g.RR);
  return launch_pdl(kern, dim3(g.grid), dim3(kThreads), g.smem, st, p);
}

namespace {

struct BGeo {
  int OH, OW, rows, QT, BN, nblk, units, grid, pitch, RR, nslots;
  std::size_t smem;
};

BGeo make_bgeo(const ConvShape& s) {
  BGeo g{};
  g.OH = s.OH();
  g.OW = s.OW();
  g.rows = s.C * s.R * s.S;
  g.QT = (g.rows + kBM - 1) / kBM;
  g.BN = (s.K + 15) / 16 * 16;
  g.nblk = (g.OW + 31) / 32;
  g.units = s.N * g.OH;
  g.grid = std::min(sm_count(), g.units);
  // ring pitch: a multiple of 4 floats (rows land by 16 B-aligned bulk
  // copies), covering the copied row (shift <= 3, pw, the 16 B round-up) and
  // every tap read of the last 32-pixel block; = 12 (mod 32) so a warp's
  // consecutive (r, s) lanes mostly fall in different banks
  const int need = std::max(s.pw + s.W + 10, (g.nblk * 32 - 1) * s.sw + s.S + 3);
  g.pitch = (need + 3) / 4 * 4;
  while (g.pitch % 32 != 12) g.pitch += 4;
  g.nslots = std::min(kMaxSlots, (512 - g.QT * g.BN) / std::max(1, g.QT * 32));
  const std::size_t fixed = std::size_t(kBfDSlots) * g.BN * 128 + 1024 + 2048;  // + barriers, eshift
  const std::size_t row_bytes = std::size_t(s.C) * g.pitch * 4;
  int rr = int((220 * 1024 - std::min<std::size_t>(fixed, 220 * 1024)) / row_bytes);
  rr = std::min(rr, s.R + (kHist - 2) * s.sh);
  // a shallow ring is faster (less shared memory, more L1 for the row
  // loads): AlexNet conv1 BF 273 -> 263 us at R + 2 sh - 1 rows, ResNet
  // conv1 398 -> 378 (scripts/r02_run98.sh)
  rr = std::min(rr, s.R + 2 * s.sh - 1);
  rr = std::min(rr, tune("fct_bf_ring", rr));
  g.RR = std::max(rr, 1);
  g.smem = fixed + row_bytes * g.RR;
  return g;
}

}  // namespace

bool fct_bwdf_supports(const ConvShape& s) {
  if (s.sh != s.sw || (s.sw != 2 && s.sw != 4) || s.C > 4 || s.K > 64 || !tune("fct_bf", 1)) return false;
  const BGeo g = make_bgeo(s);
  return g.QT <= kBfMaxQT && s.C * s.R <= 64 && g.nslots >= 2 && g.RR >= s.R + s.sh && g.smem <= 220 * 1024 &&
         std::int64_t(s.N) * s.C * s.H * s.W < (1ll << 40);
}

std::int64_t fct_bwdf_workspace(const ConvShape& s) {
  const BGeo g = make_bgeo(s);
  return (std::int64_t(g.grid) * g.rows * s.K * 4 + 255) / 256 * 256;
}

cudaError_t fct_bwdf_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha,
                         float beta, cudaStream_t st) {
  const BGeo g = make_bgeo(s);
  BParams p{};
  p.x = x; p.dy = dy; p.slices = static_cast<float*>(ws);
  p.C = s.C; p.H = s.H; p.W = s.W; p.K = s.K; p.R = s.R; p.S = s.S; p.ph = s.ph; p.pw = s.pw;
  p.sh = s.sh; p.sw = s.sw; p.OH = g.OH; p.OW = g.OW;
  p.rows = g.rows; p.BN = g.BN; p.nblk = g.nblk; p.units = g.units; p.RR = g.RR; p.pitch = g.pitch;
  p.nslots = g.nslots;
  p.CHW = std::int64_t(s.C) * s.H * s.W;
  p.KOHW = std::int64_t(s.K) * g.OH * g.OW;
  CUtensorMap dmap{};
  p.dtma = g.OW % 4 == 0 && (std::int64_t(g.OH) * g.OW) % 4 == 0 && s.K == g.BN &&
           (reinterpret_cast<std::uintptr_t>(dy) & 15) == 0 && tune("fct_bf_dtma", 1);
  if (p.dtma) {
    const cuuint64_t dims[3] = {cuuint64_t(g.OW), cuuint64_t(g.OH), cuuint64_t(s.N) * s.K};
    const cuuint64_t strides[2] = {cuuint64_t(g.OW) * 4, cuuint64_t(g.OH) * g.OW * 4};
    const cuuint32_t box[3] = {32, 1, cuuint32_t(g.BN)};
    const cuuint32_t es[3] = {1, 1, 1};
    if (encode_tiled_fct()(&dmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(dy), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  void (*kern)(const CUtensorMap, const BParams) = nullptr;
  if (s.sw == 4) kern = g.QT == 1 ? fct_bwdf_kernel<4, 1> : g.QT == 2 ? fct_bwdf_kernel<4, 2> : fct_bwdf_kernel<4, 3>;
  else kern = g.QT == 1 ? fct_bwdf_kernel<2, 1> : g.QT == 2 ? fct_bwdf_kernel<2, 2> : fct_bwdf_kernel<2, 3>;
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), int(g.smem));
  if (e != cudaSuccess) return e;
  trace_variant("fct bwdf units=%d grid=%d rows=%d QT=%d BN=%d nblk=%d pitch=%d ring=%d slots=%d dtma=%d", g.units,
                g.grid, g.rows, g.QT, g.BN, g.nblk, g.pitch, g.RR, g.nslots, p.dtma);
  e = launch_pdl(kern, dim3(g.grid), dim3(kBfThreads), g.smem, st, dmap, p);
  if (e != cudaSuccess) return e;
  BFinal f{p.slices, dw, alpha, beta, g.rows, s.K, g.grid, FastDiv(std::uint32_t(s.K))};
  const long long n = (long long)g.rows * s.K;
  return launch_pdl(fct_bwdf_finalize_kernel, dim3(int(std::min<long long>((n + 255) / 256, 4 * sm_count()))),
                    dim3(256), 0, st, f);
}

namespace {

struct DGeo {
  int T, U, Hq, Wq, TR, np, tps, SW, nstrip, units, grid, BN, AS, nslots, RR, XP, PH;
  bool pair;
  std::size_t smem;
};

DGeo make_dgeo(const ConvShape& s) {
  DGeo g{};
  const int OH = s.OH(), OW = s.OW();
  g.T = (s.R + s.sh - 1) / s.sh;
  g.U = (s.S + s.sw - 1) / s.sw;
  g.Hq = (s.H - 1 + s.ph) / s.sh + 1;
  g.Wq = (s.W - 1 + s.pw) / s.sw + 1;
  g.BN = (s.C * s.sh * s.sw + 15) / 16 * 16;
  g.AS = (g.BN + 31) / 32 * 32;
  g.nslots = std::min(kMaxSlots, (512 - 2 * g.AS) / kBdKp);
  // CTA pairs (M = 256 per MMA, each CTA holding half the filter rows):
  // exact, but measured slower (AlexNet conv1 BD 361 -> 388 us, ResNet conv1
  // 1052 -> 1571: the pair's producers run in lockstep), so opt-in
  g.pair = tune("fct_bd_pair", 0) == 1 && g.BN % 16 == 0;
  const std::size_t b_bytes = std::size_t(g.T * g.U * kBdKp / 32) * (g.pair ? g.BN / 2 : g.BN) * 128;
  const std::size_t fixed = b_bytes + 1024 + 1024;
  // column strips (each a separate pass down the image) until the dy-row
  // ring holds two tiles' rows and a strip's positions fit two 32-blocks
  const int force = tune("fct_bd_strips", 0);
  for (g.nstrip = force > 0 ? force : 1; g.nstrip <= 8; ++g.nstrip) {
    g.SW = (g.Wq + g.nstrip - 1) / g.nstrip;
    g.XP = g.SW + g.U - 1;  // ring positions x = ow - strip origin + U - 1
    g.TR = std::max(1, kBM / g.SW);
    g.PH = g.TR + g.T - 1;
    const std::size_t row_bytes = std::size_t(g.XP) * kBdKS * 4;
    int rr = int((220 * 1024 - std::min<std::size_t>(fixed, 220 * 1024)) / row_bytes);
    rr = std::min(rr, g.PH + (kHist - 2) * g.TR);
    rr = std::min(rr, tune("fct_bd_ring", rr));
    g.RR = std::max(rr, 1);
    g.smem = fixed + row_bytes * g.RR;
    if (force > 0 || (g.XP <= 64 && g.RR >= g.PH + g.TR)) break;
  }
  g.np = g.TR * g.SW;
  g.tps = (g.Hq + g.TR - 1) / g.TR;
  g.units = s.N * g.nstrip * g.tps;
  g.grid = g.pair ? 2 * std::min(sm_count() / 2, (g.units + 1) / 2) : std::min(sm_count(), g.units);
  (void)OH;
  return g;
}

}  // namespace

bool fct_bwdd_supports(const ConvShape& s) {
  if (s.sh != s.sw || (s.sh != 2 && s.sh != 4) || s.C > 4 || s.K > kBdKp || !tune("fct_bd", 1)) return false;
  const DGeo g = make_dgeo(s);
  const int tu = g.T * g.U;
  return (tu == 9 || tu == 4 || tu == 16) && g.nstrip <= 8 && g.XP <= 64 && g.BN <= 64 && g.nslots >= 2 &&
         g.RR >= g.PH + g.TR && g.smem <= 220 * 1024 && std::int64_t(s.N) * s.C * s.H * s.W < (1ll << 40);
}

cudaError_t fct_bwdd_run(const ConvShape& s, const float* dy, const float* w, float* dx, float alpha, float beta,
                         cudaStream_t st) {
  const DGeo g = make_dgeo(s);
  DParams p{};
  p.dy = dy; p.w = w; p.dx = dx; p.alpha = alpha; p.beta = beta;
  p.C = s.C; p.H = s.H; p.W = s.W; p.K = s.K; p.R = s.R; p.S = s.S; p.ph = s.ph; p.pw = s.pw; p.sh = s.sh;
  p.OH = s.OH(); p.OW = s.OW();
  p.T = g.T; p.U = g.U; p.Hq = g.Hq; p.Wq = g.Wq; p.TR = g.TR; p.np = g.np; p.tps = g.tps; p.SW = g.SW; p.nstrip = g.nstrip;
  p.units = g.units; p.BN = g.BN; p.AS = g.AS; p.nslots = g.nslots; p.RR = g.RR; p.XP = g.XP; p.PH = g.PH;
  p.OHW = std::int64_t(p.OH) * p.OW;
  p.KOHW = std::int64_t(s.K) * p.OHW;
  p.CHW = std::int64_t(s.C) * s.H * s.W;
  const int tu = g.T * g.U;
  void (*kern)(const DParams) = nullptr;
#define FCT_BD_PICK(P)                                                                                        \
  if (s.sh == 4) kern = tu == 9 ? fct_bwdd_kernel<4, 9, P> : tu == 4 ? fct_bwdd_kernel<4, 4, P> : fct_bwdd_kernel<4, 16, P>; \
  else kern = tu == 9 ? fct_bwdd_kernel<2, 9, P> : tu == 4 ? fct_bwdd_kernel<2, 4, P> : fct_bwdd_kernel<2, 16, P>;
  if (g.pair) {
    FCT_BD_PICK(true)
  } else {
    FCT_BD_PICK(false)
  }
#undef FCT_BD_PICK
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), int(g.smem));
  if (e != cudaSuccess) return e;
  trace_variant("fct bwdd units=%d grid=%d TR=%d np=%d strips=%d TU=%d BN=%d XP=%d ring=%d slots=%d pair=%d", g.units,
                g.grid, g.TR, g.np, g.nstrip, tu, g.BN, g.XP, g.RR, g.nslots, int(g.pair));
  if (!g.pair) return launch_pdl(kern, dim3(g.grid), dim3(kBdThreads), g.smem, st, p);
  count_launch();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g.grid);
  cfg.blockDim = dim3(kBdThreads);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = st;
  cudaLaunchAttribute cat[1];
  cat[0].id = cudaLaunchAttributeClusterDimension;
  cat[0].val.clusterDim.x = 2;
  cat[0].val.clusterDim.y = 1;
  cat[0].val.clusterDim.z = 1;
  cfg.attrs = cat;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_tiled_fct() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

struct B1Geo {
  int OH, OW, rows, QT, QG, G, cpg, BN, nblk, units, XW, CR, RS, RR, nslots, nds;
  std::size_t smem;
};

B1Geo make_b1geo(const ConvShape& s) {
  B1Geo g{};
  g.OH = s.OH();
  g.OW = s.OW();
  g.rows = s.C * s.R * s.S;
  g.BN = (s.K + 15) / 16 * 16;
  g.QT = g.BN <= 64 ? 3 : 2;
  g.QG = g.QT * kBM;
  // whole channels per group: CR * R * S <= QG x rows
  g.CR = std::max(1, std::min(s.C, g.QG / (s.R * s.S)));
  g.G = (s.C + g.CR - 1) / g.CR;
  g.cpg = std::max(1, sm_count() / g.G);
  g.nblk = (g.OW + 31) / 32;
  g.units = s.N * g.OH;
  // ring columns from w = -4: every tap column read, 16 B multiple, = 12 mod 32
  const int need = g.nblk * 32 - 1 + s.S - 1 + 4 - s.pw + 1;
  g.XW = (need + 3) / 4 * 4;
  while (g.XW % 32 != 12) g.XW += 4;
  // ring row stride: the box rounded up to 128 B (the TMA destination
  // alignment); the channel stride XW = 12 mod 32 spreads a warp's lanes
  g.RS = (g.CR * g.XW + 31) / 32 * 32;
  g.nslots = std::min(kMaxSlots, (512 - g.QT * g.BN) / (g.QT * 32));
  g.nds = std::min(kB1MaxDS, (96 * 1024) / (g.BN * 128));
  const std::size_t fixed = std::size_t(g.nds) * g.BN * 128 + 1024 + 512;
  const std::size_t row_bytes = std::size_t(g.RS) * 4;
  int rr = int((220 * 1024 - std::min<std::size_t>(fixed, 220 * 1024)) / row_bytes);
  rr = std::min(rr, s.R + (kHist - 2));
  // one 32-pixel block per output row: a shallow ring is faster (ResNet l2
  // 3x3 BF at 256 images 253 -> 216 us at R + 2 rows); two blocks per row
  // keep the deep ring (l1: 273 vs 286 us, scripts/r02_run100.sh)
  if (g.nblk == 1) rr = std::min(rr, s.R + 2);
  rr = std::min(rr, tune("fct_bf1_ring", rr));
  g.RR = std::max(rr, 1);
  g.smem = fixed + row_bytes * g.RR;
  return g;
}

}  // namespace

bool fct_bwdf1_supports(const ConvShape& s) {
  if (s.sh != 1 || s.sw != 1 || s.C <= 4 || s.K % 16 != 0 || s.K > 128 || !tune("fct_bf1", 1)) return false;
  const int OW = s.OW(), OH = s.OH();
  // TMA: 16 B aligned rows of x and dy, the x box starting at w = -4
  if (s.W % 4 != 0 || OW % 4 != 0 || (std::int64_t(OH) * OW) % 4 != 0 || s.pw > 4) return false;
  const B1Geo g = make_b1geo(s);
  return s.R * s.S <= g.QG && g.CR <= 256 && g.XW <= 256 && g.nslots >= 2 && g.nds >= 4 && g.RR >= s.R + 1 && g.smem <= 220 * 1024 &&
         std::int64_t(s.N) * s.K * OH * OW < (1ll << 31);
}

std::int64_t fct_bwdf1_workspace(const ConvShape& s) {
  const B1Geo g = make_b1geo(s);
  return (std::int64_t(g.G) * g.cpg * g.QG * s.K * 4 + 255) / 256 * 256;
}

cudaError_t fct_bwdf1_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha,
                          float beta, cudaStream_t st) {
  const B1Geo g = make_b1geo(s);
  CUtensorMap xmap, dmap;
  {
    const cuuint64_t dims[4] = {cuuint64_t(s.W), cuuint64_t(s.H), cuuint64_t(s.C), cuuint64_t(s.N)};
    const cuuint64_t strides[3] = {cuuint64_t(s.W) * 4, cuuint64_t(s.H) * s.W * 4, cuuint64_t(s.C) * s.H * s.W * 4};
    const cuuint32_t box[4] = {cuuint32_t(g.XW), 1, cuuint32_t(g.CR), 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    if (encode_tiled_fct()(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t dims[3] = {cuuint64_t(g.OW), cuuint64_t(g.OH), cuuint64_t(s.N) * s.K};
    const cuuint64_t strides[2] = {cuuint64_t(g.OW) * 4, cuuint64_t(g.OH) * g.OW * 4};
    const cuuint32_t box[3] = {32, 1, cuuint32_t(g.BN)};
    const cuuint32_t es[3] = {1, 1, 1};
    if (encode_tiled_fct()(&dmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(dy), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  B1Params p{};
  p.slices = static_cast<float*>(ws);
  p.C = s.C; p.H = s.H; p.W = s.W; p.K = s.K; p.R = s.R; p.S = s.S; p.ph = s.ph; p.pw = s.pw;
  p.OH = g.OH; p.OW = g.OW;
  p.rows = g.rows; p.BN = g.BN; p.nblk = g.nblk; p.units = g.units; p.RR = g.RR; p.XW = g.XW; p.RS = g.RS;
  p.CR = g.CR; p.QG = g.QG; p.cpg = g.cpg; p.nslots = g.nslots; p.nds = g.nds;
  void (*kern)(const CUtensorMap, const CUtensorMap, const B1Params) =
      g.QT == 3 ? fct_bwdf1_kernel<3> : fct_bwdf1_kernel<2>;
  cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(kern), int(g.smem));
  if (e != cudaSuccess) return e;
  trace_variant("fct bwdf1 units=%d groups=%d cpg=%d QT=%d BN=%d CR=%d XW=%d ring=%d slots=%d dslots=%d", g.units,
                g.G, g.cpg, g.QT, g.BN, g.CR, g.XW, g.RR, g.nslots, g.nds);
  e = launch_pdl(kern, dim3(g.G * g.cpg), dim3(kB1Threads), g.smem, st, xmap, dmap, p);
  if (e != cudaSuccess) return e;
  B1Final f{p.slices, dw, alpha, beta, g.rows, s.K, g.QG, g.cpg, g.CR, s.R, s.S, FastDiv(std::uint32_t(s.K))};
  const long long n = (long long)g.rows * s.K;
  return launch_pdl(fct_bwdf1_finalize_kernel, dim3(int(std::min<long long>((n + 255) / 256, 4 * sm_count()))),
                    dim3(256), 0, st, f);
}

}  // namespace ucudnn
