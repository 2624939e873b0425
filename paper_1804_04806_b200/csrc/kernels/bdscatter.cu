// UCUDNN_ALGO_IMPLICIT_GATHER_GEMM, BackwardData for few-channel strided
// layers (AlexNet / ResNet conv1): GEMM + col2im fused through shared memory.
//
//   dx[n][c][oh*sh-ph+r][ow*sw-pw+s] += alpha * sum_k W[k][c][r][s] * dy[n][k][oh][ow]
//   (reference_conv.hpp:105-135: the scatter adjoint; beta applied up front)
//
// The stride-phase implicit GEMM (precomp.cu) turns conv1's BackwardData
// into a GEMM whose output width is the handful of phase-channels (ResNet
// conv1: 4 phases x 3 channels = 12 columns) while every output pixel
// re-reads 64 dy channels x 16 taps -- tiny MMAs fed by a huge A operand.
// Here the roles follow the adjoint directly: for a 4 x 32 block of dy
// positions (128 MMA rows) and every filter tap (c, r, s) (the MMA columns,
// <= 256 per tile),
//
//   D[pixel][(c, r, s)] = sum_k dy[k][pixel] * W[k][(c, r, s)]   (tcgen05, K = dy channels)
//
// and the epilogue scatter-adds D into a shared-memory dx patch covering
// the block's receptive field ((4-1)*sh + R rows x (32-1)*sw + S columns x
// C), which is then reduced into dx with coalesced fp32 REDs (neighbouring
// blocks' patches overlap by R - sh rows / S - sw columns). dy is read once
// (cp.async gathers, lane = dy column), W stays resident in shared memory,
// and no workspace is needed.
//
// Persistent, one CTA per SM, 288 threads: warps 0-3 epilogue (one per
// TMEM lane quadrant), warp 4 TMEM owner + MMA issuer, warps 5-8 producers
// (one dy row of the block each).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "bdscatter.h"
#include "conv_common.h"
#include "launch.h"
#include "sm100.cuh"

namespace ucudnn {
using namespace sm100;

namespace {

constexpr int kBM = 128, kTW = 32, kTH = 4;
constexpr int kMaxBN = 256;
constexpr int kEpi = 4, kProd = 4;
constexpr int kThreads = (kEpi + 1 + kProd) * 32;
constexpr int kStages = 4;              // A ring: one 32-channel chunk (16 KB) per stage
constexpr int kSmemBudget = 220 * 1024;

struct SGeo {
  int N, C, H, W, K, R, S, ph, pw, sh, sw, OH, OW;
  int CRS, BN, n_tiles, kchunks;
  int th, tw, tiles;  // dy blocks per image row / column, blocks in total
  int PH, PW;         // patch rows / columns
  int PWs, PWp;       // patch columns per stride phase, row pitch (sw * PWs)
  std::size_t b_bytes, patch_bytes, smem;
};

int round_up(int a, int b) { return (a + b - 1) / b * b; }

SGeo make_sgeo(const ConvShape& s) {
  SGeo g{};
  g.N = s.N; g.C = s.C; g.H = s.H; g.W = s.W; g.K = s.K; g.R = s.R; g.S = s.S;
  g.ph = s.ph; g.pw = s.pw; g.sh = s.sh; g.sw = s.sw; g.OH = s.OH(); g.OW = s.OW();
  g.CRS = s.C * s.R * s.S;
  g.n_tiles = (g.CRS + kMaxBN - 1) / kMaxBN;
  g.BN = round_up((g.CRS + g.n_tiles - 1) / g.n_tiles, 16);
  g.kchunks = (s.K + 31) / 32;
  g.th = (g.OH + kTH - 1) / kTH;
  g.tw = (g.OW + kTW - 1) / kTW;
  g.tiles = s.N * g.th * g.tw;
  g.PH = (kTH - 1) * s.sh + s.R;
  g.PW = (kTW - 1) * s.sw + s.S;
  // phase-major patch rows: column j at (j % sw) * PWs + j / sw, so a warp's
  // 32 dy columns touch 32 consecutive words; PWs = 32 / sw (mod 32) keeps
  // the write-out's phase-interleaved reads on distinct banks
  g.PWs = (g.PW + s.sw - 1) / s.sw;
  if (s.sw > 1 && 32 % s.sw == 0)
    while (g.PWs % 32 != 32 / s.sw) ++g.PWs;
  g.PWp = g.PWs * s.sw;
  g.b_bytes = std::size_t(g.kchunks) * ((std::size_t(g.BN) * 128 + 1023) / 1024 * 1024);
  g.patch_bytes = std::size_t(g.C) * g.PH * g.PWp * 4;
  g.smem = 1024 + g.b_bytes + std::size_t(kStages) * kBM * 128 + (g.patch_bytes + 15) / 16 * 16 +
           std::size_t(g.BN) * 8 + std::size_t(g.BN + 2) * 4 + 256;
  return g;
}

struct SParams {
  const float* dy;
  const float* w;
  float* dx;
  float alpha;
  int C, H, W, K, R, S, ph, pw, sh, sw, OH, OW, CRS;
  int BN, n_tiles, kchunks, th, tw, tiles, PH, PW, PWs, PWp;
  std::uint32_t b_bytes, patch_floats;
  FastDiv fd_tpi, fd_tw, fd_RS, fd_S, fd_sw;
  int dbg;  // diagnostic (UCUDNN_TUNE=bds_dbg): bit 0 skip the scatter, bit 1 skip the write-out  // blocks per image, blocks per row, R*S, S, sw
};

__device__ __forceinline__ void cp_async4a(std::uint32_t dst, std::uint64_t src, std::uint32_t src_size) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_size) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(std::uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// one TMEM column for the warp's 32 lanes (no wait)
__device__ __forceinline__ void tmem_ld1(std::uint32_t taddr, float& v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=f"(v) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kEpi * 32) : "memory"); }
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
    if (ns < 1024) ns <<= 1;
  }
}

// SW128 K-major byte offset of element (row, k) of a 32-wide chunk
__device__ __forceinline__ std::uint32_t sw128(int row, int k) {
  return std::uint32_t(row) * 128 + ((std::uint32_t(k >> 2) ^ (row & 7)) << 4) + (k & 3) * 4;
}

__global__ void __launch_bounds__(kThreads, 1) bds_kernel(const SParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-aligned base, derived from the shared array so the compiler keeps
  // shared-space (LDS / STS) accesses
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* bsm = smem;                 // [kchunk][BN rows][128 B]
  unsigned char* asm_ = smem + p.b_bytes;    // [stage][128 rows][128 B]
  float* patch = reinterpret_cast<float*>(asm_ + kStages * kBM * 128);
  int2* sched = reinterpret_cast<int2*>(patch + (p.patch_floats + 3) / 4 * 4);  // (TMEM column, patch offset)
  int* batch = reinterpret_cast<int*>(sched + p.BN);  // batch starts (| 1 << 30: sync first), terminated by BN
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(batch + (p.BN + 2) / 2 * 2);
  std::uint64_t* empty = full + kStages;
  std::uint64_t* tfull = empty + kStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t b_chunk = (std::uint32_t(p.BN) * 128 + 1023) & ~1023u;

  // this CTA's column tile stays fixed: W's slice is loaded once
  const int groups = gridDim.x / p.n_tiles;
  const int nt = blockIdx.x % p.n_tiles, g0 = blockIdx.x / p.n_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], kProd * 32);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpi * 32);
    }
    mbar_fence_init();
  }
  if (warp == kEpi) tmem_alloc<512>(tmem_slot);
  // W[k][(c, r, s)] -> B rows (c, r, s), 32 dy channels per chunk (zero past K / CRS)
  for (int row = warp; row < p.kchunks * p.BN; row += kThreads / 32) {
    const int kc = row / p.BN, j = row - kc * p.BN;
    const int crs = nt * p.BN + j, k = kc * 32 + lane;
    const float v = (crs < p.CRS && k < p.K) ? __ldg(p.w + std::int64_t(k) * p.CRS + crs) : 0.f;
    *reinterpret_cast<float*>(bsm + kc * b_chunk + sw128(j, lane)) = v;
  }
  // Scatter schedule for this column tile, in (r, s-batch, c) order: a batch
  // is every channel of sw consecutive taps s of one filter row r -- its
  // read-add-writes touch distinct words for every lane, so they issue back
  // to back; consecutive batches of one r only overlap across lanes of the
  // same warp (program order), and the four quadrant warps sync before each
  // new r (quadrants collide only through different r).
  if (threadIdx.x == 0) {
    int ne = 0, nb = 0;
    for (int r = 0; r < p.R; ++r) {
      bool first_r = true;
      for (int s0 = 0; s0 < p.S; s0 += p.sw) {
        int start = ne;
        for (int c = 0; c < p.C; ++c)
          for (int s = s0; s < min(p.S, s0 + p.sw); ++s) {
            const int j = (c * p.R + r) * p.S + s - nt * p.BN;
            if (j < 0 || j >= p.BN) continue;
            if (ne - start == 16) {  // batch cap (registers)
              batch[nb++] = start;
              start = ne;
            }
            sched[ne++] = make_int2(j, (c * p.PH + r) * p.PWp + (s % p.sw) * p.PWs + s / p.sw);
          }
        if (ne > start) {
          batch[nb++] = start | (first_r && nb > 0 ? (1 << 30) : 0);
          first_r = false;
        }
      }
    }
    batch[nb] = ne | (1 << 29);  // end
  }
  for (std::uint32_t i = threadIdx.x; i < p.patch_floats; i += kThreads) patch[i] = 0.f;
  fence_async_smem();  // B was written through the generic proxy
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = tmem_base_uniform(tmem_slot);

  if (warp > kEpi) {
    // ------------------------------------------------ dy gather: row ty of the block
    const int ty = warp - kEpi - 1;
    const std::uint32_t abase = smem_u32(asm_);
    int st = 0;
    std::uint32_t ph = 0;
    for (int t = g0; t < p.tiles; t += groups) {
      std::uint32_t n, rem, bi, bj;
      p.fd_tpi.divmod(std::uint32_t(t), n, rem);
      p.fd_tw.divmod(rem, bi, bj);
      const int oh = int(bi) * kTH + ty, ow = int(bj) * kTW + lane;
      const bool ok = oh < p.OH && ow < p.OW;
      const std::uint64_t src0 = reinterpret_cast<std::uint64_t>(
          p.dy + (std::int64_t(n) * p.K * p.OH + (ok ? oh : 0)) * p.OW + (ok ? ow : 0));
      const std::uint64_t kstride = std::uint64_t(p.OH) * p.OW * 4;
      const int row = ty * kTW + lane;
      for (int kc = 0; kc < p.kchunks; ++kc) {
        mbar_wait(&empty[st], ph ^ 1);
        const std::uint32_t dst = abase + st * (kBM * 128);
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          const int kk = kc * 32 + k;
          cp_async4a(dst + sw128(row, k), src0 + std::uint64_t(kk < p.K ? kk : 0) * kstride,
                     (ok && kk < p.K) ? 4u : 0u);
        }
        cp_async_arrive(&full[st]);
        if (++st == kStages) {
          st = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == kEpi) {
    // ------------------------------------------------ MMA issuer
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN);
    const std::uint32_t abase = smem_u32(asm_), bbase = smem_u32(bsm);
    int it = 0, tl = 0;
    for (int t = g0; t < p.tiles; t += groups, ++tl) {
      const int acc = tl & 1;
      mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
      tc_fence_after();
      const std::uint32_t dtm = tmem + std::uint32_t(acc * kMaxBN);
      for (int kc = 0; kc < p.kchunks; ++kc, ++it) {
        const int st = it % kStages;
        mbar_wait(&full[st], (it / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          fence_async_smem();  // the dy chunk arrived through cp.async (generic proxy)
          const std::uint32_t sa = abase + st * (kBM * 128), sb = bbase + kc * b_chunk;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            mma_tf32(dtm, umma_desc_sw128(sa + q * 32), umma_desc_sw128(sb + q * 32), idesc,
                     (kc != 0 || q != 0) ? 1u : 0u);
          mma_commit(&empty[st]);
          if (kc + 1 == p.kchunks) mma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ scatter into the patch, then RED into dx
    // One warp per TMEM lane quadrant = dy row ty of the block; all four walk
    // the columns in the same order. Within one column (tap) the 128 pixels
    // hit 128 distinct patch words, and two quadrants can only collide on
    // different taps of the same (c, r) row group... of different r -- so
    // plain read-add-write is race-free if the quadrants sync at every new
    // (c, r) group (fp32 shared atomics would be CAS loops here).
    const int qd = warp;
    int tl = 0;
    for (int t = g0; t < p.tiles; t += groups, ++tl) {
      std::uint32_t n, rem, bi, bj;
      p.fd_tpi.divmod(std::uint32_t(t), n, rem);
      p.fd_tw.divmod(rem, bi, bj);
      const int acc = tl & 1;
      mbar_wait_backoff(&tfull[acc], (tl >> 1) & 1);
      tc_fence_after();
      const bool ok = int(bi) * kTH + qd < p.OH && int(bj) * kTW + lane < p.OW;
      float* pb = patch + qd * p.sh * p.PWp + lane;
      const std::uint32_t tbase = tmem + (std::uint32_t(qd * 32) << 16) + std::uint32_t(acc * kMaxBN);
      for (int bq = 0; !(p.dbg & 1); ++bq) {
        const int b0 = batch[bq];
        if (b0 & (1 << 29)) break;
        const int b1 = batch[bq + 1] & ((1 << 29) - 1);
        const int e0 = b0 & ((1 << 29) - 1), cnt = b1 - e0;
        if (b0 & (1 << 30)) epi_sync();
        float v[16];
        int off[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (e < cnt) {
            const int2 en = sched[e0 + e];
            tmem_ld1(tbase + std::uint32_t(en.x), v[e]);
            off[e] = en.y;
          }
        tmem_wait_ld();
        if (ok) {
          float o[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (e < cnt) o[e] = pb[off[e]];
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (e < cnt) pb[off[e]] = o[e] + p.alpha * v[e];
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      epi_sync();
      // patch (c, i, j) -> dx[n][c][bi*4*sh - ph + i][bj*32*sw - pw + j]; re-zero it
      const int h0 = int(bi) * kTH * p.sh - p.ph, w0 = int(bj) * kTW * p.sw - p.pw;
      float* dxn = p.dx + std::int64_t(n) * p.C * p.H * p.W;
      const int rows = p.C * p.PH;
      for (int rr = warp; rr < (p.dbg & 2 ? 0 : rows); rr += kEpi) {
        const int c = rr / p.PH, i = rr - c * p.PH, h = h0 + i;
        float* prow = patch + rr * p.PWp;
        const bool hin = unsigned(h) < unsigned(p.H);
        float* drow = dxn + (std::int64_t(c) * p.H + h) * p.W;
#pragma unroll 4
        for (int j = lane; j < p.PW; j += 32) {
          std::uint32_t jq, jp;
          p.fd_sw.divmod(std::uint32_t(j), jq, jp);
          float* src = prow + int(jp) * p.PWs + int(jq);
          const float v = *src;
          *src = 0.f;
          const int w = w0 + j;
          if (hin && unsigned(w) < unsigned(p.W) && v != 0.f) red_add(drow + w, v);
        }
      }
      epi_sync();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kEpi) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

__global__ void __launch_bounds__(256) scale_kernel(float* x, std::int64_t n, float beta) {
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < n;
       i += std::int64_t(gridDim.x) * blockDim.x)
    x[i] *= beta;
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

bool bds_supports(const ConvShape& s) {
  // Experimental, off unless UCUDNN_TUNE=bds=1: exact, but the scatter
  // epilogue is the bottleneck (AlexNet conv1 BD at 256 images: pipeline
  // alone 380 us, + write-out 1.05 ms, + scatter 3.2 ms; PRECOMP 409 us).
  if (!tune("bds", 0)) return false;
  if (s.sh == 1 && s.sw == 1) return false;  // stride 1: the implicit GEMMs have no phase blow-up
  const SGeo g = make_sgeo(s);
  return s.K <= 128 && g.CRS <= 4 * kMaxBN && g.smem <= std::size_t(kSmemBudget) && g.tiles > 0 &&
         std::int64_t(s.N) * s.C * s.H * s.W < (std::int64_t(1) << 40);
}

std::int64_t bds_workspace(const ConvShape&) { return 0; }

cudaError_t bds_run(const ConvShape& s, const float* dy, const float* w, float* dx, float alpha, float beta,
                    cudaStream_t st) {
  const SGeo g = make_sgeo(s);
  cudaError_t e;
  if (beta == 0.f) {
    e = cudaMemsetAsync(dx, 0, std::size_t(s.x_elems()) * 4, st);
  } else if (beta != 1.f) {
    e = launch_pdl(scale_kernel, dim3(4 * sm_count()), dim3(256), 0, st, dx, s.x_elems(), beta);
  } else {
    e = cudaSuccess;
  }
  if (e != cudaSuccess) return e;
  SParams p{};
  p.dy = dy;
  p.w = w;
  p.dx = dx;
  p.alpha = alpha;
  p.C = g.C; p.H = g.H; p.W = g.W; p.K = g.K; p.R = g.R; p.S = g.S;
  p.ph = g.ph; p.pw = g.pw; p.sh = g.sh; p.sw = g.sw; p.OH = g.OH; p.OW = g.OW; p.CRS = g.CRS;
  p.BN = g.BN; p.n_tiles = g.n_tiles; p.kchunks = g.kchunks;
  p.th = g.th; p.tw = g.tw; p.tiles = g.tiles; p.PH = g.PH; p.PW = g.PW; p.PWs = g.PWs; p.PWp = g.PWp;
  p.b_bytes = std::uint32_t(g.b_bytes);
  p.patch_floats = std::uint32_t(g.C * g.PH * g.PWp);
  p.fd_tpi = FastDiv(std::uint32_t(g.th * g.tw));
  p.fd_tw = FastDiv(std::uint32_t(g.tw));
  p.fd_RS = FastDiv(std::uint32_t(g.R * g.S));
  p.fd_S = FastDiv(std::uint32_t(g.S));
  p.fd_sw = FastDiv(std::uint32_t(g.sw));
  p.dbg = tune("bds_dbg", 0);
  e = set_smem_attr(reinterpret_cast<const void*>(bds_kernel), kSmemBudget + 4096);
  if (e != cudaSuccess) return e;
  const int sms = sm_count();
  const int grid = std::max(1, sms / g.n_tiles) * g.n_tiles;
  return launch_pdl(bds_kernel, dim3(grid), dim3(kThreads), g.smem, st, p);
}

}  // namespace ucudnn
