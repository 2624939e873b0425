// UCUDNN_ALGO_GEMM: explicit-layout convolution -- pack kernels lay the
// operands out as pre-tiled, K-major UMMA blocks in the workspace, then one
// persistent tcgen05 GEMM streams them with 1-D bulk copies.
//
//   Forward        A = im2col(x)   [pixels  x (c,r,s)]   B = w        [K x (c,r,s)]
//                  -> NCHW y epilogue (alpha/beta)
//   BackwardData   A = dy          [pixels  x K]         B = w^T      [(c,r,s) x K]
//                  -> dcol [pixels x (c,r,s)] in the workspace, then a col2im
//                     gather sums each dx element's taps (any stride, any C)
//   BackwardFilter A = im2col(x)^T [(c,r,s) x pixels]    B = dy       [K x pixels]
//                  -> split-K over pixels, fp32 reductions into dw (beta pre-applied)
//
// Every tf32 operand is K-major: tcgen05 kind::tf32 with MN-major (transposed)
// descriptors executes as a no-op on this part (probe in DESIGN.md), so the
// pack kernels do the transposition (through shared memory, keeping both the
// gather and the block write coalesced). The workspace grows linearly with the
// micro-batch -- e.g. 4.45 MiB per sample for AlexNet conv2's im2col -- which is
// why this algorithm is the textbook case for micro-batching.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "conv_common.h"
#include "gemm.h"
#include "sm100.cuh"

namespace ucudnn {
using namespace sm100;

namespace {

constexpr int kBM = 128;
constexpr int kStages = 4;
constexpr int kThreads = 256;
constexpr int kMaxBN = 256;

// ------------------------------------------------------------------ packing
enum PackKind : int {
  kIm2colPix = 0,  // row = output pixel (n,oh,ow), col = (c,r,s)       -> x
  kIm2colCrs = 1,  // row = (c,r,s), col = output pixel                 -> x
  kRowMajor = 2,   // row, col -> p[row * ld + col]
  kColMajor = 3,   // row, col -> p[col * ld + row]
  kDyKPix = 4,     // row = k, col = output pixel (n,p)                 -> dy
  kDyPixK = 5,     // row = output pixel (n,p), col = k                 -> dy
};

struct PackParams {
  const float* src;
  float* dst;
  int kind, rows, cols, ld;
  int ROWS;          // rows per tile block (128 or BN)
  int ksteps;        // 32-wide column blocks
  int C, H, W, K, S, ph, pw, sh, sw, OW, P;
  FastDiv fd_P, fd_OW, fd_RS, fd_S, fd_ks;
};

// Every packed element is src[ro(row) + co(col)] when (rh + ch) < Hlim and
// (rw + cw) < Wlim (unsigned), else 0: rows and columns decode separately,
// once per block, so the gather loop is two adds, two compares and a load.
struct Dec {
  int off, h, w;
};
constexpr int kBad = 1 << 20;

__device__ __forceinline__ Dec decode_pixel(const PackParams& p, int pix, bool im2col) {
  if (pix >= (p.kind == kIm2colPix || p.kind == kDyPixK ? p.rows : p.cols)) return Dec{0, kBad, 0};
  std::uint32_t n, pp, oh, ow;
  p.fd_P.divmod(std::uint32_t(pix), n, pp);
  if (!im2col) return Dec{int(n) * p.K * p.P + int(pp), 0, 0};
  p.fd_OW.divmod(pp, oh, ow);
  const int h = int(oh) * p.sh - p.ph, w = int(ow) * p.sw - p.pw;
  return Dec{int(n) * p.C * p.H * p.W + h * p.W + w, h, w};
}
__device__ __forceinline__ Dec decode_crs(const PackParams& p, int crs, int limit) {
  if (crs >= limit) return Dec{0, kBad, 0};
  std::uint32_t c, rs, r, s;
  p.fd_RS.divmod(std::uint32_t(crs), c, rs);
  p.fd_S.divmod(rs, r, s);
  return Dec{int(c) * p.H * p.W + int(r) * p.W + int(s), int(r), int(s)};
}
__device__ __forceinline__ Dec decode_row(const PackParams& p, int row) {
  switch (p.kind) {
    case kIm2colPix: return decode_pixel(p, row, true);
    case kIm2colCrs: return decode_crs(p, row, p.rows);
    case kRowMajor: return row < p.rows ? Dec{row * p.ld, 0, 0} : Dec{0, kBad, 0};
    case kColMajor: return row < p.rows ? Dec{row, 0, 0} : Dec{0, kBad, 0};
    case kDyKPix: return row < p.rows ? Dec{row * p.P, 0, 0} : Dec{0, kBad, 0};
    default: return decode_pixel(p, row, false);  // kDyPixK
  }
}
__device__ __forceinline__ Dec decode_col(const PackParams& p, int col) {
  switch (p.kind) {
    case kIm2colPix: return decode_crs(p, col, p.cols);
    case kIm2colCrs: return decode_pixel(p, col, true);
    case kRowMajor: return col < p.cols ? Dec{col, 0, 0} : Dec{0, kBad, 0};
    case kColMajor: return col < p.cols ? Dec{col * p.ld, 0, 0} : Dec{0, kBad, 0};
    case kDyKPix: return decode_pixel(p, col, false);
    default: return col < p.cols ? Dec{col * p.P, 0, 0} : Dec{0, kBad, 0};  // kDyPixK
  }
}

// One block per (row tile, 32-column step): gather with lanes along the
// source's contiguous direction into smem, then write the 8 x ROWS x 16 B
// canonical block contiguously.
__global__ void __launch_bounds__(256) pack_kernel(const PackParams p) {
  __shared__ float tile[32][kMaxBN + 1];
  __shared__ Dec rdec[kMaxBN], cdec[32];
  std::uint32_t rt, ks;
  p.fd_ks.divmod(blockIdx.x, rt, ks);
  const int row0 = int(rt) * p.ROWS, col0 = int(ks) * 32;
  for (int i = threadIdx.x; i < p.ROWS; i += blockDim.x) rdec[i] = decode_row(p, row0 + i);
  if (threadIdx.x < 32) cdec[threadIdx.x] = decode_col(p, col0 + threadIdx.x);
  __syncthreads();
  const bool im2col = p.kind == kIm2colPix || p.kind == kIm2colCrs;
  const unsigned hl = im2col ? unsigned(p.H) : 1u, wl = im2col ? unsigned(p.W) : 1u;
  const bool col_fast = p.kind == kIm2colCrs || p.kind == kRowMajor || p.kind == kDyKPix;
  for (int idx = threadIdx.x; idx < p.ROWS * 32; idx += blockDim.x) {
    int r, c;
    if (col_fast) {
      c = idx & 31;
      r = idx >> 5;
    } else {
      r = idx % p.ROWS;
      c = idx / p.ROWS;
    }
    const Dec a = rdec[r], b = cdec[c];
    tile[c][r] = (unsigned(a.h + b.h) < hl && unsigned(a.w + b.w) < wl) ? __ldg(p.src + a.off + b.off) : 0.f;
  }
  __syncthreads();
  float4* out = reinterpret_cast<float4*>(p.dst) + std::size_t(blockIdx.x) * (p.ROWS * 8);
  for (int u = threadIdx.x; u < p.ROWS * 8; u += blockDim.x) {
    const int r = u % p.ROWS, g = u / p.ROWS;
    out[u] = make_float4(tile[4 * g][r], tile[4 * g + 1][r], tile[4 * g + 2][r], tile[4 * g + 3][r]);
  }
}

// ------------------------------------------------------------------ GEMM
enum Epilogue : int { kEpiNchw = 0, kEpiRowMajor = 1, kEpiAtomicT = 2, kEpiColMajor = 3 };

struct GemmParams {
  const float* a;  // [m_tile][kstep] blocks of 128 x 32
  const float* b;  // [n_tile][kstep] blocks of BN x 32
  float* out;
  float alpha, beta;
  int m_tiles, n_tiles, ksteps, BN, splits, steps_per_unit;
  int epi, M, Nc, P, ld;
  FastDiv fd_P;
  int batch;                            // independent GEMMs (Winograd points)
  std::int64_t a_bs, b_bs, o_bs;        // their element strides
};

__global__ void __launch_bounds__(kThreads, 1) tiled_gemm_kernel(const GemmParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint32_t a_bytes = kBM * 128, b_bytes = std::uint32_t(p.BN) * 128;
  const std::uint32_t stage_bytes = a_bytes + ((b_bytes + 127) & ~127u);
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kStages * stage_bytes);
  std::uint64_t* empty = full + kStages;
  std::uint64_t* tfull = empty + kStages;
  std::uint64_t* tempty = tfull + 2;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(tempty + 2);
  if (threadIdx.x == 0) {
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
  const int tiles = p.m_tiles * p.n_tiles, per_batch = tiles * p.splits, units = per_batch * p.batch;

  if (warp == 0 || warp == 2 || warp == 3) {
    // up to three producer threads, stage s owned by thread s % 3 (one
    // thread's TMA issue stream keeps only about one stage in flight:
    // scripts/tma_probe.cu). Fixed ownership keeps every stage's parity
    // waits in order, so no producer can run two rounds ahead on a stage.
    const int pq = warp == 0 ? 0 : warp - 1;
    const int nprod = kStages < 3 ? kStages : 3;
    if (lane == 0) {
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int bi = u / per_batch, ur = u - bi * per_batch;
        const int tile = ur % tiles, split = ur / tiles;
        const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
        const int k0 = split * p.steps_per_unit, k1 = min(p.ksteps, k0 + p.steps_per_unit);
        const float* ab = p.a + bi * p.a_bs + (std::size_t(mt) * p.ksteps) * (a_bytes / 4);
        const float* bb = p.b + bi * p.b_bs + (std::size_t(nt) * p.ksteps) * (b_bytes / 4);
        for (int k = k0; k < k1; ++k, ++it) {
          if ((it % kStages) % nprod != pq) continue;
          const int s = it % kStages;
          mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          unsigned char* sa = smem + s * stage_bytes;
          mbar_expect_tx(&full[s], a_bytes + b_bytes);
          bulk_g2s(sa, ab + std::size_t(k) * (a_bytes / 4), a_bytes, &full[s]);
          bulk_g2s(sa + a_bytes, bb + std::size_t(k) * (b_bytes / 4), b_bytes, &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    const std::uint32_t idesc = idesc_tf32(kBM, p.BN);
    const std::uint32_t sbase = smem_u32(smem), lbo_b = std::uint32_t(p.BN) * 16;
    int it = 0, tl = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
      const int split = (u % per_batch) / tiles;
      const int k0 = split * p.steps_per_unit, k1 = min(p.ksteps, k0 + p.steps_per_unit);
      const int acc = tl & 1;
      mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
      tc_fence_after();
      const std::uint32_t dtm = tmem + std::uint32_t(acc * kMaxBN);
      for (int k = k0; k < k1; ++k, ++it) {
        const int s = it % kStages;
        mbar_wait(&full[s], (it / kStages) & 1);
        tc_fence_after();
        if (lane == 0) {
          const std::uint32_t sa = sbase + s * stage_bytes, sb = sa + a_bytes;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            mma_tf32(dtm, umma_desc(sa + 2 * q * (kBM * 16), kBM * 16, 128), umma_desc(sb + 2 * q * lbo_b, lbo_b, 128),
                     idesc, (k != k0 || q != 0) ? 1u : 0u);
          mma_commit(&empty[s]);
          if (k == k1 - 1) mma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
      if (k1 <= k0 && lane == 0) mma_commit(&tfull[acc]);
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    int tl = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++tl) {
      const int bi = u / per_batch, ur = u - bi * per_batch;
      const int tile = ur % tiles, split = ur / tiles;
      const int mt = tile % p.m_tiles, nt = tile / p.m_tiles;
      float* const out = p.out + bi * p.o_bs;
      const int k0 = split * p.steps_per_unit, k1 = min(p.ksteps, k0 + p.steps_per_unit);
      const int acc = tl & 1;
      mbar_wait(&tfull[acc], (tl >> 1) & 1);
      tc_fence_after();
      const int row = mt * kBM + ew * 32 + lane;
      const bool ok = row < p.M && k1 > k0;
      std::int64_t obase = 0;
      if (ok && p.epi == kEpiNchw) {
        std::uint32_t n, pix;
        p.fd_P.divmod(std::uint32_t(row), n, pix);
        obase = std::int64_t(n) * p.Nc * p.P + pix;
      }
      const std::uint32_t tbase = tmem + (std::uint32_t(ew * 32) << 16) + std::uint32_t(acc * kMaxBN);
      for (int c0 = 0; c0 < p.BN; c0 += 32) {
        float v[32];
        tmem_ld32(tbase + std::uint32_t(c0), v);
        if (!ok) continue;
        const int col0 = nt * p.BN + c0;
        if (p.epi == kEpiRowMajor && col0 + 32 <= p.Nc && c0 + 32 <= p.BN && (p.ld & 3) == 0) {
          float4* dst = reinterpret_cast<float4*>(out + std::int64_t(row) * p.ld + col0);
#pragma unroll
          for (int j = 0; j < 8; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          continue;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = col0 + j;
          if (c0 + j >= p.BN || col >= p.Nc) break;
          if (p.epi == kEpiNchw) {
            float* dst = out + obase + std::int64_t(col) * p.P;
            const float val = p.alpha * v[j];
            *dst = p.beta == 0.f ? val : val + p.beta * *dst;
          } else if (p.epi == kEpiRowMajor) {
            out[std::int64_t(row) * p.ld + col] = v[j];
          } else if (p.epi == kEpiColMajor) {
            out[std::int64_t(col) * p.ld + row] = v[j];
          } else {
            red_add(out + std::int64_t(col) * p.ld + row, p.alpha * v[j]);
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

// dx[n,c,h,w] = alpha * sum over taps (r,s) with (h+ph-r) = oh*sh, (w+pw-s) =
// ow*sw in range of dcol[(n,oh,ow)][(c,r,s)] + beta * dx: the gather form of
// the reference's scatter adjoint (reference_conv.hpp:105-135).
__global__ void col2im_kernel(const float* __restrict__ dcol, float* __restrict__ dx, int N, int C, int H, int W,
                              int R, int S, int ph, int pw, int sh, int sw, int OH, int OW, float alpha, float beta) {
  const std::int64_t total = std::int64_t(N) * C * H * W;
  const int CRS = C * R * S;
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < total;
       i += std::int64_t(gridDim.x) * blockDim.x) {
    const int w = int(i % W);
    std::int64_t t = i / W;
    const int h = int(t % H);
    t /= H;
    const int c = int(t % C);
    const int n = int(t / C);
    float acc = 0.f;
    const int th = h + ph, tw = w + pw;
    for (int r = th % sh; r < R; r += sh) {
      const int oh = (th - r) / sh;
      if (th - r < 0) break;
      if (oh >= OH) continue;
      for (int s = tw % sw; s < S; s += sw) {
        const int ow = (tw - s) / sw;
        if (tw - s < 0) break;
        if (ow >= OW) continue;
        acc += dcol[(std::int64_t(n) * OH * OW + std::int64_t(oh) * OW + ow) * CRS + (c * R + r) * S + s];
      }
    }
    dx[i] = beta == 0.f ? alpha * acc : alpha * acc + beta * dx[i];
  }
}

__global__ void scale_kernel(float* p, std::int64_t n, float beta) {
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < n;
       i += std::int64_t(gridDim.x) * blockDim.x)
    p[i] = beta == 0.f ? 0.f : p[i] * beta;
}

int sms() {
  static int v = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  return v;
}
int cdiv(std::int64_t a, std::int64_t b) { return int((a + b - 1) / b); }
std::size_t a256(std::size_t b) { return (b + 255) / 256 * 256; }
int pick_bn(int n) {
  int tiles = (n + 255) / 256;
  return ((n + tiles - 1) / tiles + 15) / 16 * 16;
}

// GEMM problem: rows M (A tiles of 128), cols Nc (B tiles of BN), reduction Kr.
struct Problem {
  int M, Nc, Kr, BN, m_tiles, n_tiles, ksteps;
  std::size_t a_bytes() const { return std::size_t(m_tiles) * ksteps * kBM * 128; }
  std::size_t b_bytes() const { return std::size_t(n_tiles) * ksteps * BN * 128; }
};
Problem make_problem(int M, int Nc, int Kr) {
  Problem q{M, Nc, Kr, pick_bn(Nc), 0, 0, 0};
  q.m_tiles = cdiv(M, kBM);
  q.n_tiles = cdiv(Nc, q.BN);
  q.ksteps = cdiv(Kr, 32);
  return q;
}

Problem problem_of(int op, const ConvShape& s) {
  const int CRS = s.C * s.R * s.S, P = s.OH() * s.OW();
  if (op == kFwd) return make_problem(s.N * P, s.K, CRS);
  if (op == kBwdData) return make_problem(s.N * P, CRS, s.K);
  return make_problem(CRS, s.K, s.N * P);
}

std::size_t workspace_of(int op, const ConvShape& s) {
  Problem q = problem_of(op, s);
  std::size_t ws = a256(q.a_bytes()) + a256(q.b_bytes());
  if (op == kBwdData) ws += a256(std::size_t(s.N) * s.OH() * s.OW() * s.C * s.R * s.S * 4);
  return ws;
}

PackParams pack_params(const ConvShape& s, int kind, const float* src, float* dst, int rows, int cols, int ld,
                       int ROWS) {
  PackParams p{};
  p.src = src;
  p.dst = dst;
  p.kind = kind;
  p.rows = rows;
  p.cols = cols;
  p.ld = ld;
  p.ROWS = ROWS;
  p.ksteps = cdiv(cols, 32);
  p.C = s.C; p.H = s.H; p.W = s.W; p.K = s.K; p.S = s.S;
  p.ph = s.ph; p.pw = s.pw; p.sh = s.sh; p.sw = s.sw; p.OW = s.OW(); p.P = s.OH() * s.OW();
  p.fd_P = FastDiv(std::uint32_t(p.P));
  p.fd_OW = FastDiv(std::uint32_t(p.OW));
  p.fd_RS = FastDiv(std::uint32_t(s.R * s.S));
  p.fd_S = FastDiv(std::uint32_t(s.S));
  p.fd_ks = FastDiv(std::uint32_t(p.ksteps));
  return p;
}

cudaError_t pack(const PackParams& p, cudaStream_t st) {
  const int blocks = cdiv(p.rows, p.ROWS) * p.ksteps;
  count_launch();
  pack_kernel<<<blocks, 256, 0, st>>>(p);
  return cudaGetLastError();
}

cudaError_t gemm(const Problem& q, const float* a, const float* b, int epi, float* out, float alpha, float beta,
                 int P, int ld, bool split_k, cudaStream_t st, int batch = 1, std::int64_t a_bs = 0,
                 std::int64_t b_bs = 0, std::int64_t o_bs = 0) {
  GemmParams g{};
  g.a = a;
  g.b = b;
  g.out = out;
  g.alpha = alpha;
  g.beta = beta;
  g.m_tiles = q.m_tiles;
  g.n_tiles = q.n_tiles;
  g.ksteps = q.ksteps;
  g.BN = q.BN;
  const int tiles = q.m_tiles * q.n_tiles;
  int splits = 1;
  if (split_k && !deterministic()) splits = std::max(1, std::min(q.ksteps / 16, cdiv(3 * sms(), tiles)));
  g.steps_per_unit = cdiv(q.ksteps, splits);
  g.splits = cdiv(q.ksteps, g.steps_per_unit);
  g.epi = epi;
  g.M = q.M;
  g.Nc = q.Nc;
  g.P = P;
  g.ld = ld;
  g.fd_P = FastDiv(std::uint32_t(P > 0 ? P : 1));
  g.batch = batch;
  g.a_bs = a_bs;
  g.b_bs = b_bs;
  g.o_bs = o_bs;
  const int stage = kBM * 128 + ((q.BN * 128 + 127) & ~127);
  const int smem = std::max(kStages * stage + 1024 + 256, 116 * 1024);
  if (smem > 48 * 1024) {
    cudaError_t e = set_smem_attr(reinterpret_cast<const void*>(tiled_gemm_kernel), 227 * 1024);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  tiled_gemm_kernel<<<std::min(std::int64_t(sms()), std::int64_t(tiles) * g.splits * batch), kThreads, smem, st>>>(g);
  return cudaGetLastError();
}

}  // namespace

int blocked_bn(int n) { return pick_bn(n); }

cudaError_t batched_gemm_colmajor(int batch, int M, int Nc, int Kr, const float* a, std::int64_t a_bs, const float* b,
                                  std::int64_t b_bs, float* out, std::int64_t o_bs, int ld, cudaStream_t st) {
  return gemm(make_problem(M, Nc, Kr), a, b, kEpiColMajor, out, 1.f, 0.f, 0, ld, false, st, batch, a_bs, b_bs, o_bs);
}

bool gemm_supports(int, const ConvShape& s) {
  return std::int64_t(s.N) * s.OH() * s.OW() < (std::int64_t(1) << 31) && s.x_elems() < (std::int64_t(1) << 31);
}

std::int64_t gemm_workspace(int op, const ConvShape& s) { return std::int64_t(workspace_of(op, s)); }

cudaError_t gemm_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                     float beta, cudaStream_t st, int flags) {
  const Problem q = problem_of(op, s);
  // B (the filter for Forward / BackwardData) first: batch-independent, so
  // later micro-batches of one call reuse it (kFilterReady)
  float* B = static_cast<float*>(ws);
  float* A = reinterpret_cast<float*>(static_cast<char*>(ws) + a256(q.b_bytes()));
  const bool filter_ready = (flags & kFilterReady) && op != kBwdFilter;
  const int CRS = s.C * s.R * s.S, P = s.OH() * s.OW();
  cudaError_t e;
  if (op == kFwd) {
    if ((e = pack(pack_params(s, kIm2colPix, a, A, q.M, CRS, 0, kBM), st)) != cudaSuccess) return e;
    if (!filter_ready && (e = pack(pack_params(s, kRowMajor, b, B, s.K, CRS, CRS, q.BN), st)) != cudaSuccess)
      return e;
    return gemm(q, A, B, kEpiNchw, out, alpha, beta, P, 0, false, st);
  }
  if (op == kBwdData) {
    float* dcol = reinterpret_cast<float*>(reinterpret_cast<char*>(A) + a256(q.a_bytes()));
    if ((e = pack(pack_params(s, kDyPixK, a, A, q.M, s.K, 0, kBM), st)) != cudaSuccess) return e;
    if (!filter_ready && (e = pack(pack_params(s, kColMajor, b, B, CRS, s.K, CRS, q.BN), st)) != cudaSuccess)
      return e;
    if ((e = gemm(q, A, B, kEpiRowMajor, dcol, 1.f, 0.f, 0, CRS, false, st)) != cudaSuccess) return e;
    const std::int64_t total = s.x_elems();
    count_launch();
    col2im_kernel<<<int(std::min<std::int64_t>(cdiv(total, 256), 16 * sms())), 256, 0, st>>>(
        dcol, out, s.N, s.C, s.H, s.W, s.R, s.S, s.ph, s.pw, s.sh, s.sw, s.OH(), s.OW(), alpha, beta);
    return cudaGetLastError();
  }
  if (beta != 1.f) {
    const std::int64_t n = s.w_elems();
    count_launch();
    scale_kernel<<<int(std::min<std::int64_t>(cdiv(n, 256), 4 * sms())), 256, 0, st>>>(out, n, beta);
  }
  if ((e = pack(pack_params(s, kIm2colCrs, a, A, CRS, q.Kr, 0, kBM), st)) != cudaSuccess) return e;
  if ((e = pack(pack_params(s, kDyKPix, b, B, s.K, q.Kr, 0, q.BN), st)) != cudaSuccess) return e;
  return gemm(q, A, B, kEpiAtomicT, out, alpha, 1.f, 0, CRS, true, st);
}

}  // namespace ucudnn
