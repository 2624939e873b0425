// UCUDNN_ALGO_WINOGRAD (F(2x2,3x3)) and UCUDNN_ALGO_WINOGRAD_4x4
// (F(4x4,3x3)): non-fused Winograd for 3x3, stride-1 Forward and
// BackwardData (= Forward of dy with the flipped, transposed filter).
//
//   V[p][t][c] = (B^T d_{t,c} B)[p]        input transform   (HBM / L2 bound)
//   U[p][k][c] = (G g_{k,c} G^T)[p]        filter transform  (tiny)
//   M[p][k][t] = sum_c V[p][t][c] U[p][k][c]   alpha^2 batched tcgen05 GEMMs
//   y tile     = A^T M_{t,k} A             output transform  (HBM / L2 bound)
//
// p runs over the alpha x alpha transform points (alpha = m + 2), t over the
// m x m output tiles of the micro-batch. The transforms write V and U straight
// into the blocked K-major layout the tiled GEMM streams with bulk copies
// (gemm.h), and the GEMM writes M column-major so the output transform reads
// it coalesced along tiles. The workspace -- alpha^2 * (T*C + K*C + K*T)
// floats -- grows with the micro-batch; small micro-batches keep V and M
// resident in the 126 MB L2, which is where micro-batching pays for Winograd.
//
// F(2x2,3x3): B, G, A hold 0, +-1 and 1/2, so on integer data in [-3, 3] every
// intermediate is a multiple of 1/4 well inside TF32's mantissa and the
// result is bit-exact. F(4x4,3x3) (1/6, 1/24 in G) is tolerance-checked only.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "conv_common.h"
#include "gemm.h"
#include "winograd.h"

namespace ucudnn {

namespace {

constexpr int kBM = 128;

// Transform matrices (row-major), F(2,3) and F(4,3) (Lavin & Gray 2016).
// constexpr so the fully unrolled transforms fold the zeros and +-1s away.
template <int M>
struct Wt {
  static constexpr int A = M + 2;
};
template <int M>
__device__ __forceinline__ float wBt(int i) {
  constexpr float b2[16] = {1, 0, -1, 0, 0, 1, 1, 0, 0, -1, 1, 0, 0, 1, 0, -1};
  constexpr float b4[36] = {4, 0, -5, 0, 1, 0, 0, -4, -4, 1, 1, 0, 0, 4, -4, -1, 1, 0,
                            0, -2, -1, 2, 1, 0, 0, 2, -1, -2, 1, 0, 0, 4, 0, -5, 0, 1};
  return M == 2 ? b2[i] : b4[i];
}
template <int M>
__device__ __forceinline__ float wG(int i) {
  constexpr float g2[12] = {1, 0, 0, 0.5f, 0.5f, 0.5f, 0.5f, -0.5f, 0.5f, 0, 0, 1};
  constexpr float g4[18] = {1.f / 4,  0,         0,        -1.f / 6, -1.f / 6, -1.f / 6,
                            -1.f / 6, 1.f / 6,   -1.f / 6, 1.f / 24, 1.f / 12, 1.f / 6,
                            1.f / 24, -1.f / 12, 1.f / 6,  0,        0,        1};
  return M == 2 ? g2[i] : g4[i];
}
template <int M>
__device__ __forceinline__ float wAt(int i) {
  constexpr float a2[8] = {1, 1, 1, 0, 0, 1, -1, -1};
  constexpr float a4[24] = {1, 1, 1, 1, 1, 0, 0, 1, -1, 2, -2, 0, 0, 1, 1, 4, 4, 0, 0, 1, -1, 8, -8, 1};
  return M == 2 ? a2[i] : a4[i];
}

struct WGeo {
  int N, Cin, Hin, Win, Cout, Hout, Wout, ph, pw;
  int m, alpha, P, th, tw, T, m_tiles, Cp, ksteps, BN, n_tiles, Mrows;
  int flip;  // BackwardData: filter read as W[c][k][2-r][2-s]
  std::int64_t a_bs, b_bs, o_bs;  // per-point strides (floats) of V, U, M
};

int cdiv(int a, int b) { return (a + b - 1) / b; }
std::size_t a256(std::size_t b) { return (b + 255) / 256 * 256; }

WGeo make_geo(int m, int N, int Cin, int Hin, int Win, int Cout, int Hout, int Wout, int ph, int pw, int flip) {
  WGeo g{};
  g.N = N; g.Cin = Cin; g.Hin = Hin; g.Win = Win; g.Cout = Cout; g.Hout = Hout; g.Wout = Wout;
  g.ph = ph; g.pw = pw; g.flip = flip;
  g.m = m;
  g.alpha = m + 2;
  g.P = g.alpha * g.alpha;
  g.th = cdiv(Hout, m);
  g.tw = cdiv(Wout, m);
  g.T = N * g.th * g.tw;
  g.m_tiles = cdiv(g.T, kBM);
  g.Mrows = g.m_tiles * kBM;
  g.Cp = cdiv(Cin, 32) * 32;
  g.ksteps = g.Cp / 32;
  g.BN = blocked_bn(Cout);
  g.n_tiles = cdiv(Cout, g.BN);
  g.a_bs = std::int64_t(g.m_tiles) * kBM * g.Cp;
  g.b_bs = std::int64_t(g.n_tiles) * g.BN * g.Cp;
  g.o_bs = std::int64_t(Cout) * g.Mrows;
  return g;
}

WGeo geo_of(int m, int op, const ConvShape& s) {
  if (op == kFwd) return make_geo(m, s.N, s.C, s.H, s.W, s.K, s.OH(), s.OW(), s.ph, s.pw, 0);
  return make_geo(m, s.N, s.K, s.OH(), s.OW(), s.C, s.H, s.W, 2 - s.ph, 2 - s.pw, 1);
}

std::size_t u_bytes(const WGeo& g) { return a256(std::size_t(g.P) * g.b_bs * 4); }
std::size_t v_bytes(const WGeo& g) { return a256(std::size_t(g.P) * g.a_bs * 4); }
std::size_t m_bytes(const WGeo& g) { return a256(std::size_t(g.P) * g.o_bs * 4); }

// Blocked position of element (row, col) inside a [tiles][kstep] blocked
// operand with `rows` rows per tile: [8 k-groups][rows][4].
__device__ __forceinline__ std::int64_t blocked(int row, int col, int rows, int ksteps) {
  const int tile = row / rows, r = row - tile * rows;
  const int ks = col >> 5, kg = (col & 31) >> 2, e = col & 3;
  return ((std::int64_t(tile) * ksteps + ks) * 8 + kg) * (rows * 4) + r * 4 + e;
}

// One thread per (tile row t, channel c); consecutive threads fill one
// 16-byte group of 4 channels, then consecutive rows -> coalesced stores.
template <int M>
__global__ void __launch_bounds__(256) input_transform(const float* __restrict__ x, float* __restrict__ V, WGeo g) {
  constexpr int A = Wt<M>::A;
  const std::int64_t total = std::int64_t(g.Mrows) * g.Cp;
  for (std::int64_t idx = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += std::int64_t(gridDim.x) * blockDim.x) {
    const int e = int(idx & 3);
    const int r = int((idx >> 2) % kBM);
    const std::int64_t rest = idx / (4 * kBM);
    const int cg = int(rest % (g.Cp / 4)), mt = int(rest / (g.Cp / 4));
    const int c = cg * 4 + e, t = mt * kBM + r;
    float d[A][A];
    const bool live = t < g.T && c < g.Cin;
    if (live) {
      const int per = g.th * g.tw, n = t / per, tt = t - n * per, ty = tt / g.tw, tx = tt - ty * g.tw;
      const int h0 = ty * M - g.ph, w0 = tx * M - g.pw;
      const float* src = x + (std::int64_t(n) * g.Cin + c) * g.Hin * g.Win;
#pragma unroll
      for (int i = 0; i < A; ++i)
#pragma unroll
        for (int j = 0; j < A; ++j) {
          const int h = h0 + i, w = w0 + j;
          d[i][j] = (unsigned(h) < unsigned(g.Hin) && unsigned(w) < unsigned(g.Win)) ? __ldg(src + h * g.Win + w) : 0.f;
        }
    }
    // tmp = Bt d ; V = tmp Bt^T
    float tmp[A][A];
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int j = 0; j < A; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < A; ++k) acc += wBt<M>(i * A + k) * (live ? d[k][j] : 0.f);
        tmp[i][j] = acc;
      }
    const std::int64_t pos = blocked(t, c, kBM, g.ksteps);
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int j = 0; j < A; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < A; ++k) acc += tmp[i][k] * wBt<M>(j * A + k);
        V[std::int64_t(i * A + j) * g.a_bs + pos] = acc;
      }
  }
}

template <int M>
__global__ void __launch_bounds__(256) filter_transform(const float* __restrict__ w, float* __restrict__ U, WGeo g) {
  constexpr int A = Wt<M>::A;
  const std::int64_t total = std::int64_t(g.n_tiles) * g.BN * g.Cp;
  for (std::int64_t idx = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += std::int64_t(gridDim.x) * blockDim.x) {
    const int e = int(idx & 3);
    const int r = int((idx >> 2) % g.BN);
    const std::int64_t rest = idx / (4 * g.BN);
    const int cg = int(rest % (g.Cp / 4)), nt = int(rest / (g.Cp / 4));
    const int c = cg * 4 + e, k = nt * g.BN + r;
    float f[3][3];
    const bool live = k < g.Cout && c < g.Cin;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        float v = 0.f;
        if (live)
          v = g.flip ? w[((std::int64_t(c) * g.Cout + k) * 3 + (2 - i)) * 3 + (2 - j)]
                     : w[((std::int64_t(k) * g.Cin + c) * 3 + i) * 3 + j];
        f[i][j] = v;
      }
    float tmp[A][3];
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) tmp[i][j] = wG<M>(i * 3 + 0) * f[0][j] + wG<M>(i * 3 + 1) * f[1][j] + wG<M>(i * 3 + 2) * f[2][j];
    const std::int64_t pos = blocked(k, c, g.BN, g.ksteps);
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int j = 0; j < A; ++j)
        U[std::int64_t(i * A + j) * g.b_bs + pos] =
            tmp[i][0] * wG<M>(j * 3 + 0) + tmp[i][1] * wG<M>(j * 3 + 1) + tmp[i][2] * wG<M>(j * 3 + 2);
  }
}

// One thread per (tile t, output channel k), lanes along t.
template <int M>
__global__ void __launch_bounds__(256) output_transform(const float* __restrict__ Mo, float* __restrict__ y, WGeo g,
                                                        float alpha, float beta) {
  constexpr int A = Wt<M>::A;
  const std::int64_t total = std::int64_t(g.Cout) * g.T;
  for (std::int64_t idx = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += std::int64_t(gridDim.x) * blockDim.x) {
    const int t = int(idx % g.T), k = int(idx / g.T);
    const float* src = Mo + std::int64_t(k) * g.Mrows + t;
    float mm[A][A];
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int j = 0; j < A; ++j) mm[i][j] = src[std::int64_t(i * A + j) * g.o_bs];
    float tmp[M][A];
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int j = 0; j < A; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < A; ++q) acc += wAt<M>(i * A + q) * mm[q][j];
        tmp[i][j] = acc;
      }
    const int per = g.th * g.tw, n = t / per, tt = t - n * per, ty = tt / g.tw, tx = tt - ty * g.tw;
    float* dst = y + (std::int64_t(n) * g.Cout + k) * g.Hout * g.Wout;
#pragma unroll
    for (int i = 0; i < M; ++i) {
      const int h = ty * M + i;
      if (h >= g.Hout) break;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const int w = tx * M + j;
        if (w >= g.Wout) break;
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < A; ++q) acc += tmp[i][q] * wAt<M>(j * A + q);
        float* o = dst + h * g.Wout + w;
        *o = beta == 0.f ? alpha * acc : alpha * acc + beta * *o;
      }
    }
  }
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

int grid_for(std::int64_t n) { return int(std::min<std::int64_t>((n + 255) / 256, 8 * sms())); }

template <int M>
cudaError_t run(const WGeo& g, const float* act, const float* w, float* out, void* ws, float alpha, float beta,
                cudaStream_t st, int flags) {
  float* U = static_cast<float*>(ws);  // filter first: reused by later micro-batches
  float* V = reinterpret_cast<float*>(static_cast<char*>(ws) + u_bytes(g));
  float* Mo = reinterpret_cast<float*>(reinterpret_cast<char*>(V) + v_bytes(g));
  if (!(flags & kFilterReady)) {
    count_launch();
    filter_transform<M><<<grid_for(std::int64_t(g.n_tiles) * g.BN * g.Cp), 256, 0, st>>>(w, U, g);
  }
  count_launch();
  input_transform<M><<<grid_for(std::int64_t(g.Mrows) * g.Cp), 256, 0, st>>>(act, V, g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = batched_gemm_colmajor(g.P, g.T, g.Cout, g.Cp, V, g.a_bs, U, g.b_bs, Mo, g.o_bs, g.Mrows, st);
  if (e != cudaSuccess) return e;
  count_launch();
  output_transform<M><<<grid_for(std::int64_t(g.Cout) * g.T), 256, 0, st>>>(Mo, out, g, alpha, beta);
  return cudaGetLastError();
}

}  // namespace

bool winograd_supports(int m, int op, const ConvShape& s) {
  if (op == kBwdFilter) return false;
  if (s.R != 3 || s.S != 3 || s.sh != 1 || s.sw != 1 || s.ph > 2 || s.pw > 2) return false;
  const WGeo g = geo_of(m, op, s);
  return std::int64_t(g.Mrows) * g.Cp < (std::int64_t(1) << 31) && std::int64_t(g.T) * g.Cout < (std::int64_t(1) << 31);
}

std::int64_t winograd_workspace(int m, int op, const ConvShape& s) {
  const WGeo g = geo_of(m, op, s);
  return std::int64_t(u_bytes(g) + v_bytes(g) + m_bytes(g));
}

cudaError_t winograd_run(int m, int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws,
                         float alpha, float beta, cudaStream_t st, int flags) {
  const WGeo g = geo_of(m, op, s);
  return m == 2 ? run<2>(g, a, b, out, ws, alpha, beta, st, flags) : run<4>(g, a, b, out, ws, alpha, beta, st, flags);
}

}  // namespace ucudnn
