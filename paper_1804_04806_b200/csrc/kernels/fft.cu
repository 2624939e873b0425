// UCUDNN_ALGO_FFT: FFT-tiled convolution for stride-1 Forward and
// BackwardData (= Forward of dy with the flipped, transposed filter).
//
// The output is cut into L x L tiles (L = F - R + 1, F = 16 or 32); each tile
// reads an F x F input window. With real 2-D DFTs of size F (F x (F/2+1)
// Hermitian bins), correlation is a per-bin complex product with the
// conjugated filter spectrum, summed over input channels:
//
//   X[f][t][c]  = DFT(x window of tile t, channel c)          input transform
//   W~[f][k][c] = conj(DFT(w[k][c] zero-padded to F x F))     filter transform
//   Y[f][k][t]  = sum_c X[f][t][c] * W~[f][k][c]              F(F/2+1) complex GEMMs
//   y tile      = IDFT(Y[.][k][t]) [0:L, 0:L] / F^2            output transform
//
// Each complex GEMM runs as one real tcgen05 GEMM: A = [Re X | Im X] (tiles x
// 2C), B rows k = [Re W | Im W] (-> Re Y) and Kp + k = [-Im W | Re W] (-> Im Y),
// which folds the conjugation in. The 2-D DFTs are row then column radix-2
// FFTs held in registers (one thread per line, shared-memory staging),
// cheap next to the GEMM. Workspace is dominated by the two spectra -- F(F/2+1) * 2C * (T + 2K)
// floats -- far above the direct algorithms', the classic FFT trade that the
// micro-batch planner arbitrates.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "conv_common.h"
#include "fft.h"
#include "gemm.h"

namespace ucudnn {

namespace {

constexpr int kBM = 128;

struct FGeo {
  int N, Cin, Hin, Win, Cout, Hout, Wout, R, S, ph, pw;
  int F, L, Fb, nf;       // DFT size, valid outputs per tile side, bins per row (F/2+1), bins
  int th, tw, T, m_tiles, Mrows;
  int Cp, Kp;             // channel counts padded to 16 (2*Cp, 2*Kp multiples of 32)
  int ksteps, BN, n_tiles;
  int flip;               // BackwardData filter indexing
  std::int64_t a_bs, b_bs, o_bs;
};

int cdiv(int a, int b) { return (a + b - 1) / b; }
std::size_t a256(std::size_t b) { return (b + 255) / 256 * 256; }

FGeo make_geo(int N, int Cin, int Hin, int Win, int Cout, int Hout, int Wout, int R, int S, int ph, int pw, int flip) {
  FGeo g{};
  g.N = N; g.Cin = Cin; g.Hin = Hin; g.Win = Win; g.Cout = Cout; g.Hout = Hout; g.Wout = Wout;
  g.R = R; g.S = S; g.ph = ph; g.pw = pw; g.flip = flip;
  // smallest DFT whose tile covers the output plane, else 32
  const int need = std::max(Hout, Wout) + std::max(R, S) - 1;
  g.F = need <= 16 ? 16 : 32;
  g.L = g.F - std::max(R, S) + 1;
  g.Fb = g.F / 2 + 1;
  g.nf = g.F * g.Fb;
  g.th = cdiv(Hout, g.L);
  g.tw = cdiv(Wout, g.L);
  g.T = N * g.th * g.tw;
  g.m_tiles = cdiv(g.T, kBM);
  g.Mrows = g.m_tiles * kBM;
  g.Cp = cdiv(Cin, 16) * 16;
  g.Kp = cdiv(Cout, 16) * 16;
  g.ksteps = 2 * g.Cp / 32;
  g.BN = blocked_bn(2 * g.Kp);
  g.n_tiles = cdiv(2 * g.Kp, g.BN);
  g.a_bs = std::int64_t(g.Mrows) * 2 * g.Cp;
  g.b_bs = std::int64_t(g.n_tiles) * g.BN * 2 * g.Cp;
  g.o_bs = std::int64_t(2 * g.Kp) * g.Mrows;
  return g;
}

FGeo geo_of(int op, const ConvShape& s) {
  if (op == kFwd) return make_geo(s.N, s.C, s.H, s.W, s.K, s.OH(), s.OW(), s.R, s.S, s.ph, s.pw, 0);
  return make_geo(s.N, s.K, s.OH(), s.OW(), s.C, s.H, s.W, s.R, s.S, s.R - 1 - s.ph, s.S - 1 - s.pw, 1);
}

std::size_t u_bytes(const FGeo& g) { return a256(std::size_t(g.nf) * g.b_bs * 4); }
std::size_t v_bytes(const FGeo& g) { return a256(std::size_t(g.nf) * g.a_bs * 4); }
std::size_t y_bytes(const FGeo& g) { return a256(std::size_t(g.nf) * g.o_bs * 4); }

__device__ __forceinline__ std::int64_t blocked(int row, int col, int rows, int ksteps) {
  const int tile = row / rows, r = row - tile * rows;
  const int ks = col >> 5, kg = (col & 31) >> 2, e = col & 3;
  return ((std::int64_t(tile) * ksteps + ks) * 8 + kg) * (rows * 4) + r * 4 + e;
}

constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }
constexpr int bitrev(int i, int bits) { return bits == 0 ? 0 : ((i & 1) << (bits - 1)) | bitrev(i >> 1, bits - 1); }

// In-register radix-2 FFT of length F: X[k] = sum_n x[n] e^{dir * 2 pi i n k / F}
// (dir = -1 forward, +1 inverse, unnormalised). tc/ts[m] = cos/sin(2 pi m / F).
template <int F>
__device__ __forceinline__ void fft_reg(float (&re)[F], float (&im)[F], const float* tc, const float* ts, float dir) {
  constexpr int LOG = ilog2(F);
#pragma unroll
  for (int i = 0; i < F; ++i) {
    const int j = bitrev(i, LOG);
    if (j > i) {
      const float tr = re[i], ti = im[i];
      re[i] = re[j];
      im[i] = im[j];
      re[j] = tr;
      im[j] = ti;
    }
  }
#pragma unroll
  for (int len = 2; len <= F; len <<= 1) {
    const int half = len >> 1, step = F / len;
#pragma unroll
    for (int i = 0; i < F; i += len)
#pragma unroll
      for (int k = 0; k < half; ++k) {
        const float c = tc[k * step], sn = dir * ts[k * step];
        const int a = i + k, b = i + k + half;
        const float xr = re[b] * c - im[b] * sn, xi = re[b] * sn + im[b] * c;
        re[b] = re[a] - xr;
        im[b] = im[a] - xi;
        re[a] += xr;
        im[a] += xi;
      }
  }
}

__device__ __forceinline__ void twiddles(float* tc, float* ts, int F) {
  for (int m = threadIdx.x; m < F / 2; m += blockDim.x) sincospif(2.f * float(m) / float(F), &ts[m], &tc[m]);
}

// Forward real 2-D DFT of 4 F x F planes held in smem `in` ([4][F][F+1]),
// result in `re`/`im` ([4][F][Fb]): row FFTs (one thread per row, real input,
// bins 0..F/2 kept) then column FFTs (one thread per column).
template <int F>
__device__ __forceinline__ void dft2_fwd(const float* in, float* re, float* im, float* tr, float* ti, const float* tc,
                         const float* ts) {
  constexpr int P = F + 1, Fb = F / 2 + 1;
  for (int row = threadIdx.x; row < 4 * F; row += blockDim.x) {
    float xr[F], xi[F];
#pragma unroll
    for (int b = 0; b < F; ++b) {
      xr[b] = in[row * P + b];
      xi[b] = 0.f;
    }
    fft_reg<F>(xr, xi, tc, ts, -1.f);
#pragma unroll
    for (int v = 0; v < Fb; ++v) {
      tr[row * Fb + v] = xr[v];
      ti[row * Fb + v] = xi[v];
    }
  }
  __syncthreads();
  for (int col = threadIdx.x; col < 4 * Fb; col += blockDim.x) {
    const int q = col / Fb, v = col - q * Fb;
    float xr[F], xi[F];
#pragma unroll
    for (int a = 0; a < F; ++a) {
      xr[a] = tr[(q * F + a) * Fb + v];
      xi[a] = ti[(q * F + a) * Fb + v];
    }
    fft_reg<F>(xr, xi, tc, ts, -1.f);
#pragma unroll
    for (int u = 0; u < F; ++u) {
      re[(q * F + u) * Fb + v] = xr[u];
      im[(q * F + u) * Fb + v] = xi[u];
    }
  }
  __syncthreads();
}

// One CTA per (tile t, 4 consecutive channels): window -> spectrum -> the
// blocked A operand (Re at column c, Im at column Cp + c).
template <int F>
__global__ void __launch_bounds__(256) fft_input(const float* __restrict__ x, float* __restrict__ A, FGeo g) {
  extern __shared__ float sm[];
  constexpr int Fb = F / 2 + 1, P = F + 1;
  float* in = sm;
  float* tr = in + 4 * F * P;
  float* ti = tr + 4 * F * Fb;
  float* re = ti + 4 * F * Fb;
  float* im = re + 4 * F * Fb;
  float* tc = im + 4 * F * Fb;
  float* ts = tc + F / 2;
  twiddles(tc, ts, F);
  const int t = blockIdx.x, c0 = blockIdx.y * 4;
  const int per = g.th * g.tw, n = t / per, tt = t - n * per, ty = tt / g.tw, tx = tt - ty * g.tw;
  const int h0 = ty * g.L - g.ph, w0 = tx * g.L - g.pw;
  for (int idx = threadIdx.x; idx < 4 * F * F; idx += blockDim.x) {
    const int b = idx % F, a = (idx / F) % F, q = idx / (F * F), c = c0 + q;
    const int h = h0 + a, w = w0 + b;
    float v = 0.f;
    if (c < g.Cin && unsigned(h) < unsigned(g.Hin) && unsigned(w) < unsigned(g.Win))
      v = __ldg(x + ((std::int64_t(n) * g.Cin + c) * g.Hin + h) * g.Win + w);
    in[(q * F + a) * P + b] = v;
  }
  __syncthreads();
  dft2_fwd<F>(in, re, im, tr, ti, tc, ts);
  for (int idx = threadIdx.x; idx < g.nf * 4; idx += blockDim.x) {
    const int q = idx & 3, f = idx >> 2;
    const float r = re[q * g.nf + f], i = im[q * g.nf + f];
    float* plane = A + std::int64_t(f) * g.a_bs;
    plane[blocked(t, c0 + q, kBM, g.ksteps)] = r;
    plane[blocked(t, g.Cp + c0 + q, kBM, g.ksteps)] = i;
  }
}

// One CTA per (output channel k, 4 input channels): filter spectrum into
// the blocked B operand (rows k and Kp + k).
template <int F>
__global__ void __launch_bounds__(256) fft_filter(const float* __restrict__ w, float* __restrict__ B, FGeo g) {
  extern __shared__ float sm[];
  constexpr int Fb = F / 2 + 1, P = F + 1;
  float* in = sm;
  float* tr = in + 4 * F * P;
  float* ti = tr + 4 * F * Fb;
  float* re = ti + 4 * F * Fb;
  float* im = re + 4 * F * Fb;
  float* tc = im + 4 * F * Fb;
  float* ts = tc + F / 2;
  twiddles(tc, ts, F);
  const int k = blockIdx.x, c0 = blockIdx.y * 4;
  for (int idx = threadIdx.x; idx < 4 * F * F; idx += blockDim.x) {
    const int b = idx % F, a = (idx / F) % F, q = idx / (F * F), c = c0 + q;
    float v = 0.f;
    if (c < g.Cin && k < g.Cout && a < g.R && b < g.S)
      v = g.flip ? w[((std::int64_t(c) * g.Cout + k) * g.R + (g.R - 1 - a)) * g.S + (g.S - 1 - b)]
                 : w[((std::int64_t(k) * g.Cin + c) * g.R + a) * g.S + b];
    in[(q * F + a) * P + b] = v;
  }
  __syncthreads();
  dft2_fwd<F>(in, re, im, tr, ti, tc, ts);
  for (int idx = threadIdx.x; idx < g.nf * 4; idx += blockDim.x) {
    const int q = idx & 3, f = idx >> 2;
    const float r = re[q * g.nf + f], i = im[q * g.nf + f];
    float* plane = B + std::int64_t(f) * g.b_bs;
    const int c = c0 + q;
    plane[blocked(k, c, g.BN, g.ksteps)] = r;            // Re Y row: [Re W | Im W]
    plane[blocked(k, g.Cp + c, g.BN, g.ksteps)] = i;
    plane[blocked(g.Kp + k, c, g.BN, g.ksteps)] = -i;    // Im Y row: [-Im W | Re W]
    plane[blocked(g.Kp + k, g.Cp + c, g.BN, g.ksteps)] = r;
  }
}

// One CTA per (8 consecutive tiles, output channel k): gather the spectrum
// (coalesced along tiles), inverse column FFTs, inverse Hermitian row FFTs,
// crop, alpha/beta store.
constexpr int kOT = 8;
template <int F>
__global__ void __launch_bounds__(256) fft_output(const float* __restrict__ Y, float* __restrict__ y, FGeo g,
                                                  float alpha, float beta) {
  extern __shared__ float sm[];
  constexpr int Fb = F / 2 + 1, nf = F * Fb;
  float* yr = sm;  // [kOT][F][Fb]
  float* yi = yr + kOT * nf;
  float* tc = yi + kOT * nf;
  float* ts = tc + F / 2;
  twiddles(tc, ts, F);
  const int t0 = blockIdx.x * kOT, k = blockIdx.y;
  for (int idx = threadIdx.x; idx < kOT * nf; idx += blockDim.x) {
    const int q = idx % kOT, f = idx / kOT, t = t0 + q;
    float r = 0.f, i = 0.f;
    if (t < g.T) {
      const float* plane = Y + std::int64_t(f) * g.o_bs;
      r = plane[std::int64_t(k) * g.Mrows + t];
      i = plane[std::int64_t(g.Kp + k) * g.Mrows + t];
    }
    yr[q * nf + f] = r;
    yi[q * nf + f] = i;
  }
  __syncthreads();
  // column inverse FFTs (over u), in place
  for (int col = threadIdx.x; col < kOT * Fb; col += blockDim.x) {
    const int q = col / Fb, v = col - q * Fb;
    float xr[F], xi[F];
#pragma unroll
    for (int u = 0; u < F; ++u) {
      xr[u] = yr[q * nf + u * Fb + v];
      xi[u] = yi[q * nf + u * Fb + v];
    }
    fft_reg<F>(xr, xi, tc, ts, 1.f);
#pragma unroll
    for (int a = 0; a < F; ++a) {
      yr[q * nf + a * Fb + v] = xr[a];
      yi[q * nf + a * Fb + v] = xi[a];
    }
  }
  __syncthreads();
  // row inverse FFTs: rebuild the full row from its Hermitian half
  const float scale = alpha / float(F * F);
  for (int row = threadIdx.x; row < kOT * g.L; row += blockDim.x) {
    const int q = row / g.L, a = row - q * g.L, t = t0 + q;
    if (t >= g.T) continue;
    float xr[F], xi[F];
#pragma unroll
    for (int v = 0; v < F; ++v) {
      const int vv = v < Fb ? v : F - v;
      const float r = yr[q * nf + a * Fb + vv], i = yi[q * nf + a * Fb + vv];
      xr[v] = r;
      xi[v] = v < Fb ? i : -i;
    }
    fft_reg<F>(xr, xi, tc, ts, 1.f);
    const int per = g.th * g.tw, n = t / per, tt = t - n * per, ty = tt / g.tw, tx = tt - ty * g.tw;
    const int h = ty * g.L + a;
    if (h >= g.Hout) continue;
    float* orow = y + ((std::int64_t(n) * g.Cout + k) * g.Hout + h) * g.Wout;
#pragma unroll
    for (int b = 0; b < F; ++b) {
      const int w = tx * g.L + b;
      if (b >= g.L || w >= g.Wout) break;
      float* o = orow + w;
      *o = beta == 0.f ? scale * xr[b] : scale * xr[b] + beta * *o;
    }
  }
}

int in_smem(const FGeo& g) { return (4 * g.F * (g.F + 1) + 4 * 4 * g.F * g.Fb + g.F) * 4; }
int out_smem(const FGeo& g) { return (2 * kOT * g.nf + g.F) * 4; }

template <int F>
cudaError_t launch(const FGeo& g, const float* a, const float* b, float* U, float* V, float* Yf, float* out,
                   float alpha, float beta, cudaStream_t st, int flags) {
  set_smem_attr(reinterpret_cast<const void*>(fft_output<F>), 200 * 1024);
  set_smem_attr(reinterpret_cast<const void*>(fft_input<F>), 200 * 1024);
  set_smem_attr(reinterpret_cast<const void*>(fft_filter<F>), 200 * 1024);
  // grid y covers the padded channels too, so their A / B columns are written
  // as zeros (garbage there would poison the GEMM); padded rows only feed
  // outputs that are never read
  if (!(flags & kFilterReady)) {
    count_launch();
    fft_filter<F><<<dim3(g.Cout, g.Cp / 4), 256, in_smem(g), st>>>(b, U, g);
  }
  count_launch();
  fft_input<F><<<dim3(g.T, g.Cp / 4), 256, in_smem(g), st>>>(a, V, g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = batched_gemm_colmajor(g.nf, g.T, 2 * g.Kp, 2 * g.Cp, V, g.a_bs, U, g.b_bs, Yf, g.o_bs, g.Mrows, st);
  if (e != cudaSuccess) return e;
  count_launch();
  fft_output<F><<<dim3(cdiv(g.T, kOT), g.Cout), 256, out_smem(g), st>>>(Yf, out, g, alpha, beta);
  return cudaGetLastError();
}

}  // namespace

bool fft_supports(int op, const ConvShape& s) {
  if (op == kBwdFilter || s.sh != 1 || s.sw != 1) return false;
  if (op == kBwdData && (s.ph > s.R - 1 || s.pw > s.S - 1)) return false;
  if (std::max(s.R, s.S) > 16) return false;
  const FGeo g = geo_of(op, s);
  return g.L >= 1 && std::int64_t(g.Mrows) * 2 * g.Cp < (std::int64_t(1) << 31) && g.T < (1 << 30) &&
         out_smem(g) <= 200 * 1024;
}

std::int64_t fft_workspace(int op, const ConvShape& s) {
  const FGeo g = geo_of(op, s);
  return std::int64_t(u_bytes(g) + v_bytes(g) + y_bytes(g));
}

cudaError_t fft_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                    float beta, cudaStream_t st, int flags) {
  const FGeo g = geo_of(op, s);
  float* U = static_cast<float*>(ws);  // filter spectrum first: reused across micro-batches
  float* V = reinterpret_cast<float*>(static_cast<char*>(ws) + u_bytes(g));
  float* Yf = reinterpret_cast<float*>(reinterpret_cast<char*>(V) + v_bytes(g));
  return g.F == 16 ? launch<16>(g, a, b, U, V, Yf, out, alpha, beta, st, flags)
                   : launch<32>(g, a, b, U, V, Yf, out, alpha, beta, st, flags);
}

}  // namespace ucudnn
