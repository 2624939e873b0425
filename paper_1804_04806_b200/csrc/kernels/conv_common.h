// Shapes and launch parameters shared by host launchers and device kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#ifdef __CUDACC__
#define UC_HD __host__ __device__ __forceinline__
#else
#define UC_HD inline
#endif

namespace ucudnn {

// Experiment knob: integer `key` from UCUDNN_TUNE="key=v,key=v" (parsed
// once), else `dflt`. Only used for A/B timing of pipeline parameters.
int tune(const char* key, int dflt);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, bytes) for `func` on the
// calling thread's current device, once per (function, device): function
// attributes belong to a device context, and the benchmarker may time
// algorithms on several devices from several host threads at once
// (ucudnnSetBenchmarkDevices). Thread-safe. Returns the CUDA error, if any.
cudaError_t set_smem_attr(const void* func, int bytes);

// Host-side count of device kernels this library has launched (evidence for
// bench.py's gpu_launches; see ucudnnGetLaunchCount).
void count_launch(int n = 1);
std::uint64_t launch_count();

// Launch-variant trace (ucudnnDebugSetTrace / ucudnnDebugGetTrace): when on,
// launchers append one line per main-kernel launch naming the variant and
// its tiling (e.g. "precomp2 m_tiles=729 n_tiles=1 clusters=74"), so tests can
// prove which code path a bench-scale call exercised. Off: one atomic load.
// Deterministic BackwardFilter (ucudnnSetDeterministic): set by the engine on
// the launching host thread around a handle's calls; split-K launchers then
// give each output element a single writer per launch (splits = 1), so dW no
// longer depends on the order of fp32 atomic additions.
bool deterministic();
void set_deterministic(bool on);
// FP32-faithful math (ucudnnSetMathMode): set like deterministic(); the engine
// then runs every algorithm as three TF32 passes over split operands.
bool faithful();
void set_faithful(bool on);

bool trace_on();
void trace_variant(const char* fmt, ...);

// Unsigned division by a runtime constant via multiply-high (valid for
// dividends < 2^31): q = umulhi(n, mul) >> shr, or n when d == 1.
struct FastDiv {
  std::uint32_t d = 1, mul = 0, shr = 0;
  FastDiv() = default;
  explicit FastDiv(std::uint32_t div) : d(div) {
    if (div <= 1) { d = 1; return; }
    std::uint32_t l = 0;
    while ((1ull << l) < div) ++l;  // ceil(log2(div))
    std::uint64_t p = 31 + l;
    mul = std::uint32_t(((1ull << p) + div - 1) / div);
    shr = std::uint32_t(p - 32);
  }
  UC_HD std::uint32_t div(std::uint32_t n) const {
#ifdef __CUDA_ARCH__
    return d == 1 ? n : (__umulhi(n, mul) >> shr);
#else
    return d == 1 ? n : std::uint32_t((std::uint64_t(n) * mul >> 32) >> shr);
#endif
  }
  UC_HD void divmod(std::uint32_t n, std::uint32_t& q, std::uint32_t& r) const {
    q = div(n);
    r = n - q * d;
  }
};

// One convolution layer at a given (micro-)batch N. Output dims derived.
struct ConvShape {
  int N = 1, C = 1, H = 1, W = 1, K = 1, R = 1, S = 1;
  int ph = 0, pw = 0, sh = 1, sw = 1;
  int OH() const { return (H + 2 * ph - R) / sh + 1; }
  int OW() const { return (W + 2 * pw - S) / sw + 1; }
  std::int64_t x_elems() const { return std::int64_t(N) * C * H * W; }
  std::int64_t y_elems() const { return std::int64_t(N) * K * OH() * OW(); }
  std::int64_t w_elems() const { return std::int64_t(K) * C * R * S; }
  double flops() const { return 2.0 * N * K * C * R * S * double(OH()) * OW(); }
};

enum ConvOp : int { kFwd = 0, kBwdData = 1, kBwdFilter = 2 };
constexpr int kFilterReady = 1;
// BackwardFilter runs of consecutive micro-batches on one algorithm that
// keeps fp32 partial sums in a workspace scratch (AlgoImpl::defer_ops):
// kAccumulate -- the previous micro-batch of this call left its partial sums
// there, keep adding (no reset); kDeferFinal -- the next micro-batch continues,
// skip the scratch -> dW finalize (the last one applies alpha / beta once).
constexpr int kAccumulate = 2;
constexpr int kDeferFinal = 4;

// Parameters of one implicit-GEMM launch. GEMM view per op:
//   Fwd : rows = output pixels (n,oh,ow), cols = K, red = (c,r,s)
//   BwdData (one stride phase (pa,pb)): rows = input pixels of the phase,
//         cols = C, red = (k, rr, ss) with r = pa + sh*rr, s = pb + sw*ss
//   BwdFilter: rows = (c,r,s), cols = K, red = pixels (n,oh,ow), split-K
struct IgemmParams {
  const float* a;  // Fwd: x, BwdData: dy, BwdFilter: x
  const float* b;  // Fwd: w, BwdData: w,  BwdFilter: dy
  float* out;      // y / dx / dw
  float alpha, beta;
  int M, Ng, Kg;          // GEMM rows, cols, reduction length
  int BN;                 // column tile (multiple of 16, <= 256)
  int chunks_per_split;   // reduction chunks (32 elements) per grid.z slice
  int stages;
  int N, C, H, W, K, R, S, ph, pw, sh, sw, OH, OW;
  // BwdData phase geometry
  int pa, pb, Ra, Sb, jh0, jw0, Hp, Wp;
  FastDiv fd_P, fd_OW, fd_RS, fd_S, fd_HWp, fd_Wp, fd_RaSb, fd_Sb;
  std::uint32_t lbo_a, lbo_b, stage_bytes, table_bytes;
};

}  // namespace ucudnn
