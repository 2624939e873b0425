#include "algos.h"

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "../kernels/bdscatter.h"
#include "../kernels/bflsu.h"
#include "../kernels/bfs.h"
#include "../kernels/bfnhwc.h"
#include "../kernels/fct.h"
#include "../kernels/fft.h"
#include "../kernels/gemm.h"
#include "../kernels/igemm.h"
#include "../kernels/precomp.h"
#include "../kernels/split.h"
#include "../kernels/winograd.h"

namespace ucudnn {

namespace {
std::atomic<std::uint64_t> g_launches{0};
}  // namespace
void count_launch(int n) { g_launches.fetch_add(std::uint64_t(n), std::memory_order_relaxed); }
std::uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

namespace {
thread_local bool t_det = false;
thread_local bool t_faithful = false;
}  // namespace
bool deterministic() { return t_det; }
void set_deterministic(bool on) { t_det = on; }
bool faithful() { return t_faithful; }
void set_faithful(bool on) { t_faithful = on; }

namespace {
std::int64_t al256(std::int64_t b) { return (b + 255) / 256 * 256; }
// elements of the two operands of op: F (x, w), BD (dy, w), BF (x, dy)
void operand_elems(int op, const ConvShape& s, std::int64_t* na, std::int64_t* nb) {
  *na = op == 1 ? s.y_elems() : s.x_elems();
  *nb = op == 2 ? s.y_elems() : s.w_elems();
}
}  // namespace

std::int64_t algo_workspace(const AlgoImpl* a, int op, const ConvShape& s) {
  const std::int64_t ws = a->workspace(op, s);
  if (!faithful()) return ws;
  std::int64_t na, nb;
  operand_elems(op, s, &na, &nb);
  return al256(ws) + 2 * al256(na * 4) + 2 * al256(nb * 4);
}

cudaError_t algo_run(const AlgoImpl* a, int op, const ConvShape& s, const float* A, const float* B, float* out,
                     void* ws, float alpha, float beta, cudaStream_t st, int flags) {
  if (!faithful()) return a->run(op, s, A, B, out, ws, alpha, beta, st, flags);
  std::int64_t na, nb;
  operand_elems(op, s, &na, &nb);
  char* base = static_cast<char*>(ws);
  float* ahi = reinterpret_cast<float*>(base + al256(a->workspace(op, s)));
  float* alo = reinterpret_cast<float*>(reinterpret_cast<char*>(ahi) + al256(na * 4));
  float* bhi = reinterpret_cast<float*>(reinterpret_cast<char*>(alo) + al256(na * 4));
  float* blo = reinterpret_cast<float*>(reinterpret_cast<char*>(bhi) + al256(nb * 4));
  cudaError_t e = split_tf32(A, ahi, alo, na, st);
  if (e == cudaSuccess) e = split_tf32(B, bhi, blo, nb, st);
  if (e != cudaSuccess) return e;
  // the three passes use two filter operands, so each repacks (no
  // kFilterReady across them) and run as complete calls (no deferral)
  const int f = flags & ~(kFilterReady | kAccumulate | kDeferFinal);
  e = a->run(op, s, ahi, bhi, out, ws, alpha, beta, st, f);
  if (e == cudaSuccess) e = a->run(op, s, alo, bhi, out, ws, alpha, 1.f, st, f | (op == 2 ? 0 : kFilterReady));
  if (e == cudaSuccess) e = a->run(op, s, ahi, blo, out, ws, alpha, 1.f, st, f);
  return e;
}

namespace {
std::atomic<bool> g_trace{false};
std::mutex g_trace_mu;
std::string g_trace_buf;
}  // namespace
bool trace_on() { return g_trace.load(std::memory_order_relaxed); }
void trace_variant(const char* fmt, ...) {
  if (!trace_on()) return;
  char line[256];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(line, sizeof line, fmt, ap);
  va_end(ap);
  std::lock_guard<std::mutex> lock(g_trace_mu);
  if (g_trace_buf.size() < (1u << 20)) g_trace_buf += std::string(line) + "\n";
}
void set_trace(bool on) {
  std::lock_guard<std::mutex> lock(g_trace_mu);
  g_trace.store(on);
  g_trace_buf.clear();
}
std::string take_trace() {
  std::lock_guard<std::mutex> lock(g_trace_mu);
  std::string s;
  s.swap(g_trace_buf);
  return s;
}

cudaError_t set_smem_attr(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (function, device) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  int& have = done[{func, dev}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

int tune(const char* key, int dflt) {
  static const std::string env = [] {
    const char* e = std::getenv("UCUDNN_TUNE");
    return std::string(e ? e : "");
  }();
  const std::string k = std::string(key) + "=";
  std::size_t pos = 0;
  while ((pos = env.find(k, pos)) != std::string::npos) {
    if (pos == 0 || env[pos - 1] == ',') return std::atoi(env.c_str() + pos + k.size());
    pos += k.size();
  }
  return dflt;
}

namespace {

bool igemm_supports(int, const ConvShape&) { return true; }
std::int64_t no_workspace(int, const ConvShape&) { return 0; }

cudaError_t igemm_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void*, float alpha,
                      float beta, cudaStream_t st, int) {
  switch (op) {
    case 0: return igemm_forward(s, a, b, out, alpha, beta, st);
    case 1: return igemm_backward_data(s, a, b, out, alpha, beta, st);
    case 2: return igemm_backward_filter(s, a, b, out, alpha, beta, st);
  }
  return cudaErrorInvalidValue;
}

bool wino2_supports(int op, const ConvShape& s) { return winograd_supports(2, op, s); }
std::int64_t wino2_workspace(int op, const ConvShape& s) { return winograd_workspace(2, op, s); }
cudaError_t wino2_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                      float beta, cudaStream_t st, int flags) {
  return winograd_run(2, op, s, a, b, out, ws, alpha, beta, st, flags);
}
bool wino4_supports(int op, const ConvShape& s) { return winograd_supports(4, op, s); }
std::int64_t wino4_workspace(int op, const ConvShape& s) { return winograd_workspace(4, op, s); }
cudaError_t wino4_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                      float beta, cudaStream_t st, int flags) {
  return winograd_run(4, op, s, a, b, out, ws, alpha, beta, st, flags);
}

// Gather/scatter family: BackwardFilter with operands gathered by cp.async
// straight from NCHW x / dy (bflsu.cu: a small fixed workspace instead of
// PRECOMP's per-image copies), and BackwardData of few-channel strided layers
// as GEMM + col2im fused through a shared-memory patch (bdscatter.cu).
// Few-channel strided BackwardFilter (AlexNet / ResNet conv1) takes the
// TMEM-operand kernel (fct.cu), else the shared-memory patch kernel (bfs.cu),
// instead of the strided L2 gather.
bool gather_supports(int op, const ConvShape& s) {
  return (op == 2 && (fct_bwdf_supports(s) || fct_bwdf1_supports(s) || bfs_supports(s) || bfl_supports(s))) ||
         (op == 1 && bds_supports(s));
}
std::int64_t gather_workspace(int op, const ConvShape& s) {
  if (op == 2)
    return fct_bwdf_supports(s)    ? fct_bwdf_workspace(s)
           : fct_bwdf1_supports(s) ? fct_bwdf1_workspace(s)
           : bfs_supports(s)       ? bfs_workspace(s)
                                   : bfl_workspace(s);
  return op == 1 ? bds_workspace(s) : 0;
}
cudaError_t gather_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                       float beta, cudaStream_t st, int) {
  if (op == 2) {
    if (fct_bwdf_supports(s)) return fct_bwdf_run(s, a, b, out, ws, alpha, beta, st);
    if (fct_bwdf1_supports(s)) return fct_bwdf1_run(s, a, b, out, ws, alpha, beta, st);
    return bfs_supports(s) ? bfs_run(s, a, b, out, ws, alpha, beta, st) : bfl_run(s, a, b, out, ws, alpha, beta, st);
  }
  if (op == 1) return bds_run(s, a, b, out, alpha, beta, st);
  return cudaErrorInvalidValue;
}

// Stride-1 F / BD whose input channels come in multiples of 32 take the
// TMEM-operand kernel (fct1.cu: input rows read once per tile, not once per
// filter tap; its workspace is only the flipped filter for BD), the others
// the precomp GEMM over reduction-channel slices.
bool sliced_supports(int op, const ConvShape& s) { return fct1_supports(op, s) || precomp_sliced_supports(op, s); }
std::int64_t sliced_workspace(int op, const ConvShape& s) {
  return fct1_supports(op, s) ? fct1_workspace(op, s) : precomp_sliced_workspace(op, s);
}
cudaError_t sliced_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                       float beta, cudaStream_t st, int flags) {
  if (fct1_supports(op, s)) return fct1_run(op, s, a, b, out, ws, alpha, beta, st, flags);
  return precomp_sliced_run(op, s, a, b, out, ws, alpha, beta, st);
}

// Channels-last family: BackwardFilter of stride-1 layers from NHWC copies of
// x and dy through TMA im2col boxes and MN-major tcgen05 operands (bfnhwc.cu).
bool nhwc_supports(int op, const ConvShape& s) { return op == 2 && bfn_supports(s); }
std::int64_t nhwc_workspace(int op, const ConvShape& s) { return op == 2 ? bfn_workspace(s) : 0; }
cudaError_t nhwc_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                     float beta, cudaStream_t st, int flags) {
  if (op == 2) return bfn_run(s, a, b, out, ws, alpha, beta, st, flags);
  return cudaErrorInvalidValue;
}

const AlgoImpl kImplicitGemm{0, "IMPLICIT_GEMM", igemm_supports, no_workspace, igemm_run};
const AlgoImpl kWinograd{1, "WINOGRAD", wino2_supports, wino2_workspace, wino2_run, 0, false};
const AlgoImpl kWinograd4{4, "WINOGRAD_4x4", wino4_supports, wino4_workspace, wino4_run, 0, false};
const AlgoImpl kFft{2, "FFT", fft_supports, fft_workspace, fft_run, 0, false};
const AlgoImpl kGemm{3, "GEMM", gemm_supports, gemm_workspace, gemm_run};
const AlgoImpl kPrecomp{5, "IMPLICIT_PRECOMP_GEMM", precomp_supports, precomp_workspace, precomp_run};
const AlgoImpl kGather{6, "IMPLICIT_GATHER_GEMM", gather_supports, gather_workspace, gather_run};
const AlgoImpl kSliced{7, "IMPLICIT_PRECOMP_GEMM_SLICED", sliced_supports, sliced_workspace, sliced_run};
const AlgoImpl kNhwc{8, "IMPLICIT_PRECOMP_GEMM_NHWC", nhwc_supports, nhwc_workspace, nhwc_run, 1 << 2};

}  // namespace

const AlgoImpl* find_algo(int id) {
  switch (id) {
    case 0: return &kImplicitGemm;
    case 1: return &kWinograd;
    case 2: return &kFft;
    case 4: return &kWinograd4;
    case 3: return &kGemm;
    case 5: return &kPrecomp;
    case 6: return &kGather;
    case 7: return &kSliced;
    case 8: return &kNhwc;
    default: return nullptr;
  }
}

int algo_count() { return 9; }

}  // namespace ucudnn
