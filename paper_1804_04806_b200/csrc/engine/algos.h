// Registry of the concrete B200 convolution algorithms. Each algorithm has a
// different workspace footprint; the cost table holds one (time, workspace,
// feasible) row per (kernel, algorithm, micro-batch) and the planner picks
// among them.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../kernels/conv_common.h"

namespace ucudnn {

struct AlgoImpl {
  int id;
  const char* name;
  // Whether the algorithm implements `op` for this shape (any micro-batch).
  bool (*supports)(int op, const ConvShape& s);
  // Workspace bytes at micro-batch s.N.
  std::int64_t (*workspace)(int op, const ConvShape& s);
  // op 0: a = x, b = w, out = y; op 1: a = dy, b = w, out = dx;
  // op 2: a = x, b = dy, out = dw. flags & kFilterReady: the previous
  // micro-batch of the same call already prepared the (batch-independent)
  // filter operand at the start of `ws`, so it is not re-packed.
  cudaError_t (*run)(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws,
                     float alpha, float beta, cudaStream_t stream, int flags);
  // bit `op` set: run() honours kAccumulate / kDeferFinal for that op
  int defer_ops = 0;
  // the tensor cores consume the caller's operands themselves (not a
  // Winograd / FFT transform of them), so the FP32-faithful mode's operand
  // split makes the products exact: false = not offered in that mode
  bool splits_exact = true;
};

// Workspace / run of an algorithm in the calling thread's math mode: plain
// TF32, or FP32-faithful (faithful(): three TF32 passes over hi / lo operand
// splits held after the algorithm's own workspace).
std::int64_t algo_workspace(const AlgoImpl* a, int op, const ConvShape& s);
cudaError_t algo_run(const AlgoImpl* a, int op, const ConvShape& s, const float* A, const float* B, float* out,
                     void* ws, float alpha, float beta, cudaStream_t st, int flags);

// nullptr for ids that are reserved / not built.
const AlgoImpl* find_algo(int id);
int algo_count();  // ids are 0 .. algo_count()-1

// ucudnnDebugSetTrace / ucudnnDebugGetTrace backing (kernels call trace_variant)
void set_trace(bool on);
std::string take_trace();

}  // namespace ucudnn
