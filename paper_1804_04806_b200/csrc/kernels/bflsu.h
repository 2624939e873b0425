// BackwardFilter of UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM fed by cp.async
// gathers straight from NCHW x / dy (see bflsu.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "conv_common.h"

namespace ucudnn {

bool bfl_supports(const ConvShape& s);
std::int64_t bfl_workspace(const ConvShape& s);
// dw = beta * dw + alpha * sum (split-K, fp32 reductions into a GEMM-layout scratch)
cudaError_t bfl_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha, float beta,
                    cudaStream_t stream, bool direct = false);

}  // namespace ucudnn
