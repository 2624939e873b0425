// BackwardFilter of UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM (TMA-tiled operands,
// no im2col; see bfilter.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "conv_common.h"

namespace ucudnn {

bool bf_supports(const ConvShape& s);
std::int64_t bf_workspace(const ConvShape& s);
// dw = beta * dw + alpha * sum (split-K, fp32 reductions)
cudaError_t bf_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha, float beta,
                   cudaStream_t stream);

void bf_profile(double out[4]);  // diagnostic (UCUDNN_TUNE=prof=1)

}  // namespace ucudnn
