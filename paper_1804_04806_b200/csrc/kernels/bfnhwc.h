// BackwardFilter of UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM_NHWC: channels-last
// copies of x and dy, TMA im2col / tiled boxes, MN-major tcgen05 operands
// (see bfnhwc.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "conv_common.h"

namespace ucudnn {

bool bfn_supports(const ConvShape& s);
std::int64_t bfn_workspace(const ConvShape& s);
// dw = beta * dw + alpha * sum (split-K, fp32 reductions into a GEMM-layout scratch)
// flags: kAccumulate / kDeferFinal (conv_common.h) for runs of micro-batches
cudaError_t bfn_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha, float beta,
                    cudaStream_t stream, int flags = 0);

}  // namespace ucudnn
