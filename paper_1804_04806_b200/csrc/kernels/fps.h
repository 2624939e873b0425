// Forward of few-channel strided layers from a space-to-depth patch in shared
// memory (UCUDNN_ALGO_IMPLICIT_GEMM's path for these shapes; see fps.cu).
#pragma once

#include <cuda_runtime.h>

#include "conv_common.h"

namespace ucudnn {

bool fps_supports(const ConvShape& s);
// y = alpha * conv(x, w) + beta * y; no workspace
cudaError_t fps_run(const ConvShape& s, const float* x, const float* w, float* y, float alpha, float beta,
                    cudaStream_t stream);

}  // namespace ucudnn
