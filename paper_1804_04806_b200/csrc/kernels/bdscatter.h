// BackwardData of UCUDNN_ALGO_IMPLICIT_GATHER_GEMM for few-channel strided
// layers: GEMM + col2im fused through a shared-memory dx patch (bdscatter.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "conv_common.h"

namespace ucudnn {

bool bds_supports(const ConvShape& s);
std::int64_t bds_workspace(const ConvShape& s);
// dx = beta * dx + alpha * BackwardData(dy, w)
cudaError_t bds_run(const ConvShape& s, const float* dy, const float* w, float* dx, float alpha, float beta,
                    cudaStream_t stream);

}  // namespace ucudnn
