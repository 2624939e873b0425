// UCUDNN_ALGO_GEMM (explicit im2col / col2im + tiled tcgen05 GEMM; see gemm.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "conv_common.h"

namespace ucudnn {

bool gemm_supports(int op, const ConvShape& s);
std::int64_t gemm_workspace(int op, const ConvShape& s);
cudaError_t gemm_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                     float beta, cudaStream_t stream, int flags);

}  // namespace ucudnn
