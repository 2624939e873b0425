// UCUDNN_ALGO_WINOGRAD (m = 2: F(2x2,3x3)) and UCUDNN_ALGO_WINOGRAD_4x4
// (m = 4: F(4x4,3x3)); non-fused transforms + batched tcgen05 GEMM
// (see winograd.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "conv_common.h"

namespace ucudnn {

bool winograd_supports(int m, int op, const ConvShape& s);
std::int64_t winograd_workspace(int m, int op, const ConvShape& s);
cudaError_t winograd_run(int m, int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws,
                         float alpha, float beta, cudaStream_t stream, int flags);

}  // namespace ucudnn
