// BackwardFilter of few-channel strided layers through a space-to-depth
// patch in shared memory (part of UCUDNN_ALGO_IMPLICIT_GATHER_GEMM; see bfs.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "conv_common.h"

namespace ucudnn {

bool bfs_supports(const ConvShape& s);
// per-CTA partial-sum slices (batch-independent)
std::int64_t bfs_workspace(const ConvShape& s);
// dw = beta * dw + alpha * sum; deterministic (slices added in a fixed order)
cudaError_t bfs_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha, float beta,
                    cudaStream_t stream);

}  // namespace ucudnn
