// UCUDNN_ALGO_IMPLICIT_GEMM for 1x1 stride-1 unpadded layers: TMA-fed batched
// GEMM over the NCHW planes (see z1x1.cu). No workspace.
#pragma once

#include <cuda_runtime.h>

#include "conv_common.h"

namespace ucudnn {

bool z1x1_supports(int op, const ConvShape& s);
// op 0: a = x -> out = y; op 1: a = dy -> out = dx
cudaError_t z1x1_run(int op, const ConvShape& s, const float* a, const float* w, float* out, float alpha, float beta,
                     cudaStream_t stream);

}  // namespace ucudnn
