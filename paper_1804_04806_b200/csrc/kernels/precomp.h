// UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM (TMA-fed implicit GEMM; see precomp.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "conv_common.h"

namespace ucudnn {

bool precomp_supports(int op, const ConvShape& s);
std::int64_t precomp_workspace(int op, const ConvShape& s);
cudaError_t precomp_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws,
                        float alpha, float beta, cudaStream_t stream, int flags);

// UCUDNN_ALGO_IMPLICIT_PRECOMP_GEMM_SLICED (Forward / BackwardData): the same
// kernels over slices of the reduction channels, bounded operand copy
bool precomp_sliced_supports(int op, const ConvShape& s);
std::int64_t precomp_sliced_workspace(int op, const ConvShape& s);
cudaError_t precomp_sliced_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws,
                               float alpha, float beta, cudaStream_t stream);

void precomp_profile(double out[4]);

// x (NCHW) -> xs[n][i][j][Cp], channel (a*Bw + b)*C + c holding
// x[n][c][i*sh + a - ph][j*sw + b - pw] (zero off the image and for padded channels)
cudaError_t space_to_depth_nhwc(const float* x, float* out, int N, int C, int H, int W, int sh, int sw, int ph,
                                int pw, int Ah, int Bw, int Hq, int Wq, int Cp, cudaStream_t st);

}  // namespace ucudnn
