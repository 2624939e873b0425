// Device algorithm entry points (all launch on `stream`, no host sync).
// Pointers address the micro-batch slice; alpha/beta follow cuDNN:
// out = alpha * conv + beta * out (beta == 0 never reads out).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "conv_common.h"

namespace ucudnn {

// IMPLICIT_GEMM (0 workspace).
cudaError_t igemm_forward(const ConvShape& s, const float* x, const float* w, float* y, float alpha, float beta,
                          cudaStream_t stream);
cudaError_t igemm_backward_data(const ConvShape& s, const float* dy, const float* w, float* dx, float alpha,
                                float beta, cudaStream_t stream);
// dw = beta * dw + alpha * sum (split-K with fp32 atomics)
cudaError_t igemm_backward_filter(const ConvShape& s, const float* x, const float* dy, float* dw, float alpha,
                                  float beta, cudaStream_t stream);

cudaError_t scale_tensor(float* p, std::int64_t n, float beta, cudaStream_t stream);

// The tcgen05 implicit GEMM with cp.async-gathered operands (igemm_tc.cu),
// Forward and BackwardData; igemm_* dispatch to it for the shapes it takes
// (taps <= 32 per axis, 32-bit offsets) and keep the SIMT-gather kernel
// below as the fallback that makes algorithm 0 total.
bool zgemm_supports(int op, const ConvShape& s);
cudaError_t zgemm_forward(const ConvShape& s, const float* x, const float* w, float* y, float alpha, float beta,
                          cudaStream_t stream);
cudaError_t zgemm_backward_data(const ConvShape& s, const float* dy, const float* w, float* dx, float alpha,
                                float beta, cudaStream_t stream);

}  // namespace ucudnn
