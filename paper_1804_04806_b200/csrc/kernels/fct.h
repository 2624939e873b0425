// Few-channel strided layers with the im2col operand built in tensor memory
// (see fct.cu).
#pragma once

#include <cuda_runtime.h>

#include "conv_common.h"

namespace ucudnn {

bool fct_fwd_supports(const ConvShape& s);
// y = alpha * conv(x, w) + beta * y; no workspace
cudaError_t fct_fwd_run(const ConvShape& s, const float* x, const float* w, float* y, float alpha, float beta,
                        cudaStream_t stream);

bool fct_bwdf_supports(const ConvShape& s);
// per-CTA partial-sum slices (batch-independent)
std::int64_t fct_bwdf_workspace(const ConvShape& s);
// dw = beta * dw + alpha * sum; deterministic (slices added in a fixed order)
cudaError_t fct_bwdf_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha,
                         float beta, cudaStream_t stream);

bool fct_bwdd_supports(const ConvShape& s);
// dx = alpha * conv_bwd_data(dy, w) + beta * dx; no workspace
cudaError_t fct_bwdd_run(const ConvShape& s, const float* dy, const float* w, float* dx, float alpha, float beta,
                         cudaStream_t stream);

// stride-1 BackwardFilter of many-channel layers (W % 4 == 0, K <= 128), operands by TMA
bool fct_bwdf1_supports(const ConvShape& s);
std::int64_t fct_bwdf1_workspace(const ConvShape& s);
cudaError_t fct_bwdf1_run(const ConvShape& s, const float* x, const float* dy, float* dw, void* ws, float alpha,
                          float beta, cudaStream_t stream);

// stride-1 Forward / BackwardData with the im2col operand in TMEM (fct1.cu):
// input channels % 32 == 0, output width <= 128, <= 256 output channels
bool fct1_supports(int op, const ConvShape& s);
std::int64_t fct1_workspace(int op, const ConvShape& s);  // BackwardData: the flipped filter
cudaError_t fct1_run(int op, const ConvShape& s, const float* in, const float* w, float* out, void* ws, float alpha,
                     float beta, cudaStream_t stream, int flags);

}  // namespace ucudnn
