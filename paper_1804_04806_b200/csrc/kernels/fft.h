// UCUDNN_ALGO_FFT: FFT-tiled stride-1 Forward / BackwardData (see fft.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "conv_common.h"

namespace ucudnn {

bool fft_supports(int op, const ConvShape& s);
std::int64_t fft_workspace(int op, const ConvShape& s);
cudaError_t fft_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                    float beta, cudaStream_t stream, int flags);

}  // namespace ucudnn
