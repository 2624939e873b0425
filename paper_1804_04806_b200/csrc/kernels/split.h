// fp32 -> TF32 hi / lo operand split (FP32-faithful math mode; see split.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace ucudnn {

cudaError_t split_tf32(const float* in, float* hi, float* lo, std::int64_t n, cudaStream_t stream);

}  // namespace ucudnn
