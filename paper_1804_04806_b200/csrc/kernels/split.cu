// fp32 -> (hi, lo) TF32 operand split for the FP32-faithful math mode
// (ucudnnSetMathMode): hi = v with its low 13 mantissa bits cleared (exactly
// representable in TF32, so the tensor core multiplies it exactly), lo = v -
// hi (exact in fp32). A convolution is bilinear, so
//   conv(a, b) = conv(a_hi, b_hi) + conv(a_lo, b_hi) + conv(a_hi, b_lo) + conv(a_lo, b_lo)
// and dropping the last term (|a_lo b_lo| <= 2^-20 |a b|) leaves an error of
// fp32 order instead of TF32's 2^-11 ("3xTF32").
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "conv_common.h"
#include "split.h"

namespace ucudnn {

namespace {
__global__ void split_kernel(const float* __restrict__ in, float* __restrict__ hi, float* __restrict__ lo,
                             std::int64_t n) {
  for (std::int64_t i = blockIdx.x * std::int64_t(blockDim.x) + threadIdx.x; i < n;
       i += std::int64_t(gridDim.x) * blockDim.x) {
    const float v = in[i];
    const float h = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
    hi[i] = h;
    lo[i] = v - h;
  }
}
}  // namespace

cudaError_t split_tf32(const float* in, float* hi, float* lo, std::int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  count_launch();
  const int blocks = int(std::min<std::int64_t>((n + 255) / 256, 148 * 16));
  split_kernel<<<blocks, 256, 0, st>>>(in, hi, lo, n);
  return cudaGetLastError();
}

}  // namespace ucudnn
