// Which cuTensorMapEncodeTiled parameter sets accept an element stride of 2
// along the innermost dimension (1x1 stride-2 Forward boxes)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/tmap_probe scripts/tmap_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
int main() {
  float* x;
  cudaMalloc(&x, 64ull << 20);
  const int W = 56, H = 56, C = 256, N = 4;
  cuuint64_t dims[4] = {cuuint64_t(W), cuuint64_t(H), cuuint64_t(C), cuuint64_t(N)};
  cuuint64_t strides[3] = {cuuint64_t(W) * 4, cuuint64_t(H) * W * 4, cuuint64_t(C) * H * W * 4};
  struct V { unsigned bx, es0; CUtensorMapSwizzle sw; const char* name; } vs[] = {
      {64, 2, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, "box64 es2 sw128_32B"},
      {32, 2, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, "box32 es2 sw128_32B"},
      {64, 2, CU_TENSOR_MAP_SWIZZLE_NONE, "box64 es2 none"},
      {64, 2, CU_TENSOR_MAP_SWIZZLE_128B, "box64 es2 sw128"},
      {32, 1, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, "box32 es1 sw128_32B"},
      {64, 2, CU_TENSOR_MAP_SWIZZLE_64B, "box64 es2 sw64"},
  };
  for (auto& v : vs) {
    CUtensorMap m;
    cuuint32_t box[4] = {v.bx, 1, 32, 1};
    cuuint32_t es[4] = {v.es0, 1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, v.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const char* s = nullptr;
    cuGetErrorString(r, &s);
    std::printf("%-24s -> %d %s\n", v.name, int(r), s ? s : "");
  }
  return 0;
}
