// UCUDNN_ALGO_GEMM (explicit im2col / col2im + tiled tcgen05 GEMM; see gemm.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "conv_common.h"

namespace ucudnn {

bool gemm_supports(int op, const ConvShape& s);
std::int64_t gemm_workspace(int op, const ConvShape& s);
cudaError_t gemm_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void* ws, float alpha,
                     float beta, cudaStream_t stream, int flags);

// Blocked operand layout of the tiled tcgen05 GEMM (shared with Winograd):
// A = [m_tile][kstep] blocks of 128 rows x 32, B = [n_tile][kstep] blocks of
// BN rows x 32, each block stored as [8 k-groups][rows][4 floats].
int blocked_bn(int n);
// batch independent GEMMs out_b[col * ld + row] = sum_k A_b[row][k] B_b[col][k]
// (rows M, cols Nc, reduction Kr), operands in the blocked layout above.
cudaError_t batched_gemm_colmajor(int batch, int M, int Nc, int Kr, const float* a, std::int64_t a_bs, const float* b,
                                  std::int64_t b_bs, float* out, std::int64_t o_bs, int ld, cudaStream_t st);

}  // namespace ucudnn
