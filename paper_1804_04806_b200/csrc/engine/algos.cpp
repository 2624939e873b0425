#include "algos.h"

#include <atomic>

#include "../kernels/gemm.h"
#include "../kernels/igemm.h"
#include "../kernels/precomp.h"

namespace ucudnn {

namespace {
std::atomic<std::uint64_t> g_launches{0};
}  // namespace
void count_launch(int n) { g_launches.fetch_add(std::uint64_t(n), std::memory_order_relaxed); }
std::uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

namespace {

bool igemm_supports(int, const ConvShape&) { return true; }
std::int64_t no_workspace(int, const ConvShape&) { return 0; }

cudaError_t igemm_run(int op, const ConvShape& s, const float* a, const float* b, float* out, void*, float alpha,
                      float beta, cudaStream_t st, int) {
  switch (op) {
    case 0: return igemm_forward(s, a, b, out, alpha, beta, st);
    case 1: return igemm_backward_data(s, a, b, out, alpha, beta, st);
    case 2: return igemm_backward_filter(s, a, b, out, alpha, beta, st);
  }
  return cudaErrorInvalidValue;
}

const AlgoImpl kImplicitGemm{0, "IMPLICIT_GEMM", igemm_supports, no_workspace, igemm_run};
const AlgoImpl kGemm{3, "GEMM", gemm_supports, gemm_workspace, gemm_run};
const AlgoImpl kPrecomp{5, "IMPLICIT_PRECOMP_GEMM", precomp_supports, precomp_workspace, precomp_run};

}  // namespace

const AlgoImpl* find_algo(int id) {
  switch (id) {
    case 0: return &kImplicitGemm;
    case 3: return &kGemm;
    case 5: return &kPrecomp;
    default: return nullptr;
  }
}

int algo_count() { return 6; }

}  // namespace ucudnn
