// TEST INFRASTRUCTURE ONLY -- the reference fp64 convolution, exported as C.
//
// Wraps the unmodified reference_conv.hpp (/root/reference/proj/include/
// ubatch/reference_conv.hpp:28-278) so Python tests can (a) pin the plain-C
// oracle (oracle/conv_oracle.c) against the reference itself and (b) time the
// reference CPU path for bench.py's cpu_baseline / --impl reference arm.
// Built by `make -C oracle ref` into oracle/_ref/ref_conv.so.
#include <cstring>

#include "ubatch/parallel.hpp"
#include "ubatch/reference_conv.hpp"

using namespace ubatch;

namespace {
Tensor4 wrap(const double* p, long long n, long long c, long long h, long long w) {
  Tensor4 t = Tensor4::zeros(n, c, h, w);
  if (p) std::memcpy(t.data.data(), p, sizeof(double) * t.data.size());
  return t;
}
KernelDescriptor kdesc(int op, const long long* s) {
  KernelDescriptor k;
  k.op_type = OpType(op);
  k.batch = s[0]; k.in_channels = s[1]; k.height = s[2]; k.width = s[3];
  k.out_channels = s[4]; k.kernel_h = s[5]; k.kernel_w = s[6];
  k.pad_h = s[7]; k.pad_w = s[8]; k.stride_h = s[9]; k.stride_w = s[10];
  k.layer_name = "ref";
  return k;
}
}  // namespace

extern "C" {

// shape = {N, C, H, W, K, R, S, pad_h, pad_w, stride_h, stride_w}
// op 0 Forward (a = x, b = w) -> y; 1 BackwardData (a = dy, b = w) -> dx;
// 2 BackwardFilter (a = x, b = dy) -> dw. micro_batches[n_micro] gives the
// plan's micro-batch sizes (any order; execute_plan runs them canonically).
int ref_execute_plan(int op, const long long* shape, const long long* micro_batches, int n_micro,
                     const double* a, const double* b, double* out) {
  try {
    KernelDescriptor k = kdesc(op, shape);
    long long oh = k.out_height(), ow = k.out_width();
    std::vector<MicroConfiguration> ms;
    for (int i = 0; i < n_micro; ++i) ms.push_back(MicroConfiguration{AlgorithmId{0}, micro_batches[i], Rat64(0), 0});
    Configuration cfg(ms);
    Tensor4 ta, tb;
    if (op == 0) {
      ta = wrap(a, k.batch, k.in_channels, k.height, k.width);
      tb = wrap(b, k.out_channels, k.in_channels, k.kernel_h, k.kernel_w);
    } else if (op == 1) {
      ta = wrap(a, k.batch, k.out_channels, oh, ow);
      tb = wrap(b, k.out_channels, k.in_channels, k.kernel_h, k.kernel_w);
    } else {
      ta = wrap(a, k.batch, k.in_channels, k.height, k.width);
      tb = wrap(b, k.batch, k.out_channels, oh, ow);
    }
    Tensor4 r = execute_plan(k, cfg, ta, tb);
    std::memcpy(out, r.data.data(), sizeof(double) * r.data.size());
    return 0;
  } catch (...) {
    return 1;
  }
}

// The reference conv loops over `threads` contiguous batch slices via the
// reference's own parallel_for (parallel.hpp:28-56); BackwardFilter slices
// accumulate privately and are summed. This is the all-cores CPU baseline.
int ref_conv_threads(int op, const long long* shape, const double* a, const double* b, double* out,
                     int threads) {
  try {
    KernelDescriptor k = kdesc(op, shape);
    long long N = k.batch, oh = k.out_height(), ow = k.out_width();
    long long per = (N + threads - 1) / threads;
    long long a_ss = op == 1 ? k.out_channels * oh * ow : k.in_channels * k.height * k.width;
    long long b_ss = op == 2 ? k.out_channels * oh * ow : 0;
    long long o_ss = op == 0 ? k.out_channels * oh * ow : (op == 1 ? k.in_channels * k.height * k.width : 0);
    std::vector<Tensor4> partial(static_cast<std::size_t>(threads));
    Tensor4 f;
    if (op != 2) f = wrap(b, k.out_channels, k.in_channels, k.kernel_h, k.kernel_w);
    parallel_for(std::size_t(threads), unsigned(threads), [&](std::size_t t) {
      long long lo = (long long)t * per, hi = std::min(N, lo + per);
      if (lo >= hi) return;
      long long n = hi - lo;
      if (op == 0) {
        Tensor4 x = wrap(a + lo * a_ss, n, k.in_channels, k.height, k.width);
        Tensor4 y = conv_forward(x, f, k.pad_h, k.pad_w, k.stride_h, k.stride_w);
        std::memcpy(out + lo * o_ss, y.data.data(), sizeof(double) * y.data.size());
      } else if (op == 1) {
        Tensor4 dy = wrap(a + lo * a_ss, n, k.out_channels, oh, ow);
        Tensor4 dx = conv_backward_data(dy, f, k.pad_h, k.pad_w, k.stride_h, k.stride_w, k.height, k.width);
        std::memcpy(out + lo * o_ss, dx.data.data(), sizeof(double) * dx.data.size());
      } else {
        Tensor4 x = wrap(a + lo * a_ss, n, k.in_channels, k.height, k.width);
        Tensor4 dy = wrap(b + lo * b_ss, n, k.out_channels, oh, ow);
        partial[t] = conv_backward_filter(x, dy, k.pad_h, k.pad_w, k.stride_h, k.stride_w, k.kernel_h,
                                          k.kernel_w);
      }
    });
    if (op == 2) {
      long long cnt = k.out_channels * k.in_channels * k.kernel_h * k.kernel_w;
      std::memset(out, 0, sizeof(double) * cnt);
      for (auto& p : partial)
        if (!p.data.empty())
          for (long long i = 0; i < cnt; ++i) out[i] += p.data[i];
    }
    return 0;
  } catch (...) {
    return 1;
  }
}
}
