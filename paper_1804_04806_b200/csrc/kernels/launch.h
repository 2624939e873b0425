// Kernel launch with optional programmatic dependent launch (PDL,
// UCUDNN_TUNE=pdl=1; off by default -- it measured slightly slower on the
// graph-replayed AlexNet step): the kernel
// may be scheduled while the previous kernel on the stream drains, overlapping
// its prologue (barrier init, TMEM allocation, tensor-map prefetch) and the
// launch latency; the kernel itself calls sm100::pdl_wait() before touching
// global memory. Also captured as a programmatic edge inside CUDA graphs.
#pragma once

#include <cuda_runtime.h>

#include <utility>

#include "conv_common.h"

namespace ucudnn {

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t st,
                       Args&&... args) {
  count_launch();
  if (!tune("pdl", 0)) {  // A/B on the AlexNet step: 5.37 (off) vs 5.49 ms (on)
    kernel<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, KArgs(std::forward<Args>(args))...);
}

}  // namespace ucudnn
