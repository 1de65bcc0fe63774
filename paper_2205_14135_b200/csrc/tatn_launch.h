// Kernel launches with programmatic dependent launch (PDL): each kernel of the path may be
// scheduled while its predecessor on the stream drains its last items; the kernel's own
// griddep_wait() (sm100_ptx.cuh) holds it before its first global-memory access. The step's
// four kernels (K1, K2, K3, K4) thereby overlap launch latency and prologues (TMEM allocation,
// barrier init, descriptor prefetch) with the previous kernel's tail. Captured into CUDA graphs
// as programmatic edges. TATN_PDL=0 in the environment launches them plainly (A/B).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace tatn_host {

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TATN_PDL");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace tatn_host
