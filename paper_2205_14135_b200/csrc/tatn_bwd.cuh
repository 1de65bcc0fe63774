// tatn_bwd.cuh — placeholder until the backward kernels land.
#pragma once
#include <cuda_runtime.h>
#include "../../include/tatn_b200.h"
#include "tatn_params.h"

static inline int tatn_bwd_launch(const tatn_attn_desc&, const void*, const void*, const void*, const void*,
                                  const void*, const float*, void*, void*, void*, void*, cudaStream_t, int*) {
  return TATN_E_UNSUPPORTED;
}
