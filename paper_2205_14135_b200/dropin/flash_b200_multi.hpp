// flash_b200_multi.hpp — the reference's concurrency model across GPUs (C++ drop-in side).
//
// The reference runs independent (batch, head) problems, each with its own MemoryModel, and combines
// the counters afterwards with AccessCounter::merge (counters.cpp:8-13). These
// entry points do exactly that over the GPUs of one box: heads are split into contiguous, balanced
// ranges (launcher.shard_range's rule), one host thread per worker runs the drop-in's
// flash_forward / flash_backward on its device (worker w uses device w % cudaGetDeviceCount, so
// more workers than devices share them), each with a private MemoryModel, and the per-worker
// counters are merged into the caller's model. No data crosses devices: there is no collective.
#pragma once

#include <vector>

#include "tatn/flash.hpp"

namespace tatn::b200 {

struct HeadProblem {
  const Matrix* q;
  const Matrix* k;
  const Matrix* v;
  AttnConfig cfg;
};

// number of CUDA devices visible to the process (0 without a driver / device)
int device_count();

// flash_forward over every head; workers <= 0 means one per visible device
std::vector<FlashSaved> flash_forward_sharded(const std::vector<HeadProblem>& heads, const TilePlan& plan,
                                              MemoryModel& mem, int workers = 0);

// flash_backward over every head (saved[i] from the forward of heads[i]; d_o[i] its upstream gradient)
std::vector<Gradients> flash_backward_sharded(const std::vector<FlashSaved>& saved,
                                              const std::vector<HeadProblem>& heads,
                                              const std::vector<const Matrix*>& d_o, MemoryModel& mem,
                                              int workers = 0);

}  // namespace tatn::b200
