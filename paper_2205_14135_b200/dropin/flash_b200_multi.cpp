// flash_b200_multi.cpp — see flash_b200_multi.hpp.
#include "flash_b200_multi.hpp"

#include <cuda_runtime.h>

#include <exception>
#include <stdexcept>
#include <thread>

namespace tatn::b200 {

int device_count() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

namespace {

// [start, end) of n items for worker w of W: contiguous, sizes differ by <= 1 (launcher.shard_range)
void shard(std::size_t n, int W, int w, std::size_t& start, std::size_t& end) {
  const std::size_t base = n / W, extra = n % W;
  start = w * base + std::min<std::size_t>(w, extra);
  end = start + base + (static_cast<std::size_t>(w) < extra ? 1 : 0);
}

// run body(worker, start, end, local_mem) on W threads, one per worker, then merge the counters
template <typename Body>
void run_sharded(std::size_t n, int workers, std::size_t m_capacity, MemoryModel& mem, Body body) {
  const int ndev = device_count();
  if (ndev < 1) throw std::runtime_error("tatn b200: no CUDA device for the sharded engines");
  const int W = static_cast<int>(std::max<std::size_t>(1, std::min<std::size_t>(n, workers > 0 ? workers : ndev)));
  std::vector<MemoryModel> local;
  local.reserve(W);
  for (int w = 0; w < W; ++w) local.emplace_back(m_capacity, mem.element_bytes());
  std::vector<std::exception_ptr> err(W);
  std::vector<std::thread> th;
  for (int w = 0; w < W; ++w)
    th.emplace_back([&, w] {
      try {
        if (cudaSetDevice(w % ndev) != cudaSuccess) throw std::runtime_error("tatn b200: cudaSetDevice failed");
        std::size_t s, e;
        shard(n, W, w, s, e);
        body(w, s, e, local[w]);
      } catch (...) {
        err[w] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
  for (auto& m : local) mem.counter().merge(m.counter());  // AccessCounter::merge (counters.cpp:8-13)
}

}  // namespace

std::vector<FlashSaved> flash_forward_sharded(const std::vector<HeadProblem>& heads, const TilePlan& plan,
                                              MemoryModel& mem, int workers) {
  std::vector<FlashSaved> out(heads.size());
  run_sharded(heads.size(), workers, plan.m_capacity, mem, [&](int, std::size_t s, std::size_t e, MemoryModel& m) {
    for (std::size_t i = s; i < e; ++i) out[i] = flash_forward(*heads[i].q, *heads[i].k, *heads[i].v, heads[i].cfg, plan, m);
  });
  return out;
}

std::vector<Gradients> flash_backward_sharded(const std::vector<FlashSaved>& saved,
                                              const std::vector<HeadProblem>& heads,
                                              const std::vector<const Matrix*>& d_o, MemoryModel& mem,
                                              int workers) {
  if (saved.size() != heads.size() || d_o.size() != heads.size())
    throw std::invalid_argument("flash_backward_sharded: saved / heads / d_o sizes differ");
  std::vector<Gradients> out(heads.size());
  const std::size_t cap = heads.empty() ? 1 : saved[0].plan.m_capacity;
  run_sharded(heads.size(), workers, cap, mem, [&](int, std::size_t s, std::size_t e, MemoryModel& m) {
    for (std::size_t i = s; i < e; ++i) out[i] = flash_backward(saved[i], *heads[i].q, *heads[i].k, *heads[i].v, *d_o[i], m);
  });
  return out;
}

}  // namespace tatn::b200
