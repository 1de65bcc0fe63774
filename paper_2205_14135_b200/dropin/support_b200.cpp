// support_b200.cpp — the reference's host-side tiling/IO/block-mask operators
// whose sources are absent from the reference tree (proj/core/CMakeLists.txt:10-13
// lists tile_plan.cpp, block_mask.cpp and io_predict.cpp, none of which ship).
// Implemented here against the reference's own headers so the drop-in library
// is a complete tatn_core: tile_plan.hpp:22-52, block_mask.hpp:26-46,
// io_predict.hpp:12-119 (counting rules in its header comment).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>

#include "tatn/block_mask.hpp"
#include "tatn/io_predict.hpp"
#include "tatn/tile_plan.hpp"

namespace tatn {

// ------------------------------------------------------------------ tile_plan.hpp
std::size_t working_set_elems(std::size_t br, std::size_t bc, std::size_t d) {
  return 2 * bc * d + 2 * br * d + br * bc + 6 * br;
}

std::size_t backward_working_set_elems(std::size_t br, std::size_t bc, std::size_t d) {
  return 4 * bc * d + 4 * br * d + 2 * br * bc + 3 * br;
}

namespace {
std::size_t cdiv(std::size_t a, std::size_t b) { return (a + b - 1) / b; }

bool default_plan_fits(std::size_t n, std::size_t d, std::size_t m) {
  if (m < 4 * d) return false;
  std::size_t bc = std::min(cdiv(m, 4 * d), n);
  std::size_t br = std::min(std::min(cdiv(m, 4 * d), d), n);
  return static_cast<double>(working_set_elems(br, bc, d)) <= kSramSlackForward * static_cast<double>(m);
}
}  // namespace

std::size_t min_feasible_m(std::size_t n, std::size_t d) {
  // Smallest M >= 4d whose default plan passes the forward check; the check is
  // not monotone in M once the block sizes clamp to n, so scan (at most ~3 d^2 steps).
  for (std::size_t m = 4 * d;; ++m)
    if (default_plan_fits(n, d, m)) return m;
}

TilePlan plan_tiles(std::size_t n, std::size_t d, std::size_t m_capacity, const TileOverrides& overrides) {
  if (n < 1 || d < 1) throw std::invalid_argument("plan_tiles: n and d must be >= 1");
  if (m_capacity < 4 * d)
    throw std::invalid_argument("plan_tiles: M=" + std::to_string(m_capacity) + " < 4d; minimum feasible M is " +
                                std::to_string(min_feasible_m(n, d)));
  TilePlan p;
  p.bc = overrides.bc.value_or(cdiv(m_capacity, 4 * d));
  p.br = overrides.br.value_or(std::min(cdiv(m_capacity, 4 * d), d));
  if (p.bc < 1 || p.br < 1) throw std::invalid_argument("plan_tiles: block sizes must be >= 1");
  p.bc = std::min(p.bc, n);
  p.br = std::min(p.br, n);
  p.tr = cdiv(n, p.br);
  p.tc = cdiv(n, p.bc);
  p.m_capacity = m_capacity;
  p.working_set = working_set_elems(p.br, p.bc, d);
  if (static_cast<double>(p.working_set) > kSramSlackForward * static_cast<double>(m_capacity))
    throw std::invalid_argument("plan_tiles: working set " + std::to_string(p.working_set) + " exceeds 1.5*M=" +
                                std::to_string(static_cast<std::uint64_t>(kSramSlackForward * m_capacity)) +
                                "; minimum feasible M is " + std::to_string(min_feasible_m(n, d)));
  return p;
}

// ------------------------------------------------------------------ block_mask.hpp
std::size_t BlockMask::count_true() const {
  return static_cast<std::size_t>(std::count_if(grid.begin(), grid.end(), [](std::uint8_t x) { return x != 0; }));
}

namespace {
BlockMask empty_mask(std::size_t tr, std::size_t tc, std::size_t br, std::size_t bc) {
  if (tr < 1 || tc < 1) throw std::invalid_argument("make_block_mask: tr, tc must be >= 1");
  BlockMask m;
  m.tr = tr;
  m.tc = tc;
  m.br = br;
  m.bc = bc;
  m.grid.assign(tr * tc, 0);
  return m;
}
void finish(BlockMask& m) { m.density = static_cast<double>(m.count_true()) / static_cast<double>(m.tr * m.tc); }
}  // namespace

BlockMask make_block_mask_random(double s, std::uint64_t seed, std::size_t tr, std::size_t tc, std::size_t br,
                                 std::size_t bc) {
  if (!(s >= 0.0 && s <= 1.0)) throw std::invalid_argument("make_block_mask_random: s must be in [0, 1]");
  BlockMask m = empty_mask(tr, tc, br, bc);
  const std::size_t total = tr * tc;
  const auto k = static_cast<std::size_t>(std::llround(s * static_cast<double>(total)));
  // Uniform k-subset without replacement: partial Fisher-Yates on mt19937_64.
  // (The reference's generator for this op is unspecified: block_mask.cpp is absent.)
  std::vector<std::size_t> idx(total);
  std::iota(idx.begin(), idx.end(), std::size_t{0});
  std::mt19937_64 rng(seed);
  for (std::size_t i = 0; i < k; ++i) {
    std::uniform_int_distribution<std::size_t> pick(i, total - 1);
    std::swap(idx[i], idx[pick(rng)]);
    m.grid[idx[i]] = 1;
  }
  finish(m);
  return m;
}

BlockMask make_block_mask_butterfly(std::size_t tr, std::size_t tc, std::size_t br, std::size_t bc) {
  BlockMask m = empty_mask(tr, tc, br, bc);
  for (std::size_t i = 0; i < tr; ++i)
    for (std::size_t j = 0; j < tc; ++j) {
      const std::size_t x = i ^ j;
      m.grid[i * tc + j] = (x == 0 || (x & (x - 1)) == 0) ? 1 : 0;
    }
  finish(m);
  return m;
}

BlockMask make_block_mask_local_global(std::size_t window, std::size_t globals, std::size_t tr, std::size_t tc,
                                       std::size_t br, std::size_t bc) {
  BlockMask m = empty_mask(tr, tc, br, bc);
  for (std::size_t i = 0; i < tr; ++i)
    for (std::size_t j = 0; j < tc; ++j) {
      const std::size_t dist = i > j ? i - j : j - i;
      m.grid[i * tc + j] = (dist <= window || i < globals || j < globals) ? 1 : 0;
    }
  finish(m);
  return m;
}

MaskSpec compose_block_mask(const MaskSpec& base, const BlockMask& bmask, std::size_t n) {
  if (bmask.br < 1 || bmask.bc < 1 || bmask.tr * bmask.br < n || bmask.tc * bmask.bc < n ||
      bmask.grid.size() != bmask.tr * bmask.tc)
    throw std::invalid_argument("compose_block_mask: block grid does not cover n x n");
  const double ninf = -std::numeric_limits<double>::infinity();
  Matrix pat(n, n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j)
      pat(i, j) = (bmask.at(i / bmask.br, j / bmask.bc) && !is_masked(base, i, j)) ? 0.0 : ninf;
  return MaskSpec::custom_additive(std::move(pat));
}

// ------------------------------------------------------------------ io_predict.hpp
IoPrediction predict_standard_forward_io(std::size_t n, std::size_t d) {
  return {3 * n * d + 4 * n * n, 2 * n * n + n * d, "standard_forward"};
}

IoPrediction predict_standard_backward_io(std::size_t n, std::size_t d) {
  return {7 * n * n + 5 * n * d, 2 * n * n + 3 * n * d, "standard_backward"};
}

IoPrediction predict_flash_forward_io(std::size_t n, std::size_t d, const TilePlan& plan) {
  const std::uint64_t tc = plan.tc;
  return {2 * n * d + tc * (2 * n * d + 2 * n), (n * d + 2 * n) + tc * (n * d + 2 * n), "flash_forward"};
}

IoPrediction predict_flash_backward_io(std::size_t n, std::size_t d, const TilePlan& plan) {
  const std::uint64_t tc = plan.tc;
  return {2 * n * d + tc * (4 * n * d + 2 * n), n * d + tc * n * d + 2 * n * d, "flash_backward"};
}

namespace {
std::uint64_t visited_blocks(const TilePlan& plan, double s) {
  if (!(s >= 0.0 && s <= 1.0)) throw std::invalid_argument("predict_blocksparse_io: s must be in [0, 1]");
  return static_cast<std::uint64_t>(std::llround(s * static_cast<double>(plan.tr * plan.tc)));
}
}  // namespace

IoPrediction predict_blocksparse_io(std::size_t n, std::size_t d, const TilePlan& plan, double s) {
  const std::uint64_t v = visited_blocks(plan, s), br = plan.br;
  return {2 * n * d + v * (2 * br * d + 2 * br), (n * d + 2 * n) + v * (br * d + 2 * br), "blocksparse_forward"};
}

IoPrediction predict_blocksparse_backward_io(std::size_t n, std::size_t d, const TilePlan& plan, double s) {
  const std::uint64_t v = visited_blocks(plan, s), br = plan.br;
  return {2 * n * d + v * (4 * br * d + 2 * br), n * d + v * br * d + 2 * n * d, "blocksparse_backward"};
}

std::uint64_t flop_model(AlgoId algo, std::size_t n, std::size_t d, const TilePlan* plan, double density) {
  const std::uint64_t N = n, D = d;
  auto need_plan = [&]() -> const TilePlan& {
    if (plan == nullptr) throw std::invalid_argument("flop_model: the tiled algorithms need a plan");
    return *plan;
  };
  switch (algo) {
    case AlgoId::StandardForward: return 4 * N * N * D + 5 * N * N;
    case AlgoId::StandardBackward: return 8 * N * N * D + 4 * N * N + 2 * N * D;
    case AlgoId::FlashForward: {
      const auto& p = need_plan();
      return 4 * N * N * D + 5 * N * N + p.tc * (2 * N * D + 7 * N);
    }
    case AlgoId::FlashBackward: {
      const auto& p = need_plan();
      return 10 * N * N * D + 5 * N * N + 4 * p.tc * N * D + 2 * p.tr * N * D;
    }
    case AlgoId::BlockSparseForward: {
      const auto& p = need_plan();
      const std::uint64_t v = visited_blocks(p, density), br = p.br, bc = p.bc;
      return v * (4 * br * bc * D + 5 * br * bc + 2 * br * D + 7 * br);
    }
    case AlgoId::BlockSparseBackward: {
      const auto& p = need_plan();
      const std::uint64_t v = visited_blocks(p, density), br = p.br, bc = p.bc;
      return v * (10 * br * bc * D + 5 * br * bc + 4 * br * D + 2 * bc * D);
    }
  }
  throw std::invalid_argument("flop_model: unknown algorithm id");
}

ByteReport byte_report(std::uint64_t read_elems, std::uint64_t write_elems, std::uint32_t element_bytes,
                       std::uint64_t multiplier) {
  return {read_elems * element_bytes * multiplier, write_elems * element_bytes * multiplier};
}

ByteReport byte_report(const AccessCounter& counter, std::uint32_t element_bytes, std::uint64_t multiplier) {
  return byte_report(counter.hbm_read_elems, counter.hbm_write_elems, element_bytes, multiplier);
}

}  // namespace tatn
