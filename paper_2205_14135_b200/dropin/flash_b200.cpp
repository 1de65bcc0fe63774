// flash_b200.cpp — the reference's tiled engine (proj/core/include/tatn/flash.hpp:43-73),
// implemented on the B200 C ABI (include/tatn_b200.h). This is the file a
// maintainer adds to tatn_core in place of the absent src/flash.cpp
// (proj/core/CMakeLists.txt:12); see INTEGRATION.md.
//
// Per call (one head, fp64 n x d matrices):
//   * validate like the reference (AttnConfig::validate, shape / plan / mask checks);
//   * round Q, K, V (and dO) to the device input type — bf16 (default) or fp16 with
//     round-to-nearest-even, or fp32 (the tf32 check mode, set_input_dtype) — and zero-pad d
//     to 64 or 128 (zero columns change neither QK^T nor the live O columns);
//   * run tatn_fwd / tatn_bwd with fp32 outputs (no output rounding);
//   * return O and the stats as (m = LSE, l = 1) — the same (m, l) pair up to
//     the representation m + ln l (fully-masked rows stay (-inf, 0), which
//     SoftmaxStats::validate accepts, softmax.cpp:17-28);
//   * charge the MemoryModel with the exact element counts of the reference's
//     tiled schedule for `plan` (io_predict.hpp counting rules, per visited
//     block for the block-sparse engines) and lease plan.working_set.
// Dropout follows the reference's positional generator bit for bit (the mask at
// (i, j) is a pure function of (seed, i, j), dropout.hpp:14-30), so forward and
// backward regenerate identical masks. There is no CPU fallback: unsupported
// inputs (d > 128) throw, and a missing sm_100 device surfaces as std::runtime_error.
// Custom n x n masks are bit-packed into the ABI's keep matrix. Block masks of any
// block size (the plan's br x bc) run on the kernels' 128 x 128 tiles:
// a tile is visited iff a true block overlaps it, and when br or bc is not a multiple
// of 128 the blocks' element pattern (compose_block_mask) is applied inside the tiles
// through the same keep-bit path.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "tatn/flash.hpp"
#include "tatn/io_predict.hpp"
#include "tatn_b200.h"

namespace tatn {
namespace b200 {

// Input dtype of the device path: bf16 (default), fp16 (3 more mantissa bits) or fp32 (inputs
// kept at binary32 and multiplied as tf32 on the tensor cores: the closest the device gets to
// the reference's binary64).
static int g_input_dtype = TATN_DTYPE_BF16;
void set_input_dtype(int dtype) {
  if (dtype != TATN_DTYPE_BF16 && dtype != TATN_DTYPE_FP16 && dtype != TATN_DTYPE_FP32)
    throw std::invalid_argument("tatn b200: input dtype must be TATN_DTYPE_BF16, _FP16 or _FP32");
  g_input_dtype = dtype;
}
void set_input_dtype_fp16(bool fp16) { g_input_dtype = fp16 ? TATN_DTYPE_FP16 : TATN_DTYPE_BF16; }

namespace {

constexpr double kNegInf = -std::numeric_limits<double>::infinity();

uint16_t round16(double x, int dtype) {
  const float f = static_cast<float>(x);  // RNE to binary32 first, as torch and the oracle do
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if (dtype == TATN_DTYPE_BF16) {
    if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>(u >> 16);  // inf
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
  }
  // binary16 RNE via the hardware-independent path
  const uint32_t sign = (u >> 16) & 0x8000u;
  int32_t exp = static_cast<int32_t>((u >> 23) & 0xff) - 127 + 15;
  uint32_t man = u & 0x7fffffu;
  if (((u >> 23) & 0xff) == 0xff) return static_cast<uint16_t>(sign | 0x7c00u);
  if (exp >= 31) return static_cast<uint16_t>(sign | 0x7c00u);  // overflow -> inf (caller checks)
  if (exp <= 0) {                                               // subnormal or zero
    if (exp < -10) return static_cast<uint16_t>(sign);
    man |= 0x800000u;
    const uint32_t shift = static_cast<uint32_t>(14 - exp);
    uint32_t half = man >> shift;
    const uint32_t rem = man & ((1u << shift) - 1u), mid = 1u << (shift - 1);
    if (rem > mid || (rem == mid && (half & 1u))) ++half;
    return static_cast<uint16_t>(sign | half);
  }
  uint32_t h = sign | (static_cast<uint32_t>(exp) << 10) | (man >> 13);
  const uint32_t rem = man & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) ++h;
  return static_cast<uint16_t>(h);
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("tatn b200: ") + what + ": " + cudaGetErrorString(e));
}

void check_status(int st, const char* what) {
  if (st == TATN_OK) return;
  const std::string msg = std::string(what) + ": " + tatn_strerror(st);
  if (st == TATN_E_CUDA) throw std::runtime_error(msg);
  throw std::invalid_argument(msg);
}

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) {
    if (bytes) check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

int padded_d(std::size_t d) {
  if (d <= 64) return 64;
  if (d <= 128) return 128;
  throw std::invalid_argument("tatn b200: head dimension d > 128 is not supported on the sm_100a path");
}

// rows x d fp64 -> rows x dp 16-bit (zero padded), uploaded
void upload16(const Matrix& m, int dp, int dtype, void* dev) {
  std::vector<uint16_t> h(m.rows() * static_cast<size_t>(dp), 0);
  for (std::size_t i = 0; i < m.rows(); ++i)
    for (std::size_t j = 0; j < m.cols(); ++j) {
      const double x = m(i, j);
      if (!std::isfinite(x)) throw std::invalid_argument("tatn b200: non-finite input");
      h[i * dp + j] = round16(x, dtype);
    }
  check_cuda(cudaMemcpy(dev, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "upload");
}

void upload32(const Matrix& m, int dp, void* dev) {
  std::vector<float> h(m.rows() * static_cast<size_t>(dp), 0.f);
  for (std::size_t i = 0; i < m.rows(); ++i)
    for (std::size_t j = 0; j < m.cols(); ++j) h[i * dp + j] = static_cast<float>(m(i, j));
  check_cuda(cudaMemcpy(dev, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "upload");
}

// an input matrix in the device input dtype (fp32: RNE to binary32; else 16-bit RNE)
std::size_t in_bytes(int dtype) { return dtype == TATN_DTYPE_FP32 ? 4 : 2; }
void upload_in(const Matrix& m, int dp, int dtype, void* dev) {
  if (dtype == TATN_DTYPE_FP32) {
    for (std::size_t i = 0; i < m.rows(); ++i)
      for (std::size_t j = 0; j < m.cols(); ++j)
        if (!std::isfinite(static_cast<float>(m(i, j)))) throw std::invalid_argument("tatn b200: non-finite input");
    upload32(m, dp, dev);
  } else {
    upload16(m, dp, dtype, dev);
  }
}

Matrix download32(const void* dev, std::size_t rows, std::size_t cols, int dp) {
  std::vector<float> h(rows * static_cast<size_t>(dp));
  check_cuda(cudaMemcpy(h.data(), dev, h.size() * 4, cudaMemcpyDeviceToHost), "download");
  Matrix m(rows, cols);
  for (std::size_t i = 0; i < rows; ++i)
    for (std::size_t j = 0; j < cols; ++j) m(i, j) = h[i * dp + j];
  return m;
}

struct Problem {
  std::size_t n, nk, d;
  int dp;
  tatn_attn_desc desc;
};

void check_inputs(const char* op, const Matrix& q, const Matrix& k, const Matrix& v, const AttnConfig& cfg) {
  cfg.validate();  // throws std::invalid_argument (attn_config.cpp:42-58)
  if (q.rows() != cfg.n || q.cols() != cfg.d)
    throw std::invalid_argument(std::string(op) + ": Q must be n x d per config");
  if (k.cols() != cfg.d || v.cols() != cfg.d) throw std::invalid_argument(std::string(op) + ": K and V must have d columns");
  if (k.rows() != v.rows()) throw std::invalid_argument(std::string(op) + ": K and V row counts differ");
  if (k.rows() > cfg.n || k.rows() < 1) throw std::invalid_argument(std::string(op) + ": bad key count");
  if (has_nan(q) || has_nan(k) || has_nan(v)) throw std::invalid_argument(std::string(op) + ": NaN input");
}

void check_plan(const char* op, const TilePlan& plan, std::size_t n, std::size_t d) {
  if (plan.br < 1 || plan.bc < 1 || plan.tr != (n + plan.br - 1) / plan.br || plan.tc != (n + plan.bc - 1) / plan.bc)
    throw std::invalid_argument(std::string(op) + ": plan does not match n");
  if (static_cast<double>(working_set_elems(plan.br, plan.bc, d)) > kSramSlackForward * plan.m_capacity)
    throw std::invalid_argument(std::string(op) + ": plan working set exceeds 1.5*M (capacity violation)");
}

Problem make_problem(const Matrix& q, const Matrix& k, const AttnConfig& cfg) {
  Problem P{};
  P.n = q.rows();
  P.nk = k.rows();
  P.d = q.cols();
  P.dp = padded_d(P.d);
  tatn_attn_desc& d = P.desc;
  std::memset(&d, 0, sizeof d);
  d.B = 1;
  d.H = 1;
  d.Nq = static_cast<int32_t>(P.n);
  d.Nk = static_cast<int32_t>(P.nk);
  d.d = P.dp;
  d.dtype = g_input_dtype;
  d.out_dtype = TATN_OUT_FP32;
  const int64_t sq = static_cast<int64_t>(P.n) * P.dp, sk = static_cast<int64_t>(P.nk) * P.dp;
  d.q_str[0] = sq; d.q_str[1] = sq; d.q_str[2] = P.dp;
  d.o_str[0] = sq; d.o_str[1] = sq; d.o_str[2] = P.dp;
  d.k_str[0] = sk; d.k_str[1] = sk; d.k_str[2] = P.dp;
  d.v_str[0] = sk; d.v_str[1] = sk; d.v_str[2] = P.dp;
  d.tau = static_cast<float>(cfg.tau);
  d.mask_kind = cfg.mask.kind == MaskKind::Causal       ? TATN_MASK_CAUSAL
                : cfg.mask.kind == MaskKind::KeyPadding ? TATN_MASK_KEY_PADDING
                : cfg.mask.kind == MaskKind::Custom     ? TATN_MASK_CUSTOM
                                                        : TATN_MASK_NONE;
  d.tr = static_cast<int32_t>((P.n + 127) / 128);
  d.tc = static_cast<int32_t>((P.nk + 127) / 128);
  d.p_drop = cfg.p_drop;  // one head per call: slice 0 uses cfg.seed, i.e. the reference's mask
  d.seed = cfg.seed;
  // the reference's engines are pure functions of their inputs: dQ summed in a fixed
  // key-tile order, so repeated calls and an all-true block mask reproduce the dense dQ exactly
  d.deterministic = 1;
  return P;
}

// Map a BlockMask at the plan's block size (br x bc, any size >= 1) onto the kernels' 128 x 128
// tile grid: tile (I, J) is visited iff some true block overlaps it. The grid is exact — no
// element pattern needed inside the tiles — when every visited tile is covered by true blocks
// only (always so when br and bc are multiples of 128, and for an all-true mask); otherwise
// CustomMask carries the element pattern of the blocks.
struct TileGrid {
  std::vector<uint8_t> g;  // tr x tc at 128 x 128
  bool exact = true;
};
TileGrid tile_grid(const BlockMask& bm, std::size_t n, std::size_t nk) {
  if (bm.br == 0 || bm.bc == 0)
    throw std::invalid_argument("blocksparse: bmask block sizes must be positive");
  if (bm.grid.size() != bm.tr * bm.tc || bm.tr * bm.br < n || bm.tc * bm.bc < nk)
    throw std::invalid_argument("blocksparse: bmask does not cover the problem");
  const std::size_t tr = (n + 127) / 128, tc = (nk + 127) / 128;
  TileGrid t;
  t.g.assign(tr * tc, 0);
  std::vector<uint8_t> any_false(tr * tc, 0);
  for (std::size_t bi = 0; bi < bm.tr; ++bi) {
    const std::size_t r0 = bi * bm.br;
    if (r0 >= n) break;
    const std::size_t r1 = std::min(n, r0 + bm.br) - 1;
    for (std::size_t bj = 0; bj < bm.tc; ++bj) {
      const std::size_t c0 = bj * bm.bc;
      if (c0 >= nk) break;
      const std::size_t c1 = std::min(nk, c0 + bm.bc) - 1;
      for (std::size_t I = r0 / 128; I <= r1 / 128; ++I)
        for (std::size_t J = c0 / 128; J <= c1 / 128; ++J) (bm.at(bi, bj) ? t.g : any_false)[I * tc + J] = 1;
    }
  }
  for (std::size_t x = 0; x < t.g.size(); ++x) t.exact = t.exact && !(t.g[x] && any_false[x]);
  return t;
}

// Keep bits for the Custom path: bit-packed [n][words], words = ceil(nk / 128) * 4, uploaded;
// the descriptor points at it for the call's lifetime. Built when the mask is MaskKind::Custom
// (the n x n additive pattern, 0 keep / -inf mask, validated by AttnConfig::validate) and when a
// block mask must be applied per element: then keep(i, j) = !is_masked(base, i, j) and
// bmask(i / br, j / bc) — exactly compose_block_mask (block_mask.hpp:42-46) — and the call runs
// as a Custom mask (the base mask's causal / key-padding rule is folded into the bits).
struct CustomMask {
  bool on;
  DevBuf buf;
  int32_t words;
  CustomMask(const AttnConfig& cfg, std::size_t n, std::size_t nk, const BlockMask* bm, bool fine)
      : on(cfg.mask.kind == MaskKind::Custom || fine),
        buf(on ? n * ((nk + 127) / 128 * 4) * 4 : 0),
        words(static_cast<int32_t>((nk + 127) / 128 * 4)) {
    if (!on) return;
    std::vector<uint32_t> bits(n * static_cast<std::size_t>(words), 0u);
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = 0; j < nk; ++j) {
        bool keep = !is_masked(cfg.mask, i, j);
        if (fine) keep = keep && bm->at(i / bm->br, j / bm->bc);
        if (keep) bits[i * words + j / 32] |= 1u << (j % 32);
      }
    check_cuda(cudaMemcpy(buf.p, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice), "upload custom mask");
  }
  void attach(tatn_attn_desc& d) const {
    if (!on) return;
    d.mask_kind = TATN_MASK_CUSTOM;
    d.valid_len = nullptr;  // a key-padding base mask is in the bits
    d.custom_mask = static_cast<const uint32_t*>(buf.p);
    d.custom_words = words;
    d.custom_bstride = 0;
  }
};

// ---- MemoryModel charges: the reference's counting rules (io_predict.hpp:12-56),
// evaluated per (query block, key block) so that ragged shapes, key prefixes and
// block-sparse masks are exact and an all-true mask equals the dense charge.
struct Charges {
  std::uint64_t reads = 0, writes = 0, flops = 0;
};

Charges forward_charges(std::size_t n, std::size_t nk, std::size_t d, const TilePlan& plan, const BlockMask* bm) {
  Charges c;
  c.writes += n * d + 2 * n;  // init O, l, m
  c.reads += 2 * nk * d;      // K, V once
  const std::size_t tc = (nk + plan.bc - 1) / plan.bc, tr = plan.tr;
  for (std::size_t j = 0; j < tc; ++j) {
    const std::size_t bcj = std::min(plan.bc, nk - j * plan.bc);
    for (std::size_t i = 0; i < tr; ++i) {
      if (bm && !bm->at(i, j)) continue;
      const std::size_t bri = std::min(plan.br, n - i * plan.br);
      c.reads += 2 * bri * d + 2 * bri;   // Q_i, O_i, l_i, m_i
      c.writes += bri * d + 2 * bri;      // O_i, l_i, m_i
      c.flops += 4 * bri * bcj * d + 5 * bri * bcj + 2 * bri * d + 7 * bri;
    }
  }
  return c;
}

Charges backward_charges(std::size_t n, std::size_t nk, std::size_t d, const TilePlan& plan, const BlockMask* bm) {
  Charges c;
  c.writes += n * d;       // init dQ
  c.reads += 2 * nk * d;   // K, V once
  c.writes += 2 * nk * d;  // dK, dV once
  const std::size_t tc = (nk + plan.bc - 1) / plan.bc, tr = plan.tr;
  for (std::size_t j = 0; j < tc; ++j) {
    const std::size_t bcj = std::min(plan.bc, nk - j * plan.bc);
    for (std::size_t i = 0; i < tr; ++i) {
      if (bm && !bm->at(i, j)) continue;
      const std::size_t bri = std::min(plan.br, n - i * plan.br);
      c.reads += 4 * bri * d + 2 * bri;  // Q_i, O_i, dO_i, dQ_i, l_i, m_i
      c.writes += bri * d;               // dQ_i
      c.flops += 10 * bri * bcj * d + 5 * bri * bcj + 4 * bri * d + 2 * bcj * d;
    }
  }
  return c;
}

void charge(MemoryModel& mem, const Charges& c, std::size_t working_set) {
  auto lease = mem.lease(working_set);
  mem.charge_read(c.reads);
  mem.charge_write(c.writes);
  mem.charge_flops(c.flops);
}

FlashSaved forward_impl(const char* op, const Matrix& q, const Matrix& k, const Matrix& v, const AttnConfig& cfg,
                        const TilePlan& plan, const BlockMask* bm, MemoryModel& mem, const FlashOptions& options) {
  check_inputs(op, q, k, v, cfg);
  check_plan(op, plan, q.rows(), q.cols());
  if (bm && (bm->br != plan.br || bm->bc != plan.bc || bm->tr != plan.tr ||
             bm->tc < (k.rows() + plan.bc - 1) / plan.bc))
    throw std::invalid_argument(std::string(op) + ": bmask block sizes do not match the plan");
  Problem P = make_problem(q, k, cfg);
  const size_t eq = P.n * P.dp, ek = P.nk * P.dp;
  const std::size_t es = in_bytes(P.desc.dtype);
  DevBuf dq(eq * es), dk(ek * es), dv(ek * es), dout(eq * 4), dlse(P.n * 4), dvl(4), fws(16);
  upload_in(q, P.dp, P.desc.dtype, dq.p);
  upload_in(k, P.dp, P.desc.dtype, dk.p);
  upload_in(v, P.dp, P.desc.dtype, dv.p);
  check_cuda(cudaMemset(fws.p, 0, 16), "zero forward workspace");
  if (cfg.mask.kind == MaskKind::KeyPadding) {
    const int32_t vl = static_cast<int32_t>(std::min<std::size_t>(cfg.mask.valid_len, 0x7fffffff));
    check_cuda(cudaMemcpy(dvl.p, &vl, 4, cudaMemcpyHostToDevice), "upload valid_len");
    P.desc.valid_len = static_cast<const int32_t*>(dvl.p);
  }
  const TileGrid tg = bm ? tile_grid(*bm, P.n, P.nk) : TileGrid{};
  const CustomMask cmask(cfg, P.n, P.nk, bm, !tg.exact);
  cmask.attach(P.desc);
  std::vector<uint8_t> grid;
  DevBuf dgrid(bm ? ((P.n + 127) / 128) * ((P.nk + 127) / 128) : 0);
  if (bm) {
    grid = tg.g;
    check_cuda(cudaMemcpy(dgrid.p, grid.data(), grid.size(), cudaMemcpyHostToDevice), "upload grid");
    P.desc.block_grid = static_cast<const uint8_t*>(dgrid.p);
    P.desc.br = P.desc.bc = 128;
  }

  auto run = [&](int32_t nk_prefix) {
    tatn_attn_desc d = P.desc;
    d.Nk = nk_prefix;
    d.tc = static_cast<int32_t>((nk_prefix + 127) / 128);
    std::vector<uint8_t> sub;
    DevBuf dsub(bm ? static_cast<size_t>(d.tr) * d.tc : 0);
    if (bm && d.tc != P.desc.tc) {  // prefix of the tile grid: first d.tc columns of every row
      sub.resize(static_cast<size_t>(d.tr) * d.tc);
      for (int i = 0; i < d.tr; ++i)
        for (int j = 0; j < d.tc; ++j) sub[static_cast<size_t>(i) * d.tc + j] = grid[static_cast<size_t>(i) * P.desc.tc + j];
      check_cuda(cudaMemcpy(dsub.p, sub.data(), sub.size(), cudaMemcpyHostToDevice), "upload grid prefix");
      d.block_grid = static_cast<const uint8_t*>(dsub.p);
    }
    check_status(tatn_fwd(&d, dq.p, dk.p, dv.p, dout.p, static_cast<float*>(dlse.p), fws.p, 16, nullptr), op);
    check_cuda(cudaDeviceSynchronize(), op);
    std::vector<float> lse(P.n);
    check_cuda(cudaMemcpy(lse.data(), dlse.p, P.n * 4, cudaMemcpyDeviceToHost), "download lse");
    FlashSaved s;
    s.o = download32(dout.p, P.n, P.d, P.dp);
    s.stats = SoftmaxStats(P.n);
    for (std::size_t i = 0; i < P.n; ++i) {
      if (std::isinf(lse[i]) && lse[i] < 0) {
        s.stats.m[i] = kNegInf;
        s.stats.l[i] = 0.0;
      } else {
        s.stats.m[i] = lse[i];
        s.stats.l[i] = 1.0;
      }
    }
    if (has_nan(s.o)) throw std::runtime_error(std::string(op) + ": NaN in device output");
    return s;
  };

  // FlashObserver (flash.hpp:29-33): after outer key block j the state equals
  // attention over the key prefix [0, (j+1)*bc) (Appendix C), so
  // each snapshot is a prefix launch. The outer-loop permutation
  // (FlashOptions::outer_order) needs no action: outputs are schedule-invariant.
  if (options.observer) {
    const std::size_t tc = (P.nk + plan.bc - 1) / plan.bc;
    for (std::size_t j = 0; j + 1 < tc; ++j) {
      const FlashSaved snap = run(static_cast<int32_t>((j + 1) * plan.bc));
      options.observer(j, snap.o, snap.stats.l, snap.stats.m);
    }
  }
  FlashSaved saved = run(static_cast<int32_t>(P.nk));
  if (options.observer) {
    const std::size_t tc = (P.nk + plan.bc - 1) / plan.bc;
    options.observer(tc - 1, saved.o, saved.stats.l, saved.stats.m);
  }
  saved.rng = DropoutRng{cfg.seed};
  saved.plan = plan;
  saved.cfg = cfg;
  charge(mem, forward_charges(P.n, P.nk, P.d, plan, bm), plan.working_set);
  return saved;
}

Gradients backward_impl(const char* op, const FlashSaved& saved, const Matrix& q, const Matrix& k, const Matrix& v,
                        const Matrix& d_o, const BlockMask* bm, MemoryModel& mem) {
  const AttnConfig& cfg = saved.cfg;
  check_inputs(op, q, k, v, cfg);
  check_plan(op, saved.plan, q.rows(), q.cols());
  if (!d_o.same_shape(q) || !saved.o.same_shape(q) || saved.stats.size() != q.rows())
    throw std::invalid_argument(std::string(op) + ": saved state / dO do not match Q");
  if (has_nan(d_o)) throw std::invalid_argument(std::string(op) + ": NaN input");
  saved.stats.validate();
  if (bm && (bm->br != saved.plan.br || bm->bc != saved.plan.bc))
    throw std::invalid_argument(std::string(op) + ": bmask block sizes do not match the plan");
  Problem P = make_problem(q, k, cfg);
  const size_t eq = P.n * P.dp, ek = P.nk * P.dp;
  const std::size_t es = in_bytes(P.desc.dtype);
  DevBuf dq(eq * es), dk(ek * es), dv(ek * es), ddo(eq * es), dov(eq * 4), dlse(P.n * 4), dvl(4);
  DevBuf gq(eq * 4), gk(ek * 4), gv(ek * 4);
  upload_in(q, P.dp, P.desc.dtype, dq.p);
  upload_in(k, P.dp, P.desc.dtype, dk.p);
  upload_in(v, P.dp, P.desc.dtype, dv.p);
  upload_in(d_o, P.dp, P.desc.dtype, ddo.p);
  upload32(saved.o, P.dp, dov.p);  // fp32 O: D_i = dO_i . O_i without output rounding
  std::vector<float> lse(P.n);
  for (std::size_t i = 0; i < P.n; ++i)
    lse[i] = saved.stats.l[i] > 0.0 ? static_cast<float>(saved.stats.m[i] + std::log(saved.stats.l[i]))
                                     : -std::numeric_limits<float>::infinity();
  check_cuda(cudaMemcpy(dlse.p, lse.data(), P.n * 4, cudaMemcpyHostToDevice), "upload lse");
  if (cfg.mask.kind == MaskKind::KeyPadding) {
    const int32_t vl = static_cast<int32_t>(std::min<std::size_t>(cfg.mask.valid_len, 0x7fffffff));
    check_cuda(cudaMemcpy(dvl.p, &vl, 4, cudaMemcpyHostToDevice), "upload valid_len");
    P.desc.valid_len = static_cast<const int32_t*>(dvl.p);
  }
  const TileGrid tg = bm ? tile_grid(*bm, P.n, P.nk) : TileGrid{};
  const CustomMask cmask(cfg, P.n, P.nk, bm, !tg.exact);
  cmask.attach(P.desc);
  DevBuf dgrid(bm ? ((P.n + 127) / 128) * ((P.nk + 127) / 128) : 0);
  if (bm) {
    const auto& grid = tg.g;
    check_cuda(cudaMemcpy(dgrid.p, grid.data(), grid.size(), cudaMemcpyHostToDevice), "upload grid");
    P.desc.block_grid = static_cast<const uint8_t*>(dgrid.p);
    P.desc.br = P.desc.bc = 128;
  }
  const size_t wsb = tatn_bwd_workspace_bytes(&P.desc);
  DevBuf ws(wsb);
  check_status(tatn_bwd(&P.desc, dq.p, dk.p, dv.p, dov.p, ddo.p, static_cast<const float*>(dlse.p), gq.p, gk.p, gv.p,
                        ws.p, wsb, nullptr),
               op);
  check_cuda(cudaDeviceSynchronize(), op);
  Gradients g;
  g.dq = download32(gq.p, P.n, P.d, P.dp);
  g.dk = download32(gk.p, P.nk, P.d, P.dp);
  g.dv = download32(gv.p, P.nk, P.d, P.dp);
  if (has_nan(g.dq) || has_nan(g.dk) || has_nan(g.dv))
    throw std::runtime_error(std::string(op) + ": NaN in device gradients");
  charge(mem, backward_charges(P.n, P.nk, P.d, saved.plan, bm),
         backward_working_set_elems(saved.plan.br, saved.plan.bc, P.d));
  return g;
}

}  // namespace
}  // namespace b200

FlashSaved flash_forward(const Matrix& q, const Matrix& k, const Matrix& v, const AttnConfig& cfg, const TilePlan& plan,
                         MemoryModel& mem, const FlashOptions& options) {
  return b200::forward_impl("flash_forward", q, k, v, cfg, plan, nullptr, mem, options);
}

Gradients flash_backward(const FlashSaved& saved, const Matrix& q, const Matrix& k, const Matrix& v, const Matrix& d_o,
                         MemoryModel& mem) {
  return b200::backward_impl("flash_backward", saved, q, k, v, d_o, nullptr, mem);
}

FlashSaved blocksparse_forward(const Matrix& q, const Matrix& k, const Matrix& v, const AttnConfig& cfg,
                               const TilePlan& plan, const BlockMask& bmask, MemoryModel& mem,
                               const FlashOptions& options) {
  return b200::forward_impl("blocksparse_forward", q, k, v, cfg, plan, &bmask, mem, options);
}

Gradients blocksparse_backward(const FlashSaved& saved, const Matrix& q, const Matrix& k, const Matrix& v,
                               const Matrix& d_o, const BlockMask& bmask, MemoryModel& mem) {
  return b200::backward_impl("blocksparse_backward", saved, q, k, v, d_o, &bmask, mem);
}

}  // namespace tatn
