// dropin_check.cpp — GPU acceptance run of the C++ drop-in (tests/test_dropin_gpu.py).
//
// Links the reference's tatn_core sources with flash_b200.cpp / support_b200.cpp
// and exercises the reference surface exactly as the reference's own (absent)
// tests would: flash_* against standard_* on the same
// 16-bit-rounded fp64 inputs, the observer/prefix invariant, block-sparse
// semantics, MemoryModel counters against the io_predict closed forms, and the
// error behaviour. Prints one "CHECK <name> ok|FAIL <detail>" line per check;
// exit code 0 iff every check passed.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "tatn/block_mask.hpp"
#include "tatn/flash.hpp"
#include "tatn/io_predict.hpp"
#include "tatn/random.hpp"
#include "tatn/reference.hpp"
#include "tatn/tile_plan.hpp"
#include "tatn_b200.h"
#include "flash_b200_multi.hpp"

namespace tatn::b200 {
void set_input_dtype_fp16(bool fp16);
void set_input_dtype(int dtype);
}

using namespace tatn;

static int g_fail = 0;

static void report(const std::string& name, bool ok, const std::string& detail = "") {
  std::printf("CHECK %s %s %s\n", name.c_str(), ok ? "ok" : "FAIL", detail.c_str());
  if (!ok) ++g_fail;
}

static double to_bf16(double x) {
  float f = static_cast<float>(x);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  std::memcpy(&f, &u, 4);
  return f;
}

static Matrix rounded(Matrix m) {
  for (double& x : m.data()) x = to_bf16(x);
  return m;
}

static double max_abs(const Matrix& a, const Matrix& b) { return max_abs_diff(a, b); }

static double rel_l2(const Matrix& a, const Matrix& b) {
  double num = 0, den = 0;
  auto da = a.data(), db = b.data();
  for (size_t i = 0; i < da.size(); ++i) {
    num += (da[i] - db[i]) * (da[i] - db[i]);
    den += db[i] * db[i];
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

static std::string fmt(double a, double b) {
  char buf[96];
  std::snprintf(buf, sizeof buf, "max_abs=%.3e rel_l2=%.3e", a, b);
  return buf;
}

// fp32-output check-mode tolerance for 16-bit inputs (the north star's 16-bit bar is 2e-2 / 1e-2;
// what remains here is P and dS rounded to 16 bits inside the MMAs)
static bool close(const Matrix& got, const Matrix& ref, double tol_abs = 1e-2, double tol_rel = 3e-3) {
  return max_abs(got, ref) <= tol_abs && rel_l2(got, ref) <= tol_rel;
}

struct Case {
  std::string name;
  size_t n, nk, d;
  MaskSpec mask;
};

static void check_dense(const Case& c) {
  AttnConfig cfg = AttnConfig::make(c.n, c.d);
  cfg.mask = c.mask;
  Matrix q = rounded(gaussian_matrix(c.n, c.d, 11)), k = rounded(gaussian_matrix(c.nk, c.d, 12)),
         v = rounded(gaussian_matrix(c.nk, c.d, 13)), dO = rounded(gaussian_matrix(c.n, c.d, 14));
  const TilePlan plan = plan_tiles(c.n, c.d, 116224);  // M = 227 KiB of bf16
  MemoryModel mem(plan.m_capacity);
  const FlashSaved s = flash_forward(q, k, v, cfg, plan, mem);
  const ForwardArtifacts ref = standard_forward(q, k, v, cfg);
  bool lse_ok = true;
  for (size_t i = 0; i < c.n; ++i) {
    const double a = s.stats.l[i] > 0 ? s.stats.m[i] + std::log(s.stats.l[i]) : -INFINITY;
    const double b = ref.stats.l[i] > 0 ? ref.stats.m[i] + std::log(ref.stats.l[i]) : -INFINITY;
    if (std::isinf(a) || std::isinf(b)) lse_ok &= (std::isinf(a) && std::isinf(b));
    else lse_ok &= std::fabs(a - b) < 1e-3;
  }
  report(c.name + "/forward_O", close(s.o, ref.o), fmt(max_abs(s.o, ref.o), rel_l2(s.o, ref.o)));
  report(c.name + "/forward_stats", lse_ok);
  s.stats.validate();
  const Gradients g = flash_backward(s, q, k, v, dO, mem);
  const Gradients rg = standard_backward(ref, q, k, v, dO, cfg);
  report(c.name + "/backward_dQ", close(g.dq, rg.dq), fmt(max_abs(g.dq, rg.dq), rel_l2(g.dq, rg.dq)));
  report(c.name + "/backward_dK", close(g.dk, rg.dk), fmt(max_abs(g.dk, rg.dk), rel_l2(g.dk, rg.dk)));
  report(c.name + "/backward_dV", close(g.dv, rg.dv), fmt(max_abs(g.dv, rg.dv), rel_l2(g.dv, rg.dv)));
}

int main() {
  try {
    // ---- SPEC.md:232 singleton: N = d = 1, Q = K = V = [[1]], tau = 1 -> O = [[1]], l = 1, m = 1
    {
      AttnConfig cfg = AttnConfig::make(1, 1);
      cfg.tau = 1.0;
      Matrix one = Matrix::filled(1, 1, 1.0);
      const TilePlan plan = plan_tiles(1, 1, 64);
      MemoryModel mem(plan.m_capacity);
      FlashSaved s = flash_forward(one, one, one, cfg, plan, mem);
      report("spec_singleton", s.o(0, 0) == 1.0 && s.stats.m[0] + std::log(s.stats.l[0]) == 1.0);
    }
    // ---- oracle equivalence over masks, ragged n, key prefixes, d in {16, 64, 100, 128}
    check_dense({"n512_d64_none", 512, 512, 64, MaskSpec::none()});
    check_dense({"n777_d128_causal", 777, 777, 128, MaskSpec::causal()});
    check_dense({"n300_d64_padding", 300, 300, 64, MaskSpec::key_padding(211)});
    check_dense({"n300_d64_padding0", 300, 300, 64, MaskSpec::key_padding(0)});
    check_dense({"n640_prefix400_d100_causal", 640, 400, 100, MaskSpec::causal()});
    check_dense({"n129_d16_none", 129, 129, 16, MaskSpec::none()});
    // ---- Custom n x n additive masks (attn_config.hpp:27): random keep pattern with a
    // fully masked row (O = 0, l = 0, m = -inf) and a key nobody attends to (dK = dV = 0)
    {
      const size_t n = 333;
      Matrix pat(n, n);
      uint64_t h = 0x9e3779b97f4a7c15ull;
      for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < n; ++j) {
          h ^= h << 13; h ^= h >> 7; h ^= h << 17;
          const bool keep = (h % 10) < 6 && i != 7 && j != 11;
          pat(i, j) = keep ? 0.0 : -std::numeric_limits<double>::infinity();
        }
      check_dense({"n333_d64_custom", n, n, 64, MaskSpec::custom_additive(pat)});
      check_dense({"n333_prefix200_d128_custom", n, 200, 128, MaskSpec::custom_additive(pat)});
    }

    // ---- counters equal the io_predict closed forms for uniform blocks
    {
      const size_t n = 1024, d = 64;
      AttnConfig cfg = AttnConfig::make(n, d);
      Matrix x = rounded(gaussian_matrix(n, d, 5));
      const TilePlan plan = plan_tiles(n, d, 65536);  // bc = 256, br = 64
      MemoryModel mem(plan.m_capacity);
      FlashSaved s = flash_forward(x, x, x, cfg, plan, mem);
      const IoPrediction pf = predict_flash_forward_io(n, d, plan);
      report("counters_forward_closed_form",
             mem.counter().hbm_read_elems == pf.reads && mem.counter().hbm_write_elems == pf.writes &&
                 mem.counter().flops == flop_model(AlgoId::FlashForward, n, d, &plan));
      MemoryModel mem2(plan.m_capacity);
      flash_backward(s, x, x, x, x, mem2);
      const IoPrediction pb = predict_flash_backward_io(n, d, plan);
      report("counters_backward_closed_form",
             mem2.counter().hbm_read_elems == pb.reads && mem2.counter().hbm_write_elems == pb.writes &&
                 mem2.counter().flops == flop_model(AlgoId::FlashBackward, n, d, &plan));
      report("peak_residency_within_1.5M",
             static_cast<double>(mem.counter().peak_resident_elems) <= 1.5 * plan.m_capacity);
    }

    // ---- block-sparse: all-true == dense bit-identical (outputs and counters), butterfly vs
    // the reference with the composed element mask, empty block row
    {
      const size_t n = 1024, d = 64;
      AttnConfig cfg = AttnConfig::make(n, d);
      Matrix q = rounded(gaussian_matrix(n, d, 21)), k = rounded(gaussian_matrix(n, d, 22)),
             v = rounded(gaussian_matrix(n, d, 23)), dO = rounded(gaussian_matrix(n, d, 24));
      TileOverrides ov;
      ov.br = 128;
      ov.bc = 128;
      const TilePlan plan = plan_tiles(n, d, 116224, ov);
      MemoryModel m1(plan.m_capacity), m2(plan.m_capacity);
      FlashSaved dense = flash_forward(q, k, v, cfg, plan, m1);
      BlockMask all = make_block_mask_random(1.0, 1, plan.tr, plan.tc, plan.br, plan.bc);
      FlashSaved sp = blocksparse_forward(q, k, v, cfg, plan, all, m2);
      report("blocksparse_alltrue_bit_identical_forward",
             dense.o == sp.o && dense.stats.m == sp.stats.m && m1.counter().hbm_read_elems == m2.counter().hbm_read_elems &&
                 m1.counter().hbm_write_elems == m2.counter().hbm_write_elems && m1.counter().flops == m2.counter().flops);
      MemoryModel m3(plan.m_capacity), m4(plan.m_capacity);
      Gradients gd = flash_backward(dense, q, k, v, dO, m3);
      Gradients gs = blocksparse_backward(sp, q, k, v, dO, all, m4);
      report("blocksparse_alltrue_backward", gd.dk == gs.dk && gd.dv == gs.dv && gd.dq == gs.dq &&
                                                 m3.counter().hbm_read_elems == m4.counter().hbm_read_elems);

      BlockMask bf = make_block_mask_butterfly(plan.tr, plan.tc, plan.br, plan.bc);
      bf.grid[3 * plan.tc + 3] = 0;  // punch a hole so some row block differs from the pattern
      bf.density = static_cast<double>(bf.count_true()) / static_cast<double>(bf.tr * bf.tc);
      MemoryModel m5(plan.m_capacity);
      FlashSaved sb = blocksparse_forward(q, k, v, cfg, plan, bf, m5);
      AttnConfig ccfg = cfg;
      ccfg.mask = compose_block_mask(cfg.mask, bf, n);
      ForwardArtifacts rb = standard_forward(q, k, v, ccfg);
      report("blocksparse_butterfly_forward", close(sb.o, rb.o), fmt(max_abs(sb.o, rb.o), rel_l2(sb.o, rb.o)));
      MemoryModel m6(plan.m_capacity);
      Gradients g = blocksparse_backward(sb, q, k, v, dO, bf, m6);
      Gradients rgb = standard_backward(rb, q, k, v, dO, ccfg);
      report("blocksparse_butterfly_backward",
             close(g.dq, rgb.dq) && close(g.dk, rgb.dk) && close(g.dv, rgb.dv),
             fmt(max_abs(g.dk, rgb.dk), rel_l2(g.dk, rgb.dk)));
      const IoPrediction pbs = predict_blocksparse_io(n, d, plan, bf.density);
      report("blocksparse_counters_closed_form",
             m5.counter().hbm_read_elems == pbs.reads && m5.counter().hbm_write_elems == pbs.writes);

      BlockMask er = make_block_mask_local_global(0, 0, plan.tr, plan.tc, plan.br, plan.bc);
      for (size_t j = 0; j < plan.tc; ++j) er.grid[2 * plan.tc + j] = 0;  // empty block row 2
      MemoryModel m7(plan.m_capacity);
      FlashSaved se = blocksparse_forward(q, k, v, cfg, plan, er, m7);
      bool empty_ok = true;
      for (size_t i = 256; i < 384; ++i) {
        empty_ok &= se.stats.l[i] == 0.0 && std::isinf(se.stats.m[i]);
        for (size_t x = 0; x < d; ++x) empty_ok &= se.o(i, x) == 0.0;
      }
      MemoryModel m8(plan.m_capacity);
      Gradients ge = blocksparse_backward(se, q, k, v, dO, er, m8);
      for (size_t i = 256; i < 384; ++i)
        for (size_t x = 0; x < d; ++x) empty_ok &= ge.dk(i, x) == 0.0 && ge.dv(i, x) == 0.0 && ge.dq(i, x) == 0.0;
      report("blocksparse_empty_row_and_uncovered_keys", empty_ok);
    }

    // ---- block-sparse at the reference's own block sizes: the default plan
    // (br = 64, bc = 256 at n = 1024, d = 64), br = bc = 16, br = bc = 1 and br = bc = n, against
    // the reference's standard path under compose_block_mask; all-true at br = 64 == dense
    {
      struct BS {
        const char* name;
        size_t n, d, br, bc;  // br = bc = 0: the default plan
        int kind;             // 0 butterfly, 1 local/global, 2 random(0.5), 3 all-true
        MaskSpec base;
      };
      const BS cases[] = {
          {"bs_default_plan_butterfly_causal", 1024, 64, 0, 0, 0, MaskSpec::causal()},
          {"bs_16x16_local_global_ragged", 300, 64, 16, 16, 1, MaskSpec::none()},
          {"bs_1x1_random_padding", 160, 64, 1, 1, 2, MaskSpec::key_padding(150)},
          {"bs_nxn_single_block", 200, 64, 200, 200, 3, MaskSpec::none()},
          {"bs_32x64_butterfly_d128", 256, 128, 32, 64, 0, MaskSpec::none()},
      };
      for (const BS& c : cases) {
        AttnConfig cfg = AttnConfig::make(c.n, c.d);
        cfg.mask = c.base;
        TileOverrides ov;
        ov.br = c.br;
        ov.bc = c.bc;
        const TilePlan plan = c.br ? plan_tiles(c.n, c.d, 65536, ov) : plan_tiles(c.n, c.d, 65536);
        BlockMask bm = c.kind == 0   ? make_block_mask_butterfly(plan.tr, plan.tc, plan.br, plan.bc)
                       : c.kind == 1 ? make_block_mask_local_global(1, 1, plan.tr, plan.tc, plan.br, plan.bc)
                       : c.kind == 2 ? make_block_mask_random(0.5, 5, plan.tr, plan.tc, plan.br, plan.bc)
                                     : make_block_mask_random(1.0, 5, plan.tr, plan.tc, plan.br, plan.bc);
        Matrix q = rounded(gaussian_matrix(c.n, c.d, 81)), k = rounded(gaussian_matrix(c.n, c.d, 82)),
               v = rounded(gaussian_matrix(c.n, c.d, 83)), dO = rounded(gaussian_matrix(c.n, c.d, 84));
        MemoryModel mf(plan.m_capacity), mb(plan.m_capacity);
        FlashSaved sb = blocksparse_forward(q, k, v, cfg, plan, bm, mf);
        Gradients g = blocksparse_backward(sb, q, k, v, dO, bm, mb);
        AttnConfig ccfg = cfg;
        ccfg.mask = compose_block_mask(cfg.mask, bm, c.n);
        ForwardArtifacts rb = standard_forward(q, k, v, ccfg);
        Gradients rg = standard_backward(rb, q, k, v, dO, ccfg);
        const std::string tag = std::string(c.name) + "_br" + std::to_string(plan.br) + "_bc" + std::to_string(plan.bc);
        report(tag + "_forward", close(sb.o, rb.o), fmt(max_abs(sb.o, rb.o), rel_l2(sb.o, rb.o)));
        report(tag + "_backward", close(g.dq, rg.dq) && close(g.dk, rg.dk) && close(g.dv, rg.dv),
               fmt(max_abs(g.dk, rg.dk), rel_l2(g.dk, rg.dk)));
        const IoPrediction pbs = predict_blocksparse_io(c.n, c.d, plan, bm.density);
        report(tag + "_counters_closed_form", c.n % plan.br != 0 || c.n % plan.bc != 0 ||
                                                  (mf.counter().hbm_read_elems == pbs.reads &&
                                                   mf.counter().hbm_write_elems == pbs.writes));
      }
      {  // all-true at br = 64 runs on the exact tile path: bit-identical to the dense engine
        const size_t n = 512, d = 64;
        AttnConfig cfg = AttnConfig::make(n, d);
        cfg.mask = MaskSpec::causal();
        TileOverrides ov;
        ov.br = 64;
        ov.bc = 64;
        const TilePlan plan = plan_tiles(n, d, 65536, ov);
        BlockMask all = make_block_mask_random(1.0, 1, plan.tr, plan.tc, plan.br, plan.bc);
        Matrix q = rounded(gaussian_matrix(n, d, 91)), k = rounded(gaussian_matrix(n, d, 92)),
               v = rounded(gaussian_matrix(n, d, 93));
        MemoryModel m1(plan.m_capacity), m2(plan.m_capacity);
        FlashSaved dense = flash_forward(q, k, v, cfg, plan, m1);
        FlashSaved sp = blocksparse_forward(q, k, v, cfg, plan, all, m2);
        report("bs_alltrue_br64_bit_identical_forward", dense.o == sp.o && dense.stats.m == sp.stats.m);
      }
    }

    // ---- the reference's concurrency model over devices: heads split across workers (one host thread
    // per worker, worker w on device w % ndev), private MemoryModels merged with AccessCounter::merge;
    // identical outputs to the per-head calls, merged counters == their sum (peak = max)
    {
      const size_t n = 384, d = 64;
      const TilePlan plan = plan_tiles(n, d, 116224);
      std::vector<Matrix> qs, ks, vs, dos;
      for (int h = 0; h < 7; ++h) {
        qs.push_back(rounded(gaussian_matrix(n, d, 300 + 4 * h)));
        ks.push_back(rounded(gaussian_matrix(n, d, 301 + 4 * h)));
        vs.push_back(rounded(gaussian_matrix(n, d, 302 + 4 * h)));
        dos.push_back(rounded(gaussian_matrix(n, d, 303 + 4 * h)));
      }
      std::vector<b200::HeadProblem> heads;
      std::vector<const Matrix*> dop;
      for (int h = 0; h < 7; ++h) {
        AttnConfig cfg = AttnConfig::make(n, d);
        cfg.mask = (h & 1) ? MaskSpec::causal() : MaskSpec::none();
        heads.push_back({&qs[h], &ks[h], &vs[h], cfg});
        dop.push_back(&dos[h]);
      }
      MemoryModel one(plan.m_capacity);
      std::vector<FlashSaved> seq;
      std::vector<Gradients> seqg;
      for (int h = 0; h < 7; ++h) seq.push_back(flash_forward(qs[h], ks[h], vs[h], heads[h].cfg, plan, one));
      for (int h = 0; h < 7; ++h) seqg.push_back(flash_backward(seq[h], qs[h], ks[h], vs[h], dos[h], one));
      for (int workers : {0, 3}) {
        MemoryModel merged(plan.m_capacity);
        auto sh = b200::flash_forward_sharded(heads, plan, merged, workers);
        auto shg = b200::flash_backward_sharded(sh, heads, dop, merged, workers);
        bool same = sh.size() == 7 && shg.size() == 7;
        for (int h = 0; same && h < 7; ++h)
          same = sh[h].o == seq[h].o && sh[h].stats.m == seq[h].stats.m && shg[h].dq == seqg[h].dq &&
                 shg[h].dk == seqg[h].dk && shg[h].dv == seqg[h].dv;
        report("sharded_workers" + std::to_string(workers) + "_outputs_equal_per_head_calls", same);
        report("sharded_workers" + std::to_string(workers) + "_counters_merged",
               merged.counter().hbm_read_elems == one.counter().hbm_read_elems &&
                   merged.counter().hbm_write_elems == one.counter().hbm_write_elems &&
                   merged.counter().flops == one.counter().flops &&
                   merged.counter().peak_resident_elems == one.counter().peak_resident_elems);
      }
    }

    // ---- observer: after outer block j the snapshot equals the oracle on the key prefix
    {
      const size_t n = 600, d = 64;
      AttnConfig cfg = AttnConfig::make(n, d);
      cfg.mask = MaskSpec::causal();
      Matrix q = rounded(gaussian_matrix(n, d, 31)), k = rounded(gaussian_matrix(n, d, 32)),
             v = rounded(gaussian_matrix(n, d, 33));
      TileOverrides ov;
      ov.bc = 200;
      ov.br = 64;
      const TilePlan plan = plan_tiles(n, d, 116224, ov);
      size_t calls = 0;
      bool ok = true;
      FlashOptions opt;
      opt.observer = [&](size_t j, const Matrix& o, const std::vector<double>& l, const std::vector<double>& m) {
        const size_t nk = std::min(n, (j + 1) * plan.bc);
        Matrix kp(nk, d), vp(nk, d);
        for (size_t r = 0; r < nk; ++r)
          for (size_t x = 0; x < d; ++x) {
            kp(r, x) = k(r, x);
            vp(r, x) = v(r, x);
          }
        const ForwardArtifacts pr = standard_forward(q, kp, vp, cfg);
        ok &= close(o, pr.o) && l.size() == n && m.size() == n;
        ++calls;
      };
      MemoryModel mem(plan.m_capacity);
      flash_forward(q, k, v, cfg, plan, mem, opt);
      report("observer_prefix_induction", ok && calls == plan.tc, "calls=" + std::to_string(calls));
    }

    // ---- schedule invariance: outer_order permutations change nothing
    {
      const size_t n = 512, d = 64;
      AttnConfig cfg = AttnConfig::make(n, d);
      Matrix x = rounded(gaussian_matrix(n, d, 41));
      const TilePlan plan = plan_tiles(n, d, 65536);
      FlashOptions opt;
      for (size_t j = plan.tc; j-- > 0;) opt.outer_order.push_back(j);
      MemoryModel m1(plan.m_capacity), m2(plan.m_capacity);
      report("outer_order_invariance", flash_forward(x, x, x, cfg, plan, m1).o == flash_forward(x, x, x, cfg, plan, m2, opt).o);
    }

    // ---- error behaviour (flash.hpp:47-48): std::invalid_argument, never a silent fallback
    {
      auto throws = [](const std::function<void()>& f) {
        try {
          f();
        } catch (const std::invalid_argument&) {
          return true;
        }
        return false;
      };
      const size_t n = 256, d = 64;
      Matrix x = rounded(gaussian_matrix(n, d, 51));
      const TilePlan plan = plan_tiles(n, d, 65536);
      MemoryModel mem(plan.m_capacity);
      AttnConfig drop = AttnConfig::make(n, d);
      drop.p_drop = 1.0;
      report("error_dropout_p_out_of_range", throws([&] { flash_forward(x, x, x, drop, plan, mem); }));
      AttnConfig cust = AttnConfig::make(n, d);
      cust.mask = MaskSpec::custom_additive(Matrix::filled(n, n, 1.0));  // entries must be 0 or -inf
      report("error_custom_mask_entries", throws([&] { flash_forward(x, x, x, cust, plan, mem); }));
      cust.mask = MaskSpec::custom_additive(Matrix(n - 1, n - 1));  // must be n x n
      report("error_custom_mask_shape", throws([&] { flash_forward(x, x, x, cust, plan, mem); }));
      AttnConfig ok = AttnConfig::make(n, d);
      const TilePlan wrong = plan_tiles(2 * n, d, 65536);
      report("error_plan_mismatch", throws([&] { flash_forward(x, x, x, ok, wrong, mem); }));
      Matrix bad = x;
      bad(3, 3) = std::numeric_limits<double>::quiet_NaN();
      report("error_nan_input", throws([&] { flash_forward(bad, x, x, ok, plan, mem); }));
      Matrix wide = rounded(gaussian_matrix(n, 160, 52));
      AttnConfig wcfg = AttnConfig::make(n, 160);
      report("error_head_dim_over_128", throws([&] { flash_forward(wide, wide, wide, wcfg, plan_tiles(n, 160, 116224), mem); }));
      BlockMask b64 = make_block_mask_butterfly(4, 4, 64, 64);
      const TilePlan p128 = plan_tiles(n, d, 65536);
      report("error_bmask_plan_mismatch", throws([&] { blocksparse_forward(x, x, x, ok, p128, b64, mem); }));
    }

    // ---- dropout: same positional mask as the reference (dropout.cpp)
    for (double pd : {0.1, 0.5}) {
      const size_t n = 300, d = 64;
      AttnConfig cfg = AttnConfig::make(n, d);
      cfg.mask = MaskSpec::causal();
      cfg.p_drop = pd;
      cfg.seed = 7;
      Matrix q = rounded(gaussian_matrix(n, d, 71)), k = rounded(gaussian_matrix(n, d, 72)),
             v = rounded(gaussian_matrix(n, d, 73)), dO = rounded(gaussian_matrix(n, d, 74));
      const TilePlan plan = plan_tiles(n, d, 116224);
      MemoryModel mem(plan.m_capacity);
      FlashSaved s = flash_forward(q, k, v, cfg, plan, mem);
      ForwardArtifacts r = standard_forward(q, k, v, cfg);
      Gradients g = flash_backward(s, q, k, v, dO, mem);
      Gradients rg = standard_backward(r, q, k, v, dO, cfg);
      const std::string tag = "dropout_p" + std::to_string(static_cast<int>(pd * 10));
      report(tag + "_forward", close(s.o, r.o), fmt(max_abs(s.o, r.o), rel_l2(s.o, r.o)));
      report(tag + "_backward", close(g.dq, rg.dq) && close(g.dk, rg.dk) && close(g.dv, rg.dv),
             fmt(max_abs(g.dv, rg.dv), rel_l2(g.dv, rg.dv)));
    }

    // ---- fp32 input mode (tf32 check mode; BASELINE configs[0]: N = 512, d = 64, non-causal, fp32): the
    // reference's fp64 engines on the same fp32 inputs, at the fp32 bar (max abs 2e-3, rel-L2 1e-3)
    {
      b200::set_input_dtype(TATN_DTYPE_FP32);
      const size_t n = 512, d = 64;
      for (int causal = 0; causal < 2; ++causal) {
        AttnConfig cfg = AttnConfig::make(n, d);
        if (causal) cfg.mask = MaskSpec::causal();
        Matrix q = gaussian_matrix(n, d, 41), k = gaussian_matrix(n, d, 42), v = gaussian_matrix(n, d, 43),
               dO = gaussian_matrix(n, d, 44);
        for (Matrix* m : {&q, &k, &v, &dO})
          for (double& x : m->data()) x = static_cast<double>(static_cast<float>(x));  // the fp32 inputs
        const TilePlan plan = plan_tiles(n, d, 65536);
        MemoryModel mem(plan.m_capacity);
        FlashSaved s = flash_forward(q, k, v, cfg, plan, mem);
        Gradients g = flash_backward(s, q, k, v, dO, mem);
        ForwardArtifacts r = standard_forward(q, k, v, cfg);
        Gradients rg = standard_backward(r, q, k, v, dO, cfg);
        const std::string tag = causal ? "fp32_inputs_c1_causal" : "fp32_inputs_c1";
        report(tag + "_forward", close(s.o, r.o, 2e-3, 1e-3), fmt(max_abs(s.o, r.o), rel_l2(s.o, r.o)));
        report(tag + "_backward",
               close(g.dq, rg.dq, 2e-3, 1e-3) && close(g.dk, rg.dk, 2e-3, 1e-3) && close(g.dv, rg.dv, 2e-3, 1e-3),
               fmt(max_abs(g.dq, rg.dq), rel_l2(g.dq, rg.dq)));
      }
      b200::set_input_dtype(TATN_DTYPE_BF16);
    }

    // ---- fp16 input mode
    {
      b200::set_input_dtype_fp16(true);
      const size_t n = 384, d = 128;
      AttnConfig cfg = AttnConfig::make(n, d);
      Matrix q = gaussian_matrix(n, d, 61), k = gaussian_matrix(n, d, 62), v = gaussian_matrix(n, d, 63);
      for (Matrix* m : {&q, &k, &v})
        for (double& x : m->data()) x = static_cast<double>(static_cast<float>(x));  // the fp16 rounding happens inside
      const TilePlan plan = plan_tiles(n, d, 116224);
      MemoryModel mem(plan.m_capacity);
      FlashSaved s = flash_forward(q, k, v, cfg, plan, mem);
      ForwardArtifacts r = standard_forward(q, k, v, cfg);
      report("fp16_inputs_forward", close(s.o, r.o, 2e-3, 1e-3), fmt(max_abs(s.o, r.o), rel_l2(s.o, r.o)));
      b200::set_input_dtype_fp16(false);
    }
  } catch (const std::exception& e) {
    report("unexpected_exception", false, e.what());
  }
  std::printf("SUMMARY %s %d failed\n", g_fail == 0 ? "ok" : "FAIL", g_fail);
  return g_fail == 0 ? 0 : 1;
}
