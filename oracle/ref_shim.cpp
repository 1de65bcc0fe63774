// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the REFERENCE's own implementation, compiled
// together with the reference sources where they lie under
// /root/reference/proj/core/src (see oracle/Makefile; output only into
// oracle/_ref/). Used to pin the C restatement (oracle/tatn_oracle.c), to
// generate tests/golden/, and as bench.py's "reference" CPU arm.
// No reference source is copied into this repository.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "tatn/attn_config.hpp"
#include "tatn/dropout.hpp"
#include "tatn/counters.hpp"
#include "tatn/matrix.hpp"
#include "tatn/matrix_io.hpp"
#include "tatn/random.hpp"
#include "tatn/reference.hpp"
#include "tatn/softmax.hpp"

namespace {

tatn::Matrix to_matrix(const double* p, int rows, int cols) {
  return tatn::Matrix(rows, cols, std::vector<double>(p, p + static_cast<size_t>(rows) * cols));
}

void from_matrix(const tatn::Matrix& m, double* out) {
  auto d = m.data();
  std::memcpy(out, d.data(), d.size() * sizeof(double));
}

// mask_kind: 0 none, 1 causal, 2 key padding. grid (tr x tc at br x bc) is
// composed into a Custom additive mask on top of the base predicate, i.e.
// the element mask compose_block_mask documents (block_mask.hpp:42-46).
tatn::AttnConfig make_cfg(int n, int d, double tau, int mask_kind, int valid_len, const uint8_t* grid, int br, int bc,
                          int tc, double p_drop = 0.0, uint64_t seed = 0) {
  tatn::AttnConfig cfg = tatn::AttnConfig::make(n, d);
  cfg.tau = tau;
  cfg.p_drop = p_drop;
  cfg.seed = seed;
  if (mask_kind == 1) cfg.mask = tatn::MaskSpec::causal();
  if (mask_kind == 2) cfg.mask = tatn::MaskSpec::key_padding(valid_len);
  if (mask_kind == 3) {
    // Custom: `grid` carries an n x nk keep matrix (1 = 0.0, 0 = -inf); the reference wants
    // an n x n additive pattern (attn_config.cpp:50-52), keys >= nk are never read
    const double ninf = -std::numeric_limits<double>::infinity();
    tatn::Matrix pat(n, n);
    const int nk = tc;  // mask_kind 3 passes nk in tc
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) pat(i, j) = (j < nk && grid[static_cast<size_t>(i) * nk + j]) ? 0.0 : ninf;
    cfg.mask = tatn::MaskSpec::custom_additive(std::move(pat));
    return cfg;
  }
  if (grid != nullptr) {
    const double ninf = -std::numeric_limits<double>::infinity();
    tatn::Matrix pat(n, n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const bool blk = grid[static_cast<size_t>(i / br) * tc + (j / bc)] != 0;
        pat(i, j) = (blk && !tatn::is_masked(cfg.mask, i, j)) ? 0.0 : ninf;
      }
    cfg.mask = tatn::MaskSpec::custom_additive(std::move(pat));
  }
  return cfg;
}

}  // namespace

extern "C" {

void ref_gaussian_matrix(int rows, int cols, uint64_t seed, double* out) {
  from_matrix(tatn::gaussian_matrix(rows, cols, seed), out);
}

// standard_forward (reference.cpp:39-100). lse = m + ln(l) (-inf when l == 0).
// counters = {hbm_read_elems, hbm_write_elems, flops}. Returns 0 or -1 on exception.
double ref_dropout_scale(uint64_t seed, long long i, long long j, double p) {
  return tatn::dropout_scale(tatn::DropoutRng{seed}, static_cast<std::size_t>(i), static_cast<std::size_t>(j), p);
}

int ref_standard_forward(int n, int nk, int d, double tau, int mask_kind, int valid_len, const uint8_t* grid, int br,
                         int bc, int tc, double p_drop, uint64_t seed, const double* q, const double* k, const double* v,
                         double* o, double* lse, double* m_out, double* l_out, uint64_t* counters) {
  try {
    const auto cfg = make_cfg(n, d, tau, mask_kind, valid_len, grid, br, bc, tc, p_drop, seed);
    tatn::AccessCounter ctr;
    const auto art = tatn::standard_forward(to_matrix(q, n, d), to_matrix(k, nk, d), to_matrix(v, nk, d), cfg, &ctr);
    from_matrix(art.o, o);
    for (int i = 0; i < n; ++i) {
      const double m = art.stats.m[i], l = art.stats.l[i];
      if (lse) lse[i] = (l > 0.0) ? m + std::log(l) : -std::numeric_limits<double>::infinity();
      if (m_out) m_out[i] = m;
      if (l_out) l_out[i] = l;
    }
    if (counters) {
      counters[0] = ctr.hbm_read_elems;
      counters[1] = ctr.hbm_write_elems;
      counters[2] = ctr.flops;
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// standard_backward (reference.cpp:102-204) on the artifacts of standard_forward.
int ref_standard_backward(int n, int nk, int d, double tau, int mask_kind, int valid_len, const uint8_t* grid, int br,
                          int bc, int tc, double p_drop, uint64_t seed, const double* q, const double* k, const double* v,
                          const double* dO, double* dq, double* dk, double* dv, uint64_t* counters) {
  try {
    const auto cfg = make_cfg(n, d, tau, mask_kind, valid_len, grid, br, bc, tc, p_drop, seed);
    const auto Q = to_matrix(q, n, d), K = to_matrix(k, nk, d), V = to_matrix(v, nk, d);
    const auto art = tatn::standard_forward(Q, K, V, cfg, nullptr);
    tatn::AccessCounter ctr;
    const auto g = tatn::standard_backward(art, Q, K, V, to_matrix(dO, n, d), cfg, &ctr);
    from_matrix(g.dq, dq);
    from_matrix(g.dk, dk);
    from_matrix(g.dv, dv);
    if (counters) {
      counters[0] = ctr.hbm_read_elems;
      counters[1] = ctr.hbm_write_elems;
      counters[2] = ctr.flops;
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// memeff_forward / memeff_backward (reference.cpp:206-326), O(n) memory.
int ref_memeff_forward(int n, int nk, int d, double tau, int mask_kind, int valid_len, const double* q,
                       const double* k, const double* v, double* o, double* lse) {
  try {
    const auto cfg = make_cfg(n, d, tau, mask_kind, valid_len, nullptr, 0, 0, 0);
    const auto r = tatn::memeff_forward(to_matrix(q, n, d), to_matrix(k, nk, d), to_matrix(v, nk, d), cfg, nullptr);
    from_matrix(r.o, o);
    for (int i = 0; i < n; ++i)
      lse[i] = (r.stats.l[i] > 0.0) ? r.stats.m[i] + std::log(r.stats.l[i]) : -std::numeric_limits<double>::infinity();
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_memeff_backward(int n, int nk, int d, double tau, int mask_kind, int valid_len, const double* q,
                        const double* k, const double* v, const double* o, const double* dO, const double* m,
                        const double* l, double* dq, double* dk, double* dv) {
  try {
    const auto cfg = make_cfg(n, d, tau, mask_kind, valid_len, nullptr, 0, 0, 0);
    tatn::SoftmaxStats st(n);
    for (int i = 0; i < n; ++i) {
      st.m[i] = m[i];
      st.l[i] = l[i];
    }
    const auto g = tatn::memeff_backward(to_matrix(q, n, d), to_matrix(k, nk, d), to_matrix(v, nk, d),
                                         to_matrix(o, n, d), to_matrix(dO, n, d), st, cfg, nullptr);
    from_matrix(g.dq, dq);
    from_matrix(g.dk, dk);
    from_matrix(g.dv, dv);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// CPU baseline: run the reference's forward+backward on `nslices` independent
// (b, h) slices of N(0,1) inputs, one std::thread per slice up to `nthreads`
// (SPEC.md:288 allows concurrent heads). memeff != 0 selects memeff_* (O(n)
// memory, for n >= 8K); otherwise standard_*. Inputs are generated before the
// clock starts. Returns wall seconds of the timed fwd+bwd, or -1 on error.
double ref_time_fwd_bwd(int nslices, int n, int d, int mask_kind, int memeff, int nthreads) {
  struct Slice {
    tatn::Matrix q, k, v, dO;
  };
  std::vector<Slice> sl(nslices);
  for (int s = 0; s < nslices; ++s) {
    sl[s].q = tatn::gaussian_matrix(n, d, 1000 + 4 * s + 0);
    sl[s].k = tatn::gaussian_matrix(n, d, 1000 + 4 * s + 1);
    sl[s].v = tatn::gaussian_matrix(n, d, 1000 + 4 * s + 2);
    sl[s].dO = tatn::gaussian_matrix(n, d, 1000 + 4 * s + 3);
  }
  const auto cfg = make_cfg(n, d, 1.0 / std::sqrt(static_cast<double>(d)), mask_kind, n, nullptr, 0, 0, 0);
  std::vector<int> err(nslices, 0);
  auto work = [&](int s) {
    try {
      if (memeff) {
        const auto f = tatn::memeff_forward(sl[s].q, sl[s].k, sl[s].v, cfg, nullptr);
        const auto g = tatn::memeff_backward(sl[s].q, sl[s].k, sl[s].v, f.o, sl[s].dO, f.stats, cfg, nullptr);
        (void)g;
      } else {
        const auto a = tatn::standard_forward(sl[s].q, sl[s].k, sl[s].v, cfg, nullptr);
        const auto g = tatn::standard_backward(a, sl[s].q, sl[s].k, sl[s].v, sl[s].dO, cfg, nullptr);
        (void)g;
      }
    } catch (const std::exception&) {
      err[s] = 1;
    }
  };
  if (nthreads < 1) nthreads = 1;
  const auto t0 = std::chrono::steady_clock::now();
  for (int base = 0; base < nslices; base += nthreads) {
    std::vector<std::thread> th;
    for (int s = base; s < nslices && s < base + nthreads; ++s) th.emplace_back(work, s);
    for (auto& t : th) t.join();
  }
  const auto t1 = std::chrono::steady_clock::now();
  for (int e : err)
    if (e) return -1.0;
  return std::chrono::duration<double>(t1 - t0).count();
}


// The reference's matrix_io (matrix_io.cpp): write rows x cols binary64 values as TATN binary
// (binary != 0) or 17-digit CSV to `path`; read one back into `out` (capacity rows*cols).
int ref_write_matrix(const char* path, int binary, int rows, int cols, const double* data) {
  try {
    const auto m = to_matrix(data, rows, cols);
    if (binary) tatn::write_matrix_binary(m, std::string(path));
    else tatn::write_matrix_csv(m, std::string(path));
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}
int ref_read_matrix(const char* path, int binary, int* rows, int* cols, double* out, long long capacity) {
  try {
    const auto m = binary ? tatn::read_matrix_binary(std::string(path)) : tatn::read_matrix_csv(std::string(path));
    *rows = static_cast<int>(m.rows());
    *cols = static_cast<int>(m.cols());
    if (static_cast<long long>(m.rows() * m.cols()) > capacity) return -2;
    from_matrix(m, out);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}
}  // extern "C"
