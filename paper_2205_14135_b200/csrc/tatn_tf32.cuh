// tatn_tf32.cuh — fp32-input check mode (TATN_DTYPE_FP32): forward and backward on
// tcgen05.mma kind::tf32.
//
// The reference computes in binary64 on fp64 carriers (matrix.hpp:11-14) and its
// CPU oracle shape C1 (BASELINE configs[0]) is fp32. These kernels take fp32 Q, K, V, dO as
// they are (no 16-bit rounding of the inputs): TMA streams fp32 tiles (128-byte swizzle, 32
// columns per atom), the tensor cores read them as tf32 and accumulate in fp32 in TMEM. The
// inputs are rounded to tf32 in shared memory (round to nearest: the tensor core itself would
// truncate, a bias towards zero), the operands produced on chip — P, dS — likewise before the
// MMAs read them, and the softmax normaliser l sums the rounded P, so O is an exact weighted
// mean of V under the weights the MMA saw. Same algorithm as K1 / K3 (Algorithm 2 and 4, PAPER.md:
// 1239-1271, 1324-1372; flash.hpp:43-73), same masks (causal, key padding, custom, block grid,
// key offset), same positional dropout (dropout.cpp:7-27), same outputs (O, LSE; dQ via the
// fp32 workspace accumulator and K4; dK, dV direct).
//
// Shared-memory layouts. A tf32 operand that is contracted over its rows (MN-major: V in
// P V; Q, dO, K and dS^T in the backward's dV, dK, dQ products) must use the 128-byte swizzle
// with 32-byte atoms (descriptor layout type 1, TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B: 32-byte
// granule g of 128-byte row r sits at g ^ (r & 3)); K-major operands use the ordinary 128-byte
// swizzle (16-byte granule j at j ^ (r & 7)). The same [rows][d] tile is needed both ways in
// the backward, so Q and dO are re-swizzled in place once the S^T / dP^T MMAs have read them,
// and K is loaded twice.
//
// This is a check mode, not a throughput path: one CTA per tile, 128 threads, each step
// waited before the next (thread = TMEM lane = row; thread 0 issues TMA and MMA).
//   forward  : grid (Q tiles of 128 rows, H, B); per key tile S = Q K^T, softmax in registers,
//              P (tf32) written over S in TMEM, O += P V with A from TMEM.
//   backward : grid (key tiles of 128, H, B); V in TMEM; per Q tile of QT rows (128 at d = 64,
//              32 at d = 128): S^T = K Q^T, dP^T = V dO^T (A from TMEM); P^T, dS^T written
//              over them in TMEM and dS^T to shared memory; dV += P^T dO, dK += dS^T Q (A from
//              TMEM), and dQ = dS K (d = 64) / dQ^T = K^T dS^T (d = 128), both M = 128, added
//              to the fp32 workspace with red.global.add.
#pragma once

#include <cuda_runtime.h>

#include <cmath>

#include "sm100_ptx.cuh"
#include "tatn_params.h"

namespace tatn_dev {

constexpr int kTf32Threads = 128;
constexpr uint32_t kFmtTf32 = 2;  // instruction-descriptor a/b format

// A fp32 tile of `rows` rows x D columns is stored as D/32 column blocks of rows x 128 bytes.
// K-major operand (K = the tile's columns), 128-byte swizzle: k-step kk (8 columns) starts at
// block kk / 4, byte (kk % 4) * 32 of each row; 8-row groups 1024 bytes apart.
__device__ __forceinline__ uint64_t tf32_kmajor(uint32_t base, int rows, int kk) {
  return make_sdesc_sw128(base + static_cast<uint32_t>((kk >> 2) * rows * 128 + (kk & 3) * 32), 16, 1024);
}
// MN-major operand (MN = the tile's columns, K = its rows), 128-byte swizzle with 32-byte atoms
// (layout type 1): k-step kk (8 rows) starts 8 rows down; 4-row groups 512 bytes apart (stride
// byte offset); column blocks `rows * 128` bytes apart (leading byte offset).
__device__ __forceinline__ uint64_t tf32_mnmajor(uint32_t base, int rows, int kk) {
  uint64_t d = make_sdesc_sw128(base + static_cast<uint32_t>(kk * 1024), static_cast<uint32_t>(rows * 128), 512);
  return (d & ~(static_cast<uint64_t>(7) << 61)) | (static_cast<uint64_t>(1) << 61);
}
// byte offset of 16-byte granule j (0..7) of row r in a 128-byte row, per layout
__device__ __forceinline__ uint32_t sw128_off(int r, int j) { return static_cast<uint32_t>(r * 128 + ((j ^ (r & 7)) << 4)); }
__device__ __forceinline__ uint32_t sw32b_off(int r, int j) {
  return static_cast<uint32_t>(r * 128 + (((((j >> 1) ^ (r & 3)) << 1) | (j & 1)) << 4));
}
// Round a shared-memory fp32 tile to tf32 in place (round to nearest, ties away), by the 128
// threads of the CTA. The tensor core would otherwise drop the 13 low mantissa bits of each
// fp32 input (truncation: a bias towards zero that shows up as a systematically low LSE);
// rounded inputs are read exactly and their errors are unbiased.
__device__ __forceinline__ void tf32_round_smem(uint32_t base, int bytes) {
  for (int u = static_cast<int>(threadIdx.x); u < bytes / 16; u += kTf32Threads) {
    const uint32_t a = base + static_cast<uint32_t>(u * 16);
    float x, y, z, w;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
    st_shared_v4(a, __float_as_uint(round_tf32(x)), __float_as_uint(round_tf32(y)), __float_as_uint(round_tf32(z)),
                 __float_as_uint(round_tf32(w)));
  }
}
// In-place re-swizzle of a rows x D fp32 tile from the K-major (128B) to the MN-major (128B,
// 32B atoms) layout, by the 128 threads of the CTA (named barrier 1 between reads and writes).
template <int D, int ROWS>
__device__ __forceinline__ void tf32_reswizzle(uint32_t base) {
  constexpr int kUnits = ROWS * D / 4 / 128;  // 16-byte units per thread
  uint4 v[kUnits];
#pragma unroll
  for (int i = 0; i < kUnits; ++i) {
    const int u = static_cast<int>(threadIdx.x) + 128 * i;
    const int c = u / (ROWS * 8), r = (u / 8) % ROWS, j = u % 8;
    const uint32_t a = base + static_cast<uint32_t>(c * ROWS * 128) + sw128_off(r, j);
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w) : "r"(a));
  }
  named_bar_sync(1, kTf32Threads);
#pragma unroll
  for (int i = 0; i < kUnits; ++i) {
    const int u = static_cast<int>(threadIdx.x) + 128 * i;
    const int c = u / (ROWS * 8), r = (u / 8) % ROWS, j = u % 8;
    st_shared_v4(base + static_cast<uint32_t>(c * ROWS * 128) + sw32b_off(r, j), v[i].x, v[i].y, v[i].z, v[i].w);
  }
}

// TMA load of a rows x D fp32 tile (D/32 boxes of 32 columns) at (row r0, head h, batch b).
template <int D>
__device__ __forceinline__ void tf32_load_tile(uint32_t dst, const void* tmap, uint32_t bar, int rows, int r0, int h,
                                               int b) {
#pragma unroll
  for (int c = 0; c < D / 32; ++c) tma_load_4d(dst + static_cast<uint32_t>(c * rows * 128), tmap, bar, 32 * c, r0, h, b);
}

// keep bit of (query row qi, global key kg) in the Custom mask of batch element b
__device__ __forceinline__ bool custom_keep(const uint32_t* m, int words, int64_t bstride, int b, int qi, int kg) {
  return (m[static_cast<size_t>(b) * bstride + static_cast<size_t>(qi) * words + (kg >> 5)] >> (kg & 31)) & 1u;
}

// ---------------------------------------------------------------- forward
template <int D>
struct Tf32FwdCfg {
  static constexpr int kTile = (D / 32) * 128 * 128;  // 128 rows x D fp32
  static constexpr int kOffQ = 0, kOffK = kTile, kOffV = 2 * kTile, kOffBar = 3 * kTile;
  static constexpr int kSmemBytes = kOffBar + 64 + 1024;  // + alignment slack
  static constexpr uint32_t kTmemS = 0, kTmemO = 128, kTmemCols = 256;
};

template <int D, bool DROP>
__global__ void __launch_bounds__(kTf32Threads, 1)
    tatn_fwd_tf32_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, const FwdParams p) {
  using Cfg = Tf32FwdCfg<D>;
#ifdef TATN_TRACE  // per-step stamps of CTA (0, 0, 0) (trace builds only)
  unsigned long long* const tatn_ev_buf = (blockIdx.x | blockIdx.y | blockIdx.z) == 0 ? g_tatn_trace : nullptr;
  if (threadIdx.x == 0) TATN_EV(0, 7);
#endif
  extern __shared__ uint8_t smem_raw[];
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));
  const uint32_t sQ = smem_base + Cfg::kOffQ, sK = smem_base + Cfg::kOffK, sV = smem_base + Cfg::kOffV;
  const uint32_t bar0 = smem_base + Cfg::kOffBar;
  const uint32_t kBarQ = bar0, kBarK = bar0 + 8, kBarV = bar0 + 16, kBarS = bar0 + 24, kBarO = bar0 + 32;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_gen + Cfg::kOffBar + 48);
  const int warp = static_cast<int>(warp_id()), lane = static_cast<int>(lane_id());
  const int r = warp * 32 + lane;  // query row within the tile == TMEM lane
  const bool leader = threadIdx.x == 0;
  const int qt = static_cast<int>(blockIdx.x), h = static_cast<int>(blockIdx.y), b = static_cast<int>(blockIdx.z);
  const int q0 = qt * 128;
  const int bh = b * p.H + h;

  if (leader) {
    for (int i = 0; i < 5; ++i) mbar_init(bar0 + 8 * i, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(smem_u32(tmem_slot), Cfg::kTmemCols);
    tmem_relinquish();
  }
  griddep_wait();
  if (threadIdx.x == 0) TATN_EV(0, 5);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  const uint32_t tS = tmem_base + lane_off + Cfg::kTmemS, tO = tmem_base + lane_off + Cfg::kTmemO;

  // key tiles of this Q tile (the same schedule as K1: key padding / causal bound the dense
  // range; a block grid visits exactly its nonzero blocks)
  int kv_limit = p.Nk;
  if (p.mask_kind == kMaskKeyPadding && p.valid_len != nullptr) kv_limit = min(kv_limit, max(p.valid_len[b] - p.k_off, 0));
  const bool sparse = p.grid != nullptr;
  int T = (kv_limit + 127) / 128;
  if (p.mask_kind == kMaskCausal) {
    const int last = q0 + 127 - p.k_off;
    T = min(T, last >= 0 ? last / 128 + 1 : 0);
  }
  const uint8_t* grow_ptr = sparse ? p.grid + static_cast<size_t>(qt) * p.tc : nullptr;
  if (sparse) T = p.tc;
  auto next_tile = [&](int t) {
    if (sparse)
      while (t < T && grow_ptr[t] == 0) ++t;
    return t;
  };

  const int qi = q0 + r;  // global query row
  const bool causal = p.mask_kind == kMaskCausal;
  const bool custom_on = p.mask_kind == kMaskCustom && p.custom != nullptr;
  uint64_t drow = 0;
  if constexpr (DROP) drow = drop_row_hash(p.drop_seed + static_cast<uint64_t>(bh), qi);
  const float sl2 = p.scale_log2;
  float m_run = -INFINITY, l_run = 0.f;

  int t = next_tile(0);
  if (leader) {
    mbar_expect_tx(kBarQ, Cfg::kTile);
    tf32_load_tile<D>(sQ, &tmQ, kBarQ, 128, q0, h, b);
    if (t < T) {
      mbar_expect_tx(kBarK, Cfg::kTile);
      tf32_load_tile<D>(sK, &tmK, kBarK, 128, t * 128, h, b);
      mbar_expect_tx(kBarV, Cfg::kTile);
      tf32_load_tile<D>(sV, &tmV, kBarV, 128, t * 128, h, b);
    }
  }
  mbar_wait(kBarQ, 0);
  if (threadIdx.x == 0) TATN_EV(0, 6);
  tf32_round_smem(sQ, Cfg::kTile);
  constexpr uint32_t idesc_qk = make_idesc_f16(kFmtTf32, 128, 128, 0, 0);
  constexpr uint32_t idesc_pv = make_idesc_f16(kFmtTf32, 128, D, 0, 1);
  int n = 0;  // tiles done
  for (; t < T; ++n) {
    const int tn = next_tile(t + 1);
    const uint32_t ph = static_cast<uint32_t>(n & 1);
    mbar_wait(kBarK, ph);
    if (threadIdx.x == 0) TATN_EV(n, 1);
    tf32_round_smem(sK, Cfg::kTile);
    fence_proxy_async_smem();  // the rounded tiles are read by the tensor core (async proxy)
    named_bar_sync(1, kTf32Threads);
    if (leader) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < D / 8; ++kk)
        mma_ss_tf32(tmem_base + Cfg::kTmemS, tf32_kmajor(sQ, 128, kk), tf32_kmajor(sK, 128, kk), idesc_qk,
                    kk > 0 ? 1u : 0u);
      mma_commit(kBarS);
      if (p.visited != nullptr) {
        const long long bit = static_cast<long long>(qt) * p.tc + t;
        atomicOr(p.visited + (bit >> 5), 1u << (bit & 31));
      }
    }
    mbar_wait(kBarS, ph);
    if (threadIdx.x == 0) TATN_EV(n, 2);
    tc_fence_after();
    if (leader && tn < T) {  // K buffer free (the QK MMA completed): prefetch the next K tile
      mbar_expect_tx(kBarK, Cfg::kTile);
      tf32_load_tile<D>(sK, &tmK, kBarK, 128, tn * 128, h, b);
    }
    const int k0 = t * 128;
    uint4 cw = make_uint4(~0u, ~0u, ~0u, ~0u);  // Custom mask: the row's keep bits of this key tile
    if (custom_on) {
      cw = make_uint4(0u, 0u, 0u, 0u);
      if (qi < p.Nq)
        cw = *reinterpret_cast<const uint4*>(p.custom + static_cast<size_t>(b) * p.custom_bstride +
                                             static_cast<size_t>(qi) * p.custom_words + (p.k_off + k0) / 32);
    }
    const uint32_t cwa[4] = {cw.x, cw.y, cw.z, cw.w};
    // Only tiles that reach past the key limit, cross the causal diagonal or carry a Custom mask
    // need the per-element predicate (uniform over the CTA: it depends on the tile, not the row).
    const bool need_mask = (k0 + 128 > kv_limit) || (causal && p.k_off + k0 + 127 > q0) || custom_on;
    // scaled score of column 32 c + i (log2 domain), -inf where masked
    auto score = [&](int c, int i, uint32_t raw) {
      const int kj = k0 + 32 * c + i;
      const bool masked = kj >= kv_limit || (causal && p.k_off + kj > qi) || ((cwa[c] >> i) & 1u) == 0u;
      return masked ? -INFINITY : __uint_as_float(raw) * sl2;
    };
    // pass 1: row max over the tile (S stays in TMEM; pass 2 reads it again). Four independent
    // partial maxima / sums: with one warp per SM sub-partition a single 128-long dependency chain
    // (fmax, then add) was the softmax's critical path (traced: ~15K cycles per tile)
    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      tmem_ld32(tS + 32 * c, v);
      if (need_mask) {
#pragma unroll
        for (int i = 0; i < 32; ++i) m4[i & 3] = fmaxf(m4[i & 3], score(c, i, v[i]));
      } else {  // sl2 > 0: scale the maximum once
#pragma unroll
        for (int i = 0; i < 32; ++i) m4[i & 3] = fmaxf(m4[i & 3], __uint_as_float(v[i]));
      }
    }
    float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    if (!need_mask) mx *= sl2;
    const float m_new = fmaxf(m_run, mx);
    const bool grow = m_new > m_run;
    const float alpha = grow ? ex2_approx(m_run - m_new) : 1.f;  // 0 when m_run == -inf
    if (grow) {
      m_run = m_new;
      l_run *= alpha;
    }
    if (n > 0 && __any_sync(0xffffffffu, grow)) {  // O holds PV(n-1) (waited below): rescale it exactly
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + 32 * c, o);
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
        tmem_st32(tO + 32 * c, o);
      }
    }
    const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
    // pass 2: P = 2^(s - m) rounded to tf32, written over S (the A operand of P V)
    float l4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      tmem_ld32(tS + 32 * c, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float x = need_mask ? score(c, i, v[i]) - m_use : fmaf(__uint_as_float(v[i]), sl2, -m_use);
        const float pv = round_tf32(ex2_approx(x));
        l4[i & 3] += pv;
        float pm = pv;
        if constexpr (DROP) pm = drop_keep(drow, p.k_off + k0 + 32 * c + i, p.drop_thresh) ? round_tf32(pv * p.drop_scale) : 0.f;
        v[i] = __float_as_uint(pm);
      }
      tmem_st32(tS + 32 * c, v);
    }
    l_run += (l4[0] + l4[1]) + (l4[2] + l4[3]);
    mbar_wait(kBarV, ph);
    tf32_round_smem(sV, Cfg::kTile);
    fence_proxy_async_smem();
    tmem_st_wait();
    tc_fence_before();
    named_bar_sync(1, kTf32Threads);
    if (threadIdx.x == 0) TATN_EV(n, 3);
    if (leader) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 128 / 8; ++kk)
        mma_ts_tf32(tmem_base + Cfg::kTmemO, tmem_base + Cfg::kTmemS + 8 * kk, tf32_mnmajor(sV, 128, kk), idesc_pv,
                    (n > 0 || kk > 0) ? 1u : 0u);
      mma_commit(kBarO);
    }
    mbar_wait(kBarO, ph);
    if (threadIdx.x == 0) TATN_EV(n, 4);
    tc_fence_after();
    if (leader && tn < T) {  // V buffer free: prefetch the next V tile
      mbar_expect_tx(kBarV, Cfg::kTile);
      tf32_load_tile<D>(sV, &tmV, kBarV, 128, tn * 128, h, b);
    }
    t = tn;
  }
  // epilogue: O / l (fp32) straight to global, LSE = ln(sum_j e^{s_j}) (-inf, O = 0 for empty rows).
  // TMEM loads are warp-collective: every thread loads, rows past Nq just do not store.
  const float inv_l = l_run > 0.f ? 1.f / l_run : 0.f;
  float* orow = p.o_f32 + static_cast<size_t>(b) * p.o_sb + static_cast<size_t>(h) * p.o_sh +
                static_cast<size_t>(qi) * p.o_sn;
#pragma unroll
  for (int c = 0; c < D / 32; ++c) {
    uint32_t o[32];
    if (n > 0) tmem_ld32(tO + 32 * c, o);  // n is uniform over the CTA
    if (qi < p.Nq) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
        if (n > 0)
          w = make_float4(__uint_as_float(o[4 * i]) * inv_l, __uint_as_float(o[4 * i + 1]) * inv_l,
                          __uint_as_float(o[4 * i + 2]) * inv_l, __uint_as_float(o[4 * i + 3]) * inv_l);
        reinterpret_cast<float4*>(orow + 32 * c)[i] = w;
      }
    }
  }
  if (qi < p.Nq)
    p.lse[static_cast<size_t>(bh) * p.Nq + qi] =
        l_run > 0.f ? (m_run + log2f(l_run)) * 0.69314718055994530942f : -INFINITY;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

// ---------------------------------------------------------------- backward (K3, tf32)
template <int D>
struct Tf32BwdCfg {
  static constexpr int QT = (D == 64) ? 128 : 32;          // query rows per Q tile
  static constexpr int kKV = (D / 32) * 128 * 128;         // 128 keys x D fp32
  static constexpr int kQ = (D / 32) * QT * 128;           // QT rows x D fp32
  static constexpr int kDS = (QT / 32) * 128 * 128;        // dS^T: 128 keys x QT fp32
  // K (K-major, for S^T = K Q^T), K (MN-major, for dQ), Q, dO, dS^T (MN-major)
  static constexpr int kOffK = 0, kOffKmn = kKV, kOffQ = 2 * kKV, kOffDO = kOffQ + kQ, kOffDS = kOffDO + kQ;
  static constexpr int kOffVec = kOffDS + kDS;             // -lse2, -D of the tile's rows
  static constexpr int kOffDrop = kOffVec + 2 * QT * 4;    // dropout row hashes
  static constexpr int kOffBar = kOffDrop + QT * 8;
  static constexpr int kSmemBytes = kOffBar + 64 + 1024;
  static_assert(kSmemBytes <= 232448, "tf32 backward shared memory exceeds the opt-in limit");
  // TMEM: V (A operand of dP^T), S^T | P^T, dP^T | dS^T, dV, dK, dQ (d = 64) / dQ^T (d = 128)
  static constexpr uint32_t kTmemV = 0, kTmemS = D, kTmemDP = D + QT, kTmemDV = D + 2 * QT, kTmemDK = 2 * D + 2 * QT,
                            kTmemDQ = 3 * D + 2 * QT, kTmemCols = 512;
  static_assert(kTmemDQ + (D == 64 ? D : QT) <= kTmemCols, "TMEM budget");
};

template <int D, bool DROP>
__global__ void __launch_bounds__(kTf32Threads, 1)
    tatn_bwd_tf32_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmKmn, const __grid_constant__ CUtensorMap tmDO,
                         const float* __restrict__ vptr, const BwdParams p, const float* __restrict__ lse2,
                         int Nq_pad) {
  using Cfg = Tf32BwdCfg<D>;
  constexpr int QT = Cfg::QT;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));
  const uint32_t sK = smem_base + Cfg::kOffK, sKmn = smem_base + Cfg::kOffKmn, sQ = smem_base + Cfg::kOffQ;
  const uint32_t sDO = smem_base + Cfg::kOffDO, sDS = smem_base + Cfg::kOffDS;
  float* vec = reinterpret_cast<float*>(smem_gen + Cfg::kOffVec);  // [0, QT): -lse2, [QT, 2QT): -D
  uint64_t* drows = reinterpret_cast<uint64_t*>(smem_gen + Cfg::kOffDrop);
  const uint32_t bar0 = smem_base + Cfg::kOffBar;
  const uint32_t kBarKV = bar0, kBarQ = bar0 + 8, kBarS = bar0 + 16, kBarB = bar0 + 24;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_gen + Cfg::kOffBar + 48);
  const int warp = static_cast<int>(warp_id()), lane = static_cast<int>(lane_id());
  const int r = warp * 32 + lane;  // key row within the tile == TMEM lane
  const bool leader = threadIdx.x == 0;
  const int j = static_cast<int>(blockIdx.x), h = static_cast<int>(blockIdx.y), b = static_cast<int>(blockIdx.z);
  const int k0 = j * 128, kj = k0 + r;
  const int bh = b * p.H + h;

  if (leader) {
    for (int i = 0; i < 4; ++i) mbar_init(bar0 + 8 * i, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(smem_u32(tmem_slot), Cfg::kTmemCols);
    tmem_relinquish();
  }
  griddep_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  const uint32_t tS = tmem_base + lane_off + Cfg::kTmemS, tDP = tmem_base + lane_off + Cfg::kTmemDP;

  int kv_limit = p.Nk;
  if (p.mask_kind == kMaskKeyPadding && p.valid_len != nullptr) kv_limit = min(kv_limit, max(p.valid_len[b] - p.k_off, 0));
  const bool sparse = p.grid != nullptr;
  const bool causal = p.mask_kind == kMaskCausal;
  const bool custom_on = p.mask_kind == kMaskCustom && p.custom != nullptr;
  const int n_qt = (p.Nq + QT - 1) / QT;
  int i_begin = 0, i_end = n_qt;
  if (!sparse) {
    if (causal) i_begin = min((k0 + p.k_off) / QT, n_qt);
    if (k0 >= kv_limit) i_end = i_begin;
  }
  auto next_q = [&](int i) {
    if (sparse)
      while (i < i_end && p.grid[static_cast<size_t>(i * QT / 128) * p.tc + j] == 0) ++i;
    return i;
  };
  const float sl2 = p.scale_log2;
  const float* lse2_bh = lse2 + static_cast<size_t>(bh) * Nq_pad;
  const float* delta_bh = p.delta + static_cast<size_t>(bh) * Nq_pad;

  if (leader) {
    mbar_expect_tx(kBarKV, 2 * Cfg::kKV);
    tf32_load_tile<D>(sK, &tmK, kBarKV, 128, k0, h, b);
    tf32_load_tile<D>(sKmn, &tmKmn, kBarKV, 128, k0, h, b);
  }
  {  // V row kj -> TMEM lane r (the A operand of dP^T = V dO^T); rows past Nk are zero
    const float* vrow = vptr + static_cast<size_t>(b) * p.v_sb + static_cast<size_t>(h) * p.v_sh +
                        static_cast<size_t>(min(kj, p.Nk - 1)) * p.v_sn;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t v[32];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
        if (kj < p.Nk) w = reinterpret_cast<const float4*>(vrow + 32 * c)[e];
        v[4 * e] = __float_as_uint(round_tf32(w.x));
        v[4 * e + 1] = __float_as_uint(round_tf32(w.y));
        v[4 * e + 2] = __float_as_uint(round_tf32(w.z));
        v[4 * e + 3] = __float_as_uint(round_tf32(w.w));
      }
      tmem_st32(tmem_base + lane_off + Cfg::kTmemV + 32 * c, v);
    }
    tmem_st_wait();
  }
  mbar_wait(kBarKV, 0);
  tf32_round_smem(sK, 2 * Cfg::kKV);  // K (K-major) and K (MN-major) are adjacent
  fence_proxy_async_smem();
  tc_fence_before();
  named_bar_sync(1, kTf32Threads);
  constexpr uint32_t idesc_front = make_idesc_f16(kFmtTf32, 128, QT, 0, 0);  // S^T, dP^T
  constexpr uint32_t idesc_acc = make_idesc_f16(kFmtTf32, 128, D, 0, 1);     // dV, dK (B MN-major)
  // dQ: d = 64 -> dQ = dS K (M = QT = 128 queries, N = 64); d = 128 -> dQ^T = K^T dS^T (M = 128, N = QT)
  constexpr uint32_t idesc_dq = make_idesc_f16(kFmtTf32, 128, D == 64 ? D : QT, 1, 1);
  int n = 0;
  for (int i = next_q(i_begin); i < i_end; i = next_q(i + 1), ++n) {
    const uint32_t ph = static_cast<uint32_t>(n & 1);
    const int i0 = i * QT;
    if (leader) {
      mbar_expect_tx(kBarQ, 2 * Cfg::kQ);
      tf32_load_tile<D>(sQ, &tmQ, kBarQ, QT, i0, h, b);
      tf32_load_tile<D>(sDO, &tmDO, kBarQ, QT, i0, h, b);
      if (p.visited != nullptr) {
        const long long bit = static_cast<long long>(i0 / 128) * p.tc + j;
        atomicOr(p.visited + (bit >> 5), 1u << (bit & 31));
      }
    }
    if (r < QT) {  // the tile's row vectors (rows past Nq have -lse2 = -inf: P = 0)
      vec[r] = lse2_bh[i0 + r];
      vec[QT + r] = delta_bh[i0 + r];
      if constexpr (DROP) drows[r] = drop_row_hash(p.drop_seed + static_cast<uint64_t>(bh), i0 + r);
    }
    mbar_wait(kBarQ, ph);
    tf32_round_smem(sQ, 2 * Cfg::kQ);  // Q and dO are adjacent
    fence_proxy_async_smem();
    named_bar_sync(1, kTf32Threads);
    if (leader) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < D / 8; ++kk) {
        mma_ss_tf32(tmem_base + Cfg::kTmemS, tf32_kmajor(sK, 128, kk), tf32_kmajor(sQ, QT, kk), idesc_front,
                    kk > 0 ? 1u : 0u);
        mma_ts_tf32(tmem_base + Cfg::kTmemDP, tmem_base + Cfg::kTmemV + 8 * kk, tf32_kmajor(sDO, QT, kk), idesc_front,
                    kk > 0 ? 1u : 0u);
      }
      mma_commit(kBarS);
    }
    mbar_wait(kBarS, ph);
    tc_fence_after();
    // the fronts have read Q and dO as K-major operands: re-swizzle them for dK / dV (MN-major)
    tf32_reswizzle<D, QT>(sQ);
    tf32_reswizzle<D, QT>(sDO);
    named_bar_sync(1, kTf32Threads);  // row vectors staged, re-swizzle done
    // only tiles that reach past the key limit, cross the causal diagonal or carry a Custom mask
    // evaluate the per-element predicate (uniform over the CTA for this Q tile)
    const bool need_mask = (k0 + 128 > kv_limit) || (causal && p.k_off + k0 + 127 > i0) || custom_on;
#pragma unroll 1
    for (int cc = 0; cc < QT / 32; ++cc) {
      uint32_t sv[32], dv[32];
      tmem_ld32(tS + 32 * cc, sv);
      tmem_ld32(tDP + 32 * cc, dv);
      uint32_t pk[32], dk[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const int c = 32 * cc + e;
        const int qi = i0 + c;
        const int kg = p.k_off + kj;
        float pv = ex2_approx(fmaf(__uint_as_float(sv[e]), sl2, vec[c]));
        if (need_mask) {  // rows past Nq need no predicate: their -lse2 = -inf gives P = 0
          const bool masked = kj >= kv_limit || (causal && kg > qi) ||
                              (custom_on && (qi >= p.Nq || !custom_keep(p.custom, p.custom_words, p.custom_bstride, b, qi, kg)));
          pv = masked ? 0.f : pv;
        }
        const float dpv = __uint_as_float(dv[e]);
        if constexpr (DROP) {  // dP through the mask, dV from P * Z / (1 - p) (reference.cpp:118-141)
          const float z = drop_keep(drows[c], kg, p.drop_thresh) ? p.drop_scale : 0.f;
          pk[e] = __float_as_uint(round_tf32(pv * z));
          dk[e] = __float_as_uint(round_tf32(pv * fmaf(dpv, z, vec[QT + c])));
        } else {
          pk[e] = __float_as_uint(round_tf32(pv));
          dk[e] = __float_as_uint(round_tf32(pv * (dpv + vec[QT + c])));
        }
      }
      tmem_st32(tS + 32 * cc, pk);
      tmem_st32(tDP + 32 * cc, dk);
      // dS^T -> shared memory [key][QT queries], MN-major layout (32-byte atoms), column block cc
      const uint32_t blk = sDS + static_cast<uint32_t>(cc * 128 * 128);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        st_shared_v4(blk + sw32b_off(r, u), dk[4 * u], dk[4 * u + 1], dk[4 * u + 2], dk[4 * u + 3]);
    }
    fence_proxy_async_smem();
    tmem_st_wait();
    tc_fence_before();
    named_bar_sync(1, kTf32Threads);
    if (leader) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < QT / 8; ++kk) {
        mma_ts_tf32(tmem_base + Cfg::kTmemDV, tmem_base + Cfg::kTmemS + 8 * kk, tf32_mnmajor(sDO, QT, kk), idesc_acc,
                    (n > 0 || kk > 0) ? 1u : 0u);
        mma_ts_tf32(tmem_base + Cfg::kTmemDK, tmem_base + Cfg::kTmemDP + 8 * kk, tf32_mnmajor(sQ, QT, kk), idesc_acc,
                    (n > 0 || kk > 0) ? 1u : 0u);
      }
#pragma unroll
      for (int kk = 0; kk < 128 / 8; ++kk) {
        if constexpr (D == 64)  // dQ = dS K: A = dS^T buffer (MN-major: queries), B = K (MN-major: d)
          mma_ss_tf32(tmem_base + Cfg::kTmemDQ, tf32_mnmajor(sDS, 128, kk), tf32_mnmajor(sKmn, 128, kk), idesc_dq,
                      kk > 0 ? 1u : 0u);
        else  // dQ^T = K^T dS^T: A = K (MN-major: d), B = dS^T buffer (MN-major: queries)
          mma_ss_tf32(tmem_base + Cfg::kTmemDQ, tf32_mnmajor(sKmn, 128, kk), tf32_mnmajor(sDS, 128, kk), idesc_dq,
                      kk > 0 ? 1u : 0u);
      }
      mma_commit(kBarB);
    }
    mbar_wait(kBarB, ph);
    tc_fence_after();
    // dQ partial (tau applied) -> the fp32 workspace accumulator (red.global.add), or in the
    // deterministic mode this key tile's own slot (plain stores; K4 sums the slots in j order)
    const uint32_t tDQ = tmem_base + lane_off + Cfg::kTmemDQ;
    const bool det = p.dq_part != nullptr;
    float* acc = det ? p.dq_part + (static_cast<size_t>(j) * p.B * p.H + bh) * Nq_pad * D
                     : p.dq_acc + static_cast<size_t>(bh) * Nq_pad * D;
    if constexpr (D == 64) {  // thread = query row i0 + r, columns = d
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tDQ + 32 * c, v);
        float* dst = acc + static_cast<size_t>(i0 + r) * D + 32 * c;
        if (det) {
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(dst + e) =
                make_float4(__uint_as_float(v[e]) * p.tau, __uint_as_float(v[e + 1]) * p.tau,
                            __uint_as_float(v[e + 2]) * p.tau, __uint_as_float(v[e + 3]) * p.tau);
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) atomicAdd(dst + e, __uint_as_float(v[e]) * p.tau);
        }
      }
    } else {  // thread = head-dim index r, columns = queries
#pragma unroll
      for (int c = 0; c < QT / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tDQ + 32 * c, v);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float* dst = acc + static_cast<size_t>(i0 + 32 * c + e) * D + r;
          if (det) *dst = __uint_as_float(v[e]) * p.tau;
          else atomicAdd(dst, __uint_as_float(v[e]) * p.tau);
        }
      }
    }
    tc_fence_before();
    named_bar_sync(1, kTf32Threads);  // TMEM / shared buffers free for the next Q tile
  }
  // epilogue: dK = tau * dS^T Q, dV = P^T dO (fp32, zero when no Q tile saw this key tile).
  // TMEM loads are warp-collective: every thread loads, rows past Nk just do not store.
  float* dkr = p.dk_f32 + static_cast<size_t>(b) * p.k_sb + static_cast<size_t>(h) * p.k_sh + static_cast<size_t>(kj) * p.k_sn;
  float* dvr = p.dv_f32 + static_cast<size_t>(b) * p.v_sb + static_cast<size_t>(h) * p.v_sh + static_cast<size_t>(kj) * p.v_sn;
#pragma unroll
  for (int c = 0; c < D / 32; ++c) {
    uint32_t a[32], v[32];
    if (n > 0) {  // n is uniform over the CTA
      tmem_ld32(tmem_base + lane_off + Cfg::kTmemDK + 32 * c, a);
      tmem_ld32(tmem_base + lane_off + Cfg::kTmemDV + 32 * c, v);
    }
    if (kj < p.Nk) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float4 wk = make_float4(0.f, 0.f, 0.f, 0.f), wv = wk;
        if (n > 0) {
          wk = make_float4(__uint_as_float(a[4 * e]) * p.tau, __uint_as_float(a[4 * e + 1]) * p.tau,
                           __uint_as_float(a[4 * e + 2]) * p.tau, __uint_as_float(a[4 * e + 3]) * p.tau);
          wv = make_float4(__uint_as_float(v[4 * e]), __uint_as_float(v[4 * e + 1]), __uint_as_float(v[4 * e + 2]),
                           __uint_as_float(v[4 * e + 3]));
        }
        reinterpret_cast<float4*>(dkr + 32 * c)[e] = wk;
        reinterpret_cast<float4*>(dvr + 32 * c)[e] = wv;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

}  // namespace tatn_dev
