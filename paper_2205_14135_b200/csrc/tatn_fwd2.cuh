// tatn_fwd2.cuh — persistent FlashAttention forward, two Q tiles per item (kernel K1, d = 128).
//
// Same algorithm and ping-pong schedule as tatn_fwd_kernel<D, .., NQ = 2> (Algorithm 2,
// PAPER.md:1239-1271; reference flash.hpp:43-67), restructured as a persistent kernel (one CTA
// per SM) over work items = pairs of 128-row Q tiles of one head, claimed from a self-resetting
// device counter and published to the roles through a shared-memory ring:
//   * the K/V ring, its mbarrier phases and the MMA tile stream continue across items, so the
//     next item's first K/V tiles are prefetched under the current item's last tiles;
//   * the Q pair is reloaded as soon as every QK of the previous item has completed (QFree), and
//     O goes from registers straight to global memory, so Q shared memory is never staging;
//   * each softmax warpgroup writes its tile's O and LSE and moves to the next item, whose S is
//     computed meanwhile; no CTA launch, TMEM allocation or barrier set-up per item.
#pragma once

#include "tatn_fwd.cuh"

namespace tatn_dev {

template <int D>
struct Fwd2Cfg {
  static constexpr int kSubs = D / 64;
  static constexpr int kSubBytes = 128 * 128;
  static constexpr int kTileBytes = kSubs * kSubBytes;  // one 128 x D tile (16-bit)
  static constexpr int kStages = 2;
  static constexpr int kOffQ = 0;  // Q_A, Q_B
  static constexpr int kOffK = 2 * kTileBytes;
  static constexpr int kOffV = kOffK + kStages * kTileBytes;
  static constexpr int kOffBar = kOffV + kStages * kTileBytes;
  static constexpr int kOffRing = kOffBar + 256;
  static constexpr int kOffMask = kOffRing + 64;  // block-sparse: 2 grid rows x 64 words per ring slot
  static constexpr int kRing = 4;
  static constexpr int kSmemBytes = kOffMask + kRing * 2 * 256 + 1024;
  static_assert(kSmemBytes <= 232448, "fwd2 shared memory");
  static constexpr uint32_t kTmemS = 0;         // S_A, S_B (P aliases the first 64 columns)
  static constexpr uint32_t kTmemO = 256;       // O_A, O_B
  static constexpr uint32_t kTmemP = 0;
  static constexpr uint32_t kTmemCols = 512;
};

// item w -> (bh, pair): head groups, heaviest causal pairs first within a group
__device__ __forceinline__ void fwd2_item(const FwdParams& p, int w, int& bh, int& pair) {
  const int per_group = p.group * p.n_pairs;
  const int grp = w / per_group;
  const int r = w - grp * per_group;
  const int gsz = min(p.group, p.B * p.H - grp * p.group);
  const int slot = r / gsz;
  bh = grp * p.group + (r - slot * gsz);
  pair = (p.mask_kind == kMaskCausal && p.grid == nullptr) ? (p.n_pairs - 1 - slot) : slot;
}

// per-item schedule of the two Q tiles (named like FwdSched so the tile step reads the same)
struct Fwd2Item {
  int bh, b, h;
  int q0[2];
  int nkv[2];
  int T;
  int kv_limit;
  bool sparse;
  const uint32_t* mask[2];
  __device__ __forceinline__ bool member(int q, int t) const {
    if (sparse) return (mask[q][t >> 5] >> (t & 31)) & 1u;
    return t < nkv[q];
  }
  __device__ __forceinline__ int next(int t) const {
    if (!sparse) return t;
    while (t < T) {
      const int w = t >> 5;
      const uint32_t m = (mask[0][w] | mask[1][w]) >> (t & 31);
      if (m) return t + __ffs(m) - 1;
      t = (w + 1) << 5;
    }
    return T;
  }
  __device__ __forceinline__ bool has_after(int q, int t) const {
    if (!sparse) return t + 1 < nkv[q];
    for (int u = t + 1; u < T;) {
      const uint32_t m = mask[q][u >> 5] >> (u & 31);
      if (m) return true;
      u = ((u >> 5) + 1) << 5;
    }
    return false;
  }
};

template <int D, bool BF16, bool OUT_F32, bool DROP>
__global__ void __launch_bounds__(384, 1)
    tatn_fwd2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const FwdParams p, int* __restrict__ ctr) {
  using Cfg = Fwd2Cfg<D>;
  constexpr int kProducerWarp = 8, kMmaWarp = 9;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));
  const uint32_t sQ = smem_base + Cfg::kOffQ;
  const uint32_t sK = smem_base + Cfg::kOffK;
  const uint32_t sV = smem_base + Cfg::kOffV;
  const uint32_t bar0 = smem_base + Cfg::kOffBar;
  auto BAR = [&](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };
  const int kBarKFull = 0, kBarKEmpty = S, kBarVFull = 2 * S, kBarVEmpty = 3 * S;  // [S] each
  const int kBarQFull = 4 * S, kBarQFree = kBarQFull + 1;
  const int kBarSFull = kBarQFree + 1;   // [2]
  const int kBarPFull = kBarSFull + 2;   // [2]
  const int kBarOFinal = kBarPFull + 2;  // [2]
  const int kBarItem = kBarOFinal + 2;   // [kRing]
  const int kBarItemFree = kBarItem + Cfg::kRing;
  const int kBarPHalf = kBarItemFree + Cfg::kRing;  // [2] P columns [0, 32) (keys 0-63) written
  const int kNumBars = kBarPHalf + 2;
  static_assert(8 * (4 * S + 10 + 2 * Cfg::kRing) <= 8 * 30, "barrier region");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_gen + Cfg::kOffBar + 8 * 30);
  volatile int* ring = reinterpret_cast<volatile int*>(smem_gen + Cfg::kOffRing);
  uint32_t* mask_smem = reinterpret_cast<uint32_t*>(smem_gen + Cfg::kOffMask);
  const int warp = static_cast<int>(warp_id());
  const int lane = static_cast<int>(lane_id());
  const bool sparse = p.grid != nullptr;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNumBars; ++i) mbar_init(BAR(i), 1);
    mbar_init(BAR(kBarPFull + 0), 128);
    mbar_init(BAR(kBarPFull + 1), 128);
    mbar_init(BAR(kBarPHalf + 0), 128);
    mbar_init(BAR(kBarPHalf + 1), 128);
    for (int k = 0; k < Cfg::kRing; ++k) mbar_init(BAR(kBarItemFree + k), 9);  // MMA warp + 8 softmax warps
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    tmem_alloc(smem_u32(tmem_slot), Cfg::kTmemCols);
    tmem_relinquish();
  }
  griddep_wait();  // the previous kernel's outputs are visible from here on
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto item = [&](int w, int n) {
    Fwd2Item it;
    int pair;
    fwd2_item(p, w, it.bh, pair);
    it.b = it.bh / p.H;
    it.h = it.bh - it.b * p.H;
    it.sparse = sparse;
    int kv_limit = p.Nk;
    if (p.mask_kind == kMaskKeyPadding && p.valid_len != nullptr)
      kv_limit = min(kv_limit, max(p.valid_len[it.b] - p.k_off, 0));
    it.kv_limit = kv_limit;
    const int ntiles_kv = (kv_limit + kBN - 1) / kBN;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      it.q0[q] = (pair * 2 + q) * kBM;
      it.mask[q] = mask_smem + ((n % Cfg::kRing) * 2 + q) * 64;
      int nt = 0;
      if (it.q0[q] < p.Nq) {
        nt = ntiles_kv;
        if (p.mask_kind == kMaskCausal) {
          const int last = it.q0[q] + kBM - 1 - p.k_off;
          nt = min(nt, last >= 0 ? last / kBN + 1 : 0);
        }
      }
      it.nkv[q] = nt;
    }
    it.T = sparse ? p.tc : max(it.nkv[0], it.nkv[1]);
    return it;
  };
  auto take_item = [&](int n) -> int {  // whole warps
    mbar_wait(BAR(kBarItem + n % Cfg::kRing), static_cast<uint32_t>((n / Cfg::kRing) & 1));
    const int w = ring[n % Cfg::kRing];
    __syncwarp();
    if (lane == 0) mbar_arrive(BAR(kBarItemFree + n % Cfg::kRing));
    return w;
  };

  if (warp >= kProducerWarp) {
  setmaxnreg_dec<80>();  // the whole third warpgroup, before it splits by role
  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ claims, Q pairs, K/V ring
    if (elect_one_sync()) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
    }
    __syncwarp();
    auto claim = [&](int n) -> int {
      if (n >= Cfg::kRing)
        mbar_wait(BAR(kBarItemFree + n % Cfg::kRing), static_cast<uint32_t>((n / Cfg::kRing - 1) & 1));
      int w = -1;
      if (lane == 0) w = atomicAdd(ctr, 1);
      w = __shfl_sync(0xffffffffu, w, 0);
      if (w >= p.n_items) w = -1;
      if (w < 0 && TATN_PDL_EARLY) griddep_launch();  // no more items: the next kernel may take freed SM slots
      if (sparse && w >= 0) {  // the pair's two grid rows -> bitmasks of ring slot n % kRing
        int bh0, pair0;
        fwd2_item(p, w, bh0, pair0);
        for (int q = 0; q < 2; ++q) {
          const int qt = pair0 * 2 + q;
          const uint8_t* row = qt < p.tr ? p.grid + static_cast<size_t>(qt) * p.tc : nullptr;
          uint32_t* dst = mask_smem + ((n % Cfg::kRing) * 2 + q) * 64;
          warp_nonzero_bits(row, p.tc, 1, static_cast<uint32_t>(lane), [&](int wd, uint32_t bits) { dst[wd] = bits; });
        }
        __syncwarp();
      }
      if (lane == 0) {
        ring[n % Cfg::kRing] = w;
        mbar_arrive(BAR(kBarItem + n % Cfg::kRing));
      }
      __syncwarp();
      return w;
    };
    auto load_q = [&](const Fwd2Item& it) {
      if (elect_one_sync()) {
        mbar_expect_tx(BAR(kBarQFull), 2 * Cfg::kTileBytes);
        for (int q = 0; q < 2; ++q)
          for (int s = 0; s < Cfg::kSubs; ++s)
            tma_load_4d(sQ + q * Cfg::kTileBytes + s * Cfg::kSubBytes, &tmQ, BAR(kBarQFull), s * 64, it.q0[q], it.h,
                        it.b);
      }
      __syncwarp();
    };
    int g = 0;  // K/V tiles loaded (ring position)
    int w = claim(0);
    if (w >= 0) load_q(item(w, 0));
    for (int n = 0; w >= 0; ++n) {
      const Fwd2Item it = item(w, n);
      for (int t = it.next(0); t < it.T; t = it.next(t + 1), ++g) {
        const int stage = g % S;
        const uint32_t ph = static_cast<uint32_t>((g / S) & 1);
        mbar_wait(BAR(kBarKEmpty + stage), ph ^ 1);
        if (elect_one_sync()) {
          mbar_expect_tx(BAR(kBarKFull + stage), Cfg::kTileBytes);
          for (int s = 0; s < Cfg::kSubs; ++s)
            tma_load_4d(sK + stage * Cfg::kTileBytes + s * Cfg::kSubBytes, &tmK, BAR(kBarKFull + stage), s * 64,
                        t * kBN, it.h, it.b);
        }
        __syncwarp();
        mbar_wait(BAR(kBarVEmpty + stage), ph ^ 1);
        if (elect_one_sync()) {
          mbar_expect_tx(BAR(kBarVFull + stage), Cfg::kTileBytes);
          for (int s = 0; s < Cfg::kSubs; ++s)
            tma_load_4d(sV + stage * Cfg::kTileBytes + s * Cfg::kSubBytes, &tmV, BAR(kBarVFull + stage), s * 64,
                        t * kBN, it.h, it.b);
        }
        __syncwarp();
      }
      w = claim(n + 1);
      if (w >= 0) {
        mbar_wait(BAR(kBarQFree), static_cast<uint32_t>(n & 1));  // every QK of item n has read Q
        load_q(item(w, n + 1));
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer: ping-pong across items
    constexpr uint32_t ab = BF16 ? 1u : 0u;
    constexpr uint32_t idesc_qk = make_idesc_f16(ab, 128, kBN, 0, 0);
    constexpr uint32_t idesc_pv = make_idesc_f16(ab, 128, D, 0, 1);
    const uint64_t qdesc0 = make_sdesc_sw128(sQ, 16, 1024);
    const uint64_t kdesc0 = make_sdesc_sw128(sK, 16, 1024);
    const uint64_t vdesc0 = make_sdesc_sw128(sV, Cfg::kSubBytes, 1024);
    int g = 0;  // global K/V tile index (ring position)
    uint32_t pph[2] = {0, 0};
    for (int n = 0;; ++n) {
      const int w = take_item(n);
      if (w < 0) break;
      const Fwd2Item sc = item(w, n);
      auto issue_qk = [&](int q, int t, int stage) {
        if (elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * Cfg::kSubBytes + (kk & 3) * 32;
            mma_ss(tmem_base + Cfg::kTmemS + q * 128, qdesc0 + ((q * Cfg::kTileBytes + off) >> 4),
                   kdesc0 + ((stage * Cfg::kTileBytes + off) >> 4), idesc_qk, kk > 0 ? 1u : 0u);
          }
          mma_commit(BAR(kBarSFull + q));
          if (p.visited != nullptr) {
            const long long bit = static_cast<long long>(sc.q0[q] / kBM) * p.tc + t;
            atomicOr(p.visited + (bit >> 5), 1u << (bit & 31));
          }
        }
        __syncwarp();
      };
      int t = sc.next(0);
      // every item consumes a QFull phase (also items without tiles): wait in order, so no wait is
      // ever two phases ahead of the barrier
      mbar_wait(BAR(kBarQFull), static_cast<uint32_t>(n & 1));
      if (t < sc.T) {
        mbar_wait(BAR(kBarKFull + g % S), static_cast<uint32_t>((g / S) & 1));
        tc_fence_after();
        for (int q = 0; q < 2; ++q)
          if (sc.member(q, t)) issue_qk(q, t, g % S);
        if (elect_one_sync()) mma_commit(BAR(kBarKEmpty + g % S));
        __syncwarp();
      }
      uint32_t acc[2] = {0, 0};
      while (t < sc.T) {
        const int tn = sc.next(t + 1);
        const int stage = g % S, sn = (g + 1) % S;
        const uint32_t ph = static_cast<uint32_t>((g / S) & 1), phn = static_cast<uint32_t>(((g + 1) / S) & 1);
        bool k_ready = false;
        bool qk_done[2] = {false, false};
        mbar_wait(BAR(kBarVFull + stage), ph);
        tc_fence_after();
        for (int q = 0; q < 2; ++q) {
          if (!sc.member(q, t)) continue;
          // P·V in two halves: keys 0-63 as soon as the softmax has written their P (PHalf), under
          // its exponentials of keys 64-127
          mbar_wait(BAR(kBarPHalf + q), pph[q]);
          tc_fence_after();
          if (elect_one_sync()) {
#pragma unroll
            for (int kk = 0; kk < kBN / 32; ++kk)
              mma_ts(tmem_base + Cfg::kTmemO + q * D, tmem_base + Cfg::kTmemP + q * 128 + kk * 8,
                     vdesc0 + ((stage * Cfg::kTileBytes + kk * 2048) >> 4), idesc_pv, (acc[q] | (kk > 0 ? 1u : 0u)));
          }
          __syncwarp();
          mbar_wait(BAR(kBarPFull + q), pph[q]);
          pph[q] ^= 1;
          tc_fence_after();
          if (elect_one_sync()) {
#pragma unroll
            for (int kk = kBN / 32; kk < kBN / 16; ++kk)
              mma_ts(tmem_base + Cfg::kTmemO + q * D, tmem_base + Cfg::kTmemP + q * 128 + kk * 8,
                     vdesc0 + ((stage * Cfg::kTileBytes + kk * 2048) >> 4), idesc_pv, 1u);
            if (!sc.has_after(q, t)) mma_commit(BAR(kBarOFinal + q));  // tile q's O is final
          }
          __syncwarp();
          acc[q] = 1;
          if (tn < sc.T && sc.member(q, tn)) {
            if (!k_ready) {
              mbar_wait(BAR(kBarKFull + sn), phn);
              tc_fence_after();
              k_ready = true;
            }
            issue_qk(q, tn, sn);
            qk_done[q] = true;
          }
        }
        if (elect_one_sync()) mma_commit(BAR(kBarVEmpty + stage));
        __syncwarp();
        if (tn < sc.T) {
          for (int q = 0; q < 2; ++q) {
            if (qk_done[q] || !sc.member(q, tn)) continue;
            if (!k_ready) {
              mbar_wait(BAR(kBarKFull + sn), phn);
              tc_fence_after();
              k_ready = true;
            }
            issue_qk(q, tn, sn);
          }
          if (elect_one_sync()) mma_commit(BAR(kBarKEmpty + sn));
          __syncwarp();
        }
        t = tn;
        ++g;
      }
      // every QK of item n issued: Q may be reloaded once they complete
      if (elect_one_sync()) mma_commit(BAR(kBarQFree));
      __syncwarp();
    }
  }
  } else {
    setmaxnreg_inc<208>();
    // ------------------------------------------------------------ softmax + epilogue warpgroups
    const int q = warp >> 2;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t tS = tmem_base + lane_off + Cfg::kTmemS + q * 128;
    const uint32_t tO = tmem_base + lane_off + Cfg::kTmemO + q * D;
    const uint32_t tP = tmem_base + lane_off + Cfg::kTmemP + q * 128;
    const float sl2 = p.scale_log2;
    const bool causal = p.mask_kind == kMaskCausal;
    const uint64_t sl2x2 = f2_pack(sl2, sl2);
    const bool custom_on = p.custom != nullptr;
    uint32_t sph = 0, ofph = 0;
    for (int n = 0;; ++n) {
      const int w = take_item(n);
      if (w < 0) break;
      const Fwd2Item sc = item(w, n);
      const int b = sc.b;
      const int my_q0 = sc.q0[q];
      auto is_member = [&](int t) -> bool { return sc.member(q, t); };
      const int grow = my_q0 + row;
      const int my_q0c = my_q0 - p.k_off, growc = grow - p.k_off;
      uint64_t drow = 0;
      if constexpr (DROP) drow = drop_row_hash(p.drop_seed + static_cast<uint64_t>(sc.bh), grow);
      auto load_cw = [&](int t, uint32_t (&cw)[4]) {
        if (p.custom != nullptr && grow < p.Nq) {
          const uint4 wv = *reinterpret_cast<const uint4*>(p.custom + static_cast<size_t>(b) * p.custom_bstride +
                                                           static_cast<size_t>(grow) * p.custom_words + p.k_off / 32 +
                                                           4 * t);
          cw[0] = wv.x;
          cw[1] = wv.y;
          cw[2] = wv.z;
          cw[3] = wv.w;
        } else {
          cw[0] = cw[1] = cw[2] = cw[3] = (p.custom != nullptr) ? 0u : ~0u;
        }
      };
      float m_run = -INFINITY;
      float l_run = 0.f;
      int n_done = 0;
      for (int t = sc.next(0); t < sc.T; t = sc.next(t + 1)) {
        if (!is_member(t)) continue;
        mbar_wait(BAR(kBarSFull + q), sph);
        sph ^= 1;
        tc_fence_after();
        const int k0 = t * kBN;
        const bool need_mask = (k0 + kBN > sc.kv_limit) || (causal && k0 + kBN - 1 > my_q0c) || custom_on;
        uint32_t cw[4];
        load_cw(t, cw);
        // masked scores -> -inf (diagonal / boundary tiles only)
        auto apply_mask = [&](uint32_t (&r)[32], int c) {
          if (need_mask) {
  #pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int kj = k0 + c * 32 + i;
              if ((kj >= sc.kv_limit) || (causal && kj > growc) || ((cw[c] >> i) & 1u) == 0u)
                r[i] = __float_as_uint(-INFINITY);
            }
          }
        };
        auto rescale_o = [&](float alpha, bool mine) {
          if (__any_sync(0xffffffffu, mine)) {
  #pragma unroll
            for (int c = 0; c < D / 32; ++c) {
              uint32_t o[32];
              tmem_ld32(tO + c * 32, o);
  #pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tmem_st32(tO + c * 32, o);
            }
          }
        };
        float row_sum = 0.f;
        // one pass: all of S(t) in registers (128 of the warpgroup's 208), then the row max, the
        // lazy rescale and the exponentials from registers; P (16-bit) overwrites S columns
        // [16c, 16c + 16) in TMEM, all of which are already in registers. One TMEM read of the
        // 64 KB tile instead of two (row max pass + exponential pass).
        uint32_t sv[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32_async(tS + c * 32, sv[c]);
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_wait32(sv[c]);
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          apply_mask(sv[c], c);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            mx0 = fmax3(mx0, __uint_as_float(sv[c][i]), __uint_as_float(sv[c][i + 1]));
            mx1 = fmax3(mx1, __uint_as_float(sv[c][i + 2]), __uint_as_float(sv[c][i + 3]));
          }
        }
        const float m_tile = fmaxf(mx0, mx1) * sl2;
        float alpha = 1.f;
        if (m_tile - m_run > kRescaleThreshold) {  // false for NaN (both -inf)
          alpha = ex2_approx(m_run - m_tile);      // 0 when m_run == -inf
          m_run = m_tile;
        }
        l_run *= alpha;
        rescale_o(alpha, (n_done > 0) && (alpha != 1.f));
        const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
        const uint64_t negm = f2_pack(-m_use, -m_use);
        uint64_t rsum0 = f2_pack(0.f, 0.f), rsum1 = rsum0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
          auto exp_chunk = [&](auto emu_on) {
            constexpr bool kEmu = decltype(emu_on)::value;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const int i = c * 16 + k;
              const uint64_t x =
                  f2_fma(f2_pack(__uint_as_float(sv[c][2 * k]), __uint_as_float(sv[c][2 * k + 1])), sl2x2, negm);
              uint64_t pv;
              if (kEmu && (i & 7) < kEmuPairsD<D>) {
                pv = exp2_poly_f2(x);
              } else {
                float x0, x1;
                f2_unpack(x, x0, x1);
                pv = f2_pack(ex2_approx(x0), ex2_approx(x1));
              }
              float p0, p1;
              f2_unpack(pv, p0, p1);
              if constexpr (DROP) {  // the MMA takes P * Z / (1 - p); l keeps the undropped P
                const int j0 = p.k_off + k0 + c * 32 + 2 * k;  // global key index
                p0 = drop_keep(drow, j0, p.drop_thresh) ? p0 * p.drop_scale : 0.f;
                p1 = drop_keep(drow, j0 + 1, p.drop_thresh) ? p1 * p.drop_scale : 0.f;
              }
              pk[k] = pack2<BF16>(p0, p1);
              if (k & 1) rsum1 = f2_add(rsum1, pv);
              else rsum0 = f2_add(rsum0, pv);
            }
          };
          if (kEmuPairsD<D> > 0 && !need_mask && !DROP) exp_chunk(std::true_type{});
          else exp_chunk(std::false_type{});
          tmem_st16(tP + c * 16, pk);
          if (c == 1) {  // P of keys 0-63 in TMEM: the first half of P·V may start
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(BAR(kBarPHalf + q));
          }
        }
        float rs0, rs1, rs2, rs3;
        f2_unpack(rsum0, rs0, rs1);
        f2_unpack(rsum1, rs2, rs3);
        row_sum = (rs0 + rs1) + (rs2 + rs3);
        l_run += row_sum;
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(BAR(kBarPFull + q));
        ++n_done;
      }
      // ---------------- epilogue: O / l from TMEM straight to global memory, LSE
      if (my_q0 < p.Nq) {
        const float inv_l = (l_run > 0.f) ? 1.f / l_run : 0.f;
        if (n_done > 0) {
          mbar_wait(BAR(kBarOFinal + q), ofph);
          ofph ^= 1;
          tc_fence_after();
        }
        const size_t obase = static_cast<size_t>(sc.b) * p.o_sb + static_cast<size_t>(sc.h) * p.o_sh +
                             static_cast<size_t>(grow) * p.o_sn;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          if (n_done > 0) {
            tmem_ld32(tO + c * 32, o);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = 0u;
          }
          if (grow < p.Nq) {
            if constexpr (OUT_F32) {
              float4* dst = reinterpret_cast<float4*>(p.o_f32 + obase + c * 32);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                dst[i] = make_float4(__uint_as_float(o[4 * i]) * inv_l, __uint_as_float(o[4 * i + 1]) * inv_l,
                                     __uint_as_float(o[4 * i + 2]) * inv_l, __uint_as_float(o[4 * i + 3]) * inv_l);
            } else {
              uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(p.o16) + obase + c * 32);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                dst[j] = make_uint4(
                    pack2<BF16>(__uint_as_float(o[8 * j]) * inv_l, __uint_as_float(o[8 * j + 1]) * inv_l),
                    pack2<BF16>(__uint_as_float(o[8 * j + 2]) * inv_l, __uint_as_float(o[8 * j + 3]) * inv_l),
                    pack2<BF16>(__uint_as_float(o[8 * j + 4]) * inv_l, __uint_as_float(o[8 * j + 5]) * inv_l),
                    pack2<BF16>(__uint_as_float(o[8 * j + 6]) * inv_l, __uint_as_float(o[8 * j + 7]) * inv_l));
            }
          }
        }
        if (grow < p.Nq) {
          const float lse = (l_run > 0.f) ? (m_run + __log2f(l_run)) * 0.69314718055994530942f : -INFINITY;
          p.lse[static_cast<size_t>(sc.bh) * p.Nq + grow] = lse;
        }
        tc_fence_before();  // O read before the next item's first PV into it (ordered by PFull)
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    // self-resetting counter: the last CTA to finish zeroes it for the next launch
    __threadfence();
    if (atomicAdd(ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
  if (warp == kMmaWarp) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

}  // namespace tatn_dev
