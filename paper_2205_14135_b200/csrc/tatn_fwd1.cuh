// tatn_fwd1.cuh — persistent FlashAttention forward for d = 64 (kernel K1, one Q tile per item).
//
// Algorithm 2 of the paper (reference flash.hpp:43-67) as a persistent
// kernel: two CTAs per SM each loop
// over work items (one 128-row Q tile of one head) claimed from a device counter, so the fixed
// per-tile costs — launch, barrier / TMEM setup, the Q and first K/V load latency, the O
// epilogue — overlap the previous item's softmax instead of idling the SM:
//   * the producer prefetches the next item's Q into the other of two Q buffers and keeps the
//     K/V ring streaming across item boundaries;
//   * the MMA warp runs one global tile stream: QK of the next tile (possibly the next item's
//     first) is issued as soon as the softmax has pulled S into registers;
//   * the softmax warpgroup writes item n's O (staged in item n's Q buffer, TMA store) and goes
//     straight on to item n+1's first tile, whose S is already computed.
// Items are claimed from a self-resetting device counter (the last CTA to finish zeroes it for the
// next launch). Block-sparse launches: the producer reads the claimed item's grid row into a
// shared-memory bitmask slot (one per ring slot) before publishing the item.
#pragma once

#include "tatn_fwd.cuh"

namespace tatn_dev {

struct Fwd1Cfg {
  static constexpr int D = 64;
  static constexpr int kTileBytes = 128 * 128;  // 128 rows x 64 x 2 B (one 128B-swizzle column block)
  static constexpr int kStages = 2;
  static constexpr int kOffQ = 0;               // two Q buffers (item parity); O staging reuses them
  static constexpr int kOffK = 2 * kTileBytes;
  static constexpr int kOffV = kOffK + kStages * kTileBytes;
  static constexpr int kOffBar = kOffV + kStages * kTileBytes;
  static constexpr int kOffRing = kOffBar + 256;
  static constexpr int kOffMask = kOffRing + 64;  // block-sparse grid row bitmasks, 64 words per ring slot
  static constexpr int kSmemBytes = kOffMask + 4 * 256 + 1024;
  static constexpr uint32_t kTmemS = 0, kTmemO = 128, kTmemP = 192, kTmemCols = 256;
  static constexpr int kRing = 4;
};

// item w -> (bh, q tile): head groups (K/V of the group's heads stay L2-resident), heaviest causal
// tiles first within a group (longest-processing-time order)
__device__ __forceinline__ void fwd1_item(const FwdParams& p, int w, int& bh, int& qt) {
  const int per_group = p.group * p.n_pairs;
  const int grp = w / per_group;
  const int r = w - grp * per_group;
  const int gsz = min(p.group, p.B * p.H - grp * p.group);
  const int slot = r / gsz;
  bh = grp * p.group + (r - slot * gsz);
  qt = (p.mask_kind == kMaskCausal && p.grid == nullptr) ? (p.n_pairs - 1 - slot) : slot;
}

constexpr int kFwd1Threads = 192;

template <bool BF16, bool OUT_F32, bool DROP>
__global__ void __launch_bounds__(kFwd1Threads, 2)
    tatn_fwd1_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                     const FwdParams p, int* __restrict__ ctr) {
  using Cfg = Fwd1Cfg;
  constexpr int D = Cfg::D;
  constexpr int kProducerWarp = 4, kMmaWarp = 5;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));
  const uint32_t sQ = smem_base + Cfg::kOffQ;
  const uint32_t sK = smem_base + Cfg::kOffK;
  const uint32_t sV = smem_base + Cfg::kOffV;
  const uint32_t bar0 = smem_base + Cfg::kOffBar;
  auto BAR = [&](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };
  const int kBarKFull = 0, kBarKEmpty = 2, kBarVFull = 4, kBarVEmpty = 6;  // [2] each
  const int kBarQFull = 8, kBarQFree = 10;                                 // [2] each (Q buffer)
  const int kBarSFull = 12, kBarSFree = 13, kBarPFull = 14, kBarPVDone = 15, kBarOFinal = 16;
  const int kBarItem = 17, kBarItemFree = kBarItem + Cfg::kRing;  // [kRing] each
  const int kBarPHalf = kBarItemFree + Cfg::kRing;  // P of keys 0-63 written
  const int kNumBars = kBarPHalf + 1;
  static_assert(8 * (18 + 2 * Cfg::kRing) <= 8 * 28, "barrier region");
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_gen + Cfg::kOffBar + 8 * 28);
  volatile int* ring = reinterpret_cast<volatile int*>(smem_gen + Cfg::kOffRing);
  uint32_t* mask_smem = reinterpret_cast<uint32_t*>(smem_gen + Cfg::kOffMask);
  const int warp = static_cast<int>(warp_id());
  const int lane = static_cast<int>(lane_id());
  const bool sparse = p.grid != nullptr;
  TATN_EV_INIT();
  if (threadIdx.x == 0) TATN_TRACE_AT(0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNumBars; ++i) mbar_init(BAR(i), 1);
    mbar_init(BAR(kBarSFree), 128);
    mbar_init(BAR(kBarPFull), 128);
    mbar_init(BAR(kBarPHalf), 128);
    for (int b = 0; b < 2; ++b) mbar_init(BAR(kBarQFree + b), 128);  // O staged by every softmax thread
    for (int k = 0; k < Cfg::kRing; ++k) mbar_init(BAR(kBarItemFree + k), 5);  // MMA warp + 4 softmax warps
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

  // per-item schedule (identical in every role)
  struct Item {
    int bh, b, h, q0, T, kv_limit;
    const uint32_t* mask;  // block-sparse: the item's grid row bitmask (ring slot)
  };
  auto item = [&](int w, int n) {
    Item it;
    it.mask = mask_smem + (n % Cfg::kRing) * 64;
    int qt;
    fwd1_item(p, w, it.bh, qt);
    it.b = it.bh / p.H;
    it.h = it.bh - it.b * p.H;
    it.q0 = qt * kBM;
    int kv_limit = p.Nk;
    if (p.mask_kind == kMaskKeyPadding && p.valid_len != nullptr)
      kv_limit = min(kv_limit, max(p.valid_len[it.b] - p.k_off, 0));
    it.kv_limit = kv_limit;
    int nt = (kv_limit + kBN - 1) / kBN;
    if (p.mask_kind == kMaskCausal) {
      const int last = it.q0 + kBM - 1 - p.k_off;
      nt = min(nt, last >= 0 ? last / kBN + 1 : 0);
    }
    it.T = sparse ? p.tc : (it.q0 < p.Nq ? nt : 0);
    return it;
  };
  // first visited key tile >= t of an item (T when none)
  auto next_tile = [&](const Item& it, int t) -> int {
    if (!sparse) return t;
    while (t < it.T) {
      const uint32_t m = it.mask[t >> 5] >> (t & 31);
      if (m) return t + __ffs(m) - 1;
      t = ((t >> 5) + 1) << 5;
    }
    return it.T;
  };
  auto take_item = [&](int n) -> int {  // whole warps
    mbar_wait(BAR(kBarItem + n % Cfg::kRing), static_cast<uint32_t>((n / Cfg::kRing) & 1));
    const int w = ring[n % Cfg::kRing];
    __syncwarp();
    if (lane == 0) mbar_arrive(BAR(kBarItemFree + n % Cfg::kRing));
    return w;
  };

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ TMA producer + item claims
    if (elect_one_sync()) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmO);
    }
    __syncwarp();
    // The producer also issues the O stores: item m's O is staged in its Q buffer (m & 1) by the
    // softmax warpgroup, which arrives QFree and moves on; the store is issued here right before
    // that buffer is refilled with Q(m + 2) (or at the end), keeping the store issue and its
    // read latency off the softmax warpgroup.
    Item pend0, pend1;  // by Q buffer (no dynamically indexed array: it would live in local memory)
    auto store_o = [&](int m) {
      const int b = m & 1;
      mbar_wait(BAR(kBarQFree + b), static_cast<uint32_t>((m >> 1) & 1));
      if constexpr (!OUT_F32) {
        if (lane == 0) {
          const Item& pi = b ? pend1 : pend0;
          tma_store_4d(&tmO, sQ + b * Cfg::kTileBytes, 0, pi.q0, pi.h, pi.b);
          bulk_commit();
          bulk_wait_read_all();  // staging read: the buffer may be refilled
        }
        __syncwarp();
      }
    };
    int g = 0;  // K/V tiles loaded so far (ring position)
    int n = 0;
    for (;; ++n) {
      if (n >= Cfg::kRing)
        mbar_wait(BAR(kBarItemFree + n % Cfg::kRing), static_cast<uint32_t>((n / Cfg::kRing - 1) & 1));
      int w = -1;
      if (lane == 0) w = atomicAdd(ctr, 1);
      w = __shfl_sync(0xffffffffu, w, 0);
      if (w >= p.n_items) w = -1;
      if (w < 0 && TATN_PDL_EARLY) griddep_launch();  // no more items: the next kernel may take freed SM slots
      if (sparse && w >= 0) {  // the item's grid row -> bitmask slot n % kRing (read once, coalesced)
        int bh0, qt0;
        fwd1_item(p, w, bh0, qt0);
        const uint8_t* grow_ptr = qt0 < p.tr ? p.grid + static_cast<size_t>(qt0) * p.tc : nullptr;
        uint32_t* slot_mask = mask_smem + (n % Cfg::kRing) * 64;
        warp_nonzero_bits(grow_ptr, p.tc, 1, lane, [&](int wd, uint32_t bits) { slot_mask[wd] = bits; });
        __syncwarp();
      }
      if (lane == 0) {
        ring[n % Cfg::kRing] = w;
        mbar_arrive(BAR(kBarItem + n % Cfg::kRing));
      }
      __syncwarp();
      if (w < 0) break;
      const Item it = item(w, n);
      const int qb = n & 1;
      if (n >= 2) store_o(n - 2);
      if (qb) pend1 = it;
      else pend0 = it;
      if (elect_one_sync()) {
        mbar_expect_tx(BAR(kBarQFull + qb), Cfg::kTileBytes);
        tma_load_4d(sQ + qb * Cfg::kTileBytes, &tmQ, BAR(kBarQFull + qb), 0, it.q0, it.h, it.b);
      }
      __syncwarp();
      for (int t = next_tile(it, 0); t < it.T; t = next_tile(it, t + 1), ++g) {
        const int stage = g & 1;
        const uint32_t ph = static_cast<uint32_t>((g >> 1) & 1);
        mbar_wait(BAR(kBarKEmpty + stage), ph ^ 1);
        if (elect_one_sync()) {
          mbar_expect_tx(BAR(kBarKFull + stage), Cfg::kTileBytes);
          tma_load_4d(sK + stage * Cfg::kTileBytes, &tmK, BAR(kBarKFull + stage), 0, t * kBN, it.h, it.b);
        }
        __syncwarp();
        mbar_wait(BAR(kBarVEmpty + stage), ph ^ 1);
        if (elect_one_sync()) {
          mbar_expect_tx(BAR(kBarVFull + stage), Cfg::kTileBytes);
          tma_load_4d(sV + stage * Cfg::kTileBytes, &tmV, BAR(kBarVFull + stage), 0, t * kBN, it.h, it.b);
        }
        __syncwarp();
      }
    }
    for (int m = max(n - 2, 0); m < n; ++m) store_o(m);
    if (lane == 0) bulk_wait_all();
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer: one global tile stream
    constexpr uint32_t ab = BF16 ? 1u : 0u;
    constexpr uint32_t idesc_qk = make_idesc_f16(ab, 128, kBN, 0, 0);
    constexpr uint32_t idesc_pv = make_idesc_f16(ab, 128, D, 0, 1);
    const uint64_t qdesc0 = make_sdesc_sw128(sQ, 16, 1024);
    const uint64_t kdesc0 = make_sdesc_sw128(sK, 16, 1024);
    const uint64_t vdesc0 = make_sdesc_sw128(sV, Cfg::kTileBytes, 1024);
    // iterator over (item n, key tile t) in stream order, skipping items without tiles
    struct Pos {
      int n, w, t, first;
      Item it;
    };
    int n_taken = 0;  // items read from the ring
    auto next_item = [&](Pos& ps) -> bool {  // advance to the first tile of the next item with tiles
      for (;;) {
        const int w = take_item(n_taken);
        if (w < 0) return false;
        ps.n = n_taken++;
        ps.w = w;
        ps.it = item(w, ps.n);
        ps.t = next_tile(ps.it, 0);
        ps.first = 1;
        if (ps.t < ps.it.T) return true;
      }
    };
    auto advance = [&](Pos& ps) -> bool {
      const int t = next_tile(ps.it, ps.t + 1);
      if (t < ps.it.T) {
        ps.t = t;
        ps.first = 0;
        return true;
      }
      return next_item(ps);
    };
    // Every item (also one without tiles) completes one QFull phase of buffer n & 1. The MMA
    // warp waits only for the items it has tiles of, directly on item n's phase: Q(n + 2) is
    // loaded into the same buffer only after item n's epilogue (which needs this warp's PVs) and
    // Q(n) only after item n - 2's, so when the wait is issued the barrier is exactly at phase
    // n >> 1 or one before it. (Waiting the skipped items' phases later, in order, as round 1 did,
    // aliased parities once the softmax warpgroup had run the producer two or more phases ahead
    // through items without tiles — all-padded batches deadlocked.)
    auto issue_qk = [&](const Pos& ps, int g) {
      const int stage = g & 1;
      const int qb = ps.n & 1;
      if (ps.first) mbar_wait(BAR(kBarQFull + qb), static_cast<uint32_t>((ps.n >> 1) & 1));
      mbar_wait(BAR(kBarKFull + stage), static_cast<uint32_t>((g >> 1) & 1));
      tc_fence_after();
      if (elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_ss(tmem_base + Cfg::kTmemS, qdesc0 + ((qb * Cfg::kTileBytes + kk * 32) >> 4),
                 kdesc0 + ((stage * Cfg::kTileBytes + kk * 32) >> 4), idesc_qk, kk > 0 ? 1u : 0u);
        mma_commit(BAR(kBarSFull));
        mma_commit(BAR(kBarKEmpty + stage));
        if (p.visited != nullptr) {
          const long long bit = static_cast<long long>(ps.it.q0 / kBM) * p.tc + ps.t;
          atomicOr(p.visited + (bit >> 5), 1u << (bit & 31));
        }
      }
      __syncwarp();
    };
    // P·V in two halves: keys 0-63 once the softmax has written their P (PHalf), under its
    // exponentials of keys 64-127, then keys 64-127 after PFull
    auto issue_pv = [&](const Pos& ps, int g, bool last_of_item) {
      const int stage = g & 1;
      mbar_wait(BAR(kBarPHalf), static_cast<uint32_t>(g & 1));
      mbar_wait(BAR(kBarVFull + stage), static_cast<uint32_t>((g >> 1) & 1));
      tc_fence_after();
      if (elect_one_sync()) {
#pragma unroll
        for (int kk = 0; kk < kBN / 32; ++kk)
          mma_ts(tmem_base + Cfg::kTmemO, tmem_base + Cfg::kTmemP + kk * 8,
                 vdesc0 + ((stage * Cfg::kTileBytes + kk * 2048) >> 4), idesc_pv,
                 (ps.first ? 0u : 1u) | (kk > 0 ? 1u : 0u));
      }
      __syncwarp();
      mbar_wait(BAR(kBarPFull), static_cast<uint32_t>(g & 1));
      if (lane == 0) TATN_EV(g, 3);
      tc_fence_after();
      if (elect_one_sync()) {
#pragma unroll
        for (int kk = kBN / 32; kk < kBN / 16; ++kk)
          mma_ts(tmem_base + Cfg::kTmemO, tmem_base + Cfg::kTmemP + kk * 8,
                 vdesc0 + ((stage * Cfg::kTileBytes + kk * 2048) >> 4), idesc_pv, 1u);
        mma_commit(BAR(kBarPVDone));
        mma_commit(BAR(kBarVEmpty + stage));
        if (last_of_item) mma_commit(BAR(kBarOFinal));
      }
      __syncwarp();
    };
    Pos cur;
    if (next_item(cur)) {
      int g = 0;  // global tile index of `cur`
      issue_qk(cur, 0);
      for (;;) {
        Pos nx = cur;
        const bool has_next = advance(nx);
        // QK of the next tile is issued before PV(cur) (it runs under softmax(cur)) when both
        // belong to the same item. At an item boundary PV(cur) goes first: the softmax warpgroup
        // needs it for the epilogue (O) before it needs S(next), and QK(next) may still wait for the
        // next item's Q / K to land — issued first it held PV(cur), and so the epilogue, behind those
        // loads (traced: ~1.6K clk per boundary). An item two or more ahead reuses cur's Q buffer,
        // which is reloaded only after cur's epilogue, so it must follow PV(cur) anyway.
#ifndef TATN_FWD1_QK_BEFORE_LAST_PV
#define TATN_FWD1_QK_BEFORE_LAST_PV 0  // 1: round-1 order (next item's first QK before the last PV)
#endif
        const bool early = has_next && (TATN_FWD1_QK_BEFORE_LAST_PV ? nx.n <= cur.n + 1 : nx.n == cur.n);
        if (early) {
          mbar_wait(BAR(kBarSFree), static_cast<uint32_t>(g & 1));  // S(g) is in registers
          issue_qk(nx, g + 1);
          if (lane == 0) TATN_EV(g + 1, 4);
        }
        issue_pv(cur, g, !has_next || nx.n != cur.n);
        if (has_next && !early) {
          mbar_wait(BAR(kBarSFree), static_cast<uint32_t>(g & 1));
          issue_qk(nx, g + 1);
        }
        if (!has_next) break;
        cur = nx;
        ++g;
      }
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ softmax + epilogue warpgroup
    const int row = warp * 32 + lane;  // row within the tile == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    const uint32_t tS = tmem_base + lane_off + Cfg::kTmemS;
    const uint32_t tO = tmem_base + lane_off + Cfg::kTmemO;
    const uint32_t tP = tmem_base + lane_off + Cfg::kTmemP;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2_pack(sl2, sl2);
    const bool causal = p.mask_kind == kMaskCausal;
    const bool custom_on = p.custom != nullptr;
    int g = 0;   // global tile index
    int nf = 0;  // OFinal phases consumed (items with tiles)
    // the next item is taken (and decoded) under the current item's last PV, ahead of its epilogue
    int w_next = take_item(0);
    Item it_next = item(max(w_next, 0), 0);
    for (int n = 0; w_next >= 0; ++n) {
      if (threadIdx.x == 0) TATN_EV(g, 5);
      const Item it = it_next;
      const int qb = n & 1;
      const int grow = it.q0 + row;
      const int growc = grow - p.k_off;
      uint64_t drow = 0;
      if constexpr (DROP) drow = drop_row_hash(p.drop_seed + static_cast<uint64_t>(it.bh), grow);
      float m_run = -INFINITY, l_run = 0.f;
      int n_done = 0;
      for (int t = next_tile(it, 0); t < it.T; t = next_tile(it, t + 1), ++g, ++n_done) {
        mbar_wait(BAR(kBarSFull), static_cast<uint32_t>(g & 1));
        tc_fence_after();
        if (threadIdx.x == 0) TATN_EV(g, 0);
        uint32_t sv[4][32];
        tmem_ld32_async(tS, sv[0]);
        tmem_ld32_async(tS + 32, sv[1]);
        tmem_ld32_async(tS + 64, sv[2]);
        tmem_ld32_async(tS + 96, sv[3]);
        tmem_ld_wait32(sv[0]);
        tmem_ld_wait32(sv[1]);
        tmem_ld_wait32(sv[2]);
        tmem_ld_wait32(sv[3]);
        tc_fence_before();
        mbar_arrive(BAR(kBarSFree));
        if (threadIdx.x == 0) TATN_EV(g, 1);
        const int k0 = t * kBN;
        const bool need_mask = (k0 + kBN > it.kv_limit) || (causal && k0 + kBN - 1 > it.q0 - p.k_off) || custom_on;
        const int lim = min(it.kv_limit, causal ? growc + 1 : it.kv_limit) - k0;  // columns >= lim masked
        // PV(g-1) has drained P / finished O; within an item only (the previous item's last PV
        // completed before its epilogue read O)
        bool pv_ready = n_done == 0;
        auto wait_pv = [&]() {
          mbar_wait(BAR(kBarPVDone), static_cast<uint32_t>((g - 1) & 1));
          tc_fence_after();
        };
        if (custom_on) {  // Custom mask: -inf where the row's keep bit is 0
          uint32_t cw[4] = {0u, 0u, 0u, 0u};
          if (grow < p.Nq) {
            const uint4 wv = *reinterpret_cast<const uint4*>(p.custom + static_cast<size_t>(it.b) * p.custom_bstride +
                                                             static_cast<size_t>(grow) * p.custom_words + p.k_off / 32 +
                                                             4 * t);
            cw[0] = wv.x;
            cw[1] = wv.y;
            cw[2] = wv.z;
            cw[3] = wv.w;
          }
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i) sv[c][i] = ((cw[c] >> i) & 1u) ? sv[c][i] : __float_as_uint(-INFINITY);
        }
        auto step = [&](auto masked_t) {
          constexpr bool kMasked = decltype(masked_t)::value;
          if constexpr (kMasked) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int i = 0; i < 32; ++i) sv[c][i] = (c * 32 + i >= lim) ? __float_as_uint(-INFINITY) : sv[c][i];
          }
          float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int i = 0; i < 32; i += 4) {
                mx0 = fmax3(mx0, __uint_as_float(sv[c][i]), __uint_as_float(sv[c][i + 1]));
                mx1 = fmax3(mx1, __uint_as_float(sv[c][i + 2]), __uint_as_float(sv[c][i + 3]));
              }
          const float m_tile = fmaxf(mx0, mx1) * sl2;
          const bool jump = m_tile - m_run > kRescaleThreshold;  // false when both are -inf
          if (__any_sync(0xffffffffu, jump)) {                   // warp-uniform: TMEM ld/st are .sync.aligned
            float alpha = 1.f;
            if (jump) {
              alpha = ex2_approx(m_run - m_tile);  // 0 when m_run == -inf
              m_run = m_tile;
              l_run *= alpha;
            }
            if (!pv_ready) {
              wait_pv();  // O is final up to the previous tile
              pv_ready = true;
#pragma unroll 1
              for (int c = 0; c < D / 16; ++c) {
                uint32_t o[16];
                tmem_ld16(tO + c * 16, o);
#pragma unroll
                for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                tmem_st16(tO + c * 16, o);
              }
            }
          }
          const float m_use = (m_run == -INFINITY) ? 0.f : m_run;
          const uint64_t negm = f2_pack(-m_use, -m_use);
          uint64_t rsum0 = f2_pack(0.f, 0.f), rsum1 = rsum0;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t pk[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const int i = c * 16 + k;
              const uint64_t x =
                  f2_fma(f2_pack(__uint_as_float(sv[c][2 * k]), __uint_as_float(sv[c][2 * k + 1])), sl2x2, negm);
              uint64_t pv;
              if (!kMasked && !DROP && kEmuPairs > 0 && (i & 7) < kEmuPairs) {
                pv = exp2_poly_f2(x);  // finite x only: full tiles, m_run <= true max + threshold
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
            if (c == 0 && !pv_ready) wait_pv();  // PV(g-1) has read P(g-1)
            tmem_st16(tP + c * 16, pk);
            if (c == 1) {  // P of keys 0-63 in TMEM: the first half of P·V may start
              tmem_st_wait();
              tc_fence_before();
              mbar_arrive(BAR(kBarPHalf));
            }
          }
          float rs0, rs1, rs2, rs3;
          f2_unpack(rsum0, rs0, rs1);
          f2_unpack(rsum1, rs2, rs3);
          l_run += (rs0 + rs1) + (rs2 + rs3);
        };
        if (need_mask) step(std::true_type{});
        else step(std::false_type{});
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(BAR(kBarPFull));
        if (threadIdx.x == 0) TATN_EV(g, 2);
      }
      w_next = take_item(n + 1);
      if (w_next >= 0) it_next = item(w_next, n + 1);
      // ---------------- epilogue of item n: O / l -> staging in Q buffer qb -> TMA store; LSE
      mbar_wait(BAR(kBarQFull + qb), static_cast<uint32_t>((n >> 1) & 1));  // Q landed (and is not in flight)
      if (n_done > 0) {
        mbar_wait(BAR(kBarOFinal), static_cast<uint32_t>(nf & 1));  // every MMA of the item done
        ++nf;
        tc_fence_after();
        if (threadIdx.x == 0) TATN_EV(g - 1, 6);
      }
      const float inv_l = (l_run > 0.f) ? 1.f / l_run : 0.f;
      const uint32_t sO = sQ + qb * Cfg::kTileBytes;
      float* orow = nullptr;
      if constexpr (OUT_F32)
        orow = p.o_f32 + static_cast<size_t>(it.b) * p.o_sb + static_cast<size_t>(it.h) * p.o_sh +
               static_cast<size_t>(grow) * p.o_sn;
      uint32_t oall[D / 32][32];
      if (n_done > 0) {  // both loads in flight before the first wait
#pragma unroll
        for (int c = 0; c < D / 32; ++c) tmem_ld32_async(tO + c * 32, oall[c]);
#pragma unroll
        for (int c = 0; c < D / 32; ++c) tmem_ld_wait32(oall[c]);
      } else {
#pragma unroll
        for (int c = 0; c < D / 32; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) oall[c][i] = 0u;
      }
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t* o = oall[c];
        if constexpr (OUT_F32) {
          if (grow < p.Nq) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              reinterpret_cast<float4*>(orow + c * 32)[i] =
                  make_float4(__uint_as_float(o[4 * i]) * inv_l, __uint_as_float(o[4 * i + 1]) * inv_l,
                              __uint_as_float(o[4 * i + 2]) * inv_l, __uint_as_float(o[4 * i + 3]) * inv_l);
          }
        } else {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i)
            pk[i] = pack2<BF16>(__uint_as_float(o[2 * i]) * inv_l, __uint_as_float(o[2 * i + 1]) * inv_l);
          const int chunk0 = (c * 32) / 8;
          const uint32_t rbase = sO + row * 128;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            st_shared_v4(rbase + (((chunk0 + j) ^ (row & 7)) << 4), pk[4 * j], pk[4 * j + 1], pk[4 * j + 2],
                         pk[4 * j + 3]);
        }
      }
      if (grow < p.Nq) {
        const float lse = (l_run > 0.f) ? (m_run + __log2f(l_run)) * 0.69314718055994530942f : -INFINITY;
        p.lse[static_cast<size_t>(it.bh) * p.Nq + grow] = lse;
      }
      tc_fence_before();  // O read out of TMEM before the next item's first PV (ordered by PFull)
      if constexpr (!OUT_F32) fence_proxy_async_smem();
      if (threadIdx.x == 0 && n_done > 0) TATN_EV(g - 1, 7);
      mbar_arrive(BAR(kBarQFree + qb));  // O staged: the producer issues the store
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    TATN_TRACE_AT(7);
#ifdef TATN_TRACE
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    if (g_tatn_trace) g_tatn_trace[static_cast<size_t>(blockIdx.x) * 16 + 5] = smid;
#endif
    // self-resetting counter: the last CTA to finish (every claim done) zeroes it for the next launch
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
