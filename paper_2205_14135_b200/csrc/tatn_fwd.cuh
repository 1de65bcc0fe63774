// tatn_fwd.cuh — FlashAttention forward for sm_100a (kernel K1).
//
// Replaces the body of tatn::flash_forward / tatn::blocksparse_forward
// (reference proj/core/include/tatn/flash.hpp:43-67), i.e. Algorithm 2 of the
// paper without dropout. The reference's loop order is
// K/V-block outer, Q-block inner with O/l/m read-modify-written to HBM each
// outer pass; outputs are schedule-invariant (flash.hpp:37-40),
// so here each CTA owns two 128-row Q tiles and streams K/V tiles through
// shared memory: O, l, m never leave the SM until the final write.
//
// CTA layout (384 threads; setmaxnreg gives the softmax warpgroups 208 registers):
//   warps 0-3  softmax/correction/epilogue for Q tile A (one TMEM lane per thread)
//   warps 4-7  same for Q tile B
//   warp  8    TMA producer (Q once, K/V ring)
//   warp  9    TMEM allocator + single-thread tcgen05.mma issuer
//   warps 10-11 idle (complete the third warpgroup for setmaxnreg)
// TMEM (512 cols): S_A [0,128) S_B [128,256) O_A [256,256+D) O_B [256+D, 256+2D);
// P (bf16/fp16) overwrites the first 64 columns of S_q once S_q is in registers.
// Per K/V tile t the MMA issues S_q = Q_q K_t^T for both tiles, then
// O_q += P_q V_t after softmax_q signals P ready; tcgen05 ops from one thread
// execute in order, so the next S_q write cannot overtake the P_q read.
#pragma once

#include <type_traits>

#include "sm100_ptx.cuh"
#include "tatn_params.h"

namespace tatn_dev {

constexpr int kBM = 128;  // query rows per Q tile
constexpr int kBN = 128;  // keys per K/V tile
// NQ = 2: 384 threads (softmax A, softmax B, {TMA, MMA, 2 idle}), 1 CTA/SM.
// NQ = 1: 192 threads (softmax, TMA, MMA), 2 CTAs/SM (d = 64).
template <int NQ>
constexpr int fwd_threads() { return NQ == 2 ? 384 : 192; }
constexpr float kRescaleThreshold = 8.0f;  // lazy O rescale (log2 units)
// 16-bit exponentials (ex2.approx.{bf16x2,f16x2}, one MUFU op per pair) instead of fp32
// ex2: measured slower on B200 (r01 sweep) and less accurate, so off by default.
#ifndef TATN_EX2_16
#define TATN_EX2_16 0
#endif
// exp2 pairs per group of 8 computed by the polynomial on the FMA pipe instead of MUFU
// (MUFU.EX2 retires 16/clk/SM). Swept on B200 (r01): 1 of 8 is best (+3-5%); 2 or 3 of 8
// lose to the extra FMA-pipe issue. Full tiles only (masked tiles hold -inf).
#ifndef TATN_EMU_PAIRS
#define TATN_EMU_PAIRS 1
#endif
constexpr int kEmuPairs = TATN_EMU_PAIRS;
// d = 128 keeps every exp2 on MUFU: there the MMA and MUFU are balanced and the FMA-pipe
// polynomial measured slower (N = 8K causal fwd 889 -> 912 TFLOP/s without it)
#ifndef TATN_EMU_PAIRS_D128
#define TATN_EMU_PAIRS_D128 0
#endif
template <int D>
constexpr int kEmuPairsD = D == 128 ? TATN_EMU_PAIRS_D128 : TATN_EMU_PAIRS;

template <int D, int NQ = 2>
struct FwdCfg {
  static constexpr int kSubs = D / 64;                   // 128B-swizzle column blocks
  static constexpr int kSubBytes = 128 * 128;            // 128 rows x 128 bytes
  static constexpr int kTileBytes = kSubs * kSubBytes;   // one 128 x D tile (16-bit)
  static constexpr int kStages = (NQ == 2 && D == 64) ? 4 : 2;
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = NQ * kTileBytes;
  static constexpr int kOffV = kOffK + kStages * kTileBytes;
  static constexpr int kOffBar = kOffV + kStages * kTileBytes;
  static constexpr int kOffMask = kOffBar + 256;           // block-sparse row bitmasks, 2 x 64 words
  static constexpr int kSmemBytes = kOffMask + 512 + 1024;  // + alignment slack
  static constexpr uint32_t kTmemS = 0;
  static constexpr uint32_t kTmemO = NQ * 128;
  static constexpr uint32_t kTmemCols = NQ == 2 ? 512 : 256;  // power of two
  // P (16-bit, 64 columns per Q tile) gets its own columns when TMEM has room
  // (d = 64 layouts); otherwise it overwrites the first 64 columns of S.
  static constexpr bool kSeparateP = (NQ * (128 + D + 64)) <= static_cast<int>(kTmemCols);
  static constexpr uint32_t kTmemP = kSeparateP ? NQ * (128 + D) : kTmemS;
};

constexpr int kMaxSparseTiles = 2048;  // tc limit of the block-sparse path (N <= 256K)

struct FwdSched {
  int q0[2];    // first global query row of each tile
  int nkv[2];   // dense mode: number of leading K/V tiles the tile visits
  int T;        // union length (tiles 0..T-1 are candidates)
  int kv_limit; // keys >= kv_limit are masked (Nk, or min(Nk, valid_len[b]))
  const uint8_t* row[2];      // block-sparse grid rows in global memory (read once)
  const uint32_t* mask[2];    // the same rows as shared-memory bitmasks
  bool sparse;

  __device__ __forceinline__ bool member(int q, int t) const {
    if (sparse) return (mask[q][t >> 5] >> (t & 31)) & 1u;
    return t < nkv[q];
  }
  // does Q tile q visit any tile after t?
  __device__ __forceinline__ bool has_after(int q, int t) const {
    if (!sparse) return t + 1 < nkv[q];
    for (int u = t + 1; u < T;) {
      const uint32_t m = mask[q][u >> 5] >> (u & 31);
      if (m) return true;
      u = ((u >> 5) + 1) << 5;
    }
    return false;
  }
  // first tile >= t visited by either Q tile (T when none)
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
};

template <int NQ>
__device__ __forceinline__ FwdSched make_fwd_sched(const FwdParams& p, int b, int pair) {
  FwdSched s;
  s.sparse = p.grid != nullptr;
  int kv_limit = p.Nk;
  // key j of this call is global key k_off + j (sequence-parallel shards); valid_len is global
  if (p.mask_kind == kMaskKeyPadding && p.valid_len != nullptr) kv_limit = min(kv_limit, max(p.valid_len[b] - p.k_off, 0));
  s.kv_limit = kv_limit;
  const int ntiles_kv = (kv_limit + kBN - 1) / kBN;
  s.T = 0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int qt = pair * NQ + q;
    s.q0[q] = qt * kBM;
    s.row[q] = nullptr;
    int n = 0;
    if (q < NQ && s.q0[q] < p.Nq) {
      if (s.sparse) {
        s.row[q] = (qt < p.tr) ? p.grid + static_cast<size_t>(qt) * p.tc : nullptr;
      } else {
        n = ntiles_kv;
        if (p.mask_kind == kMaskCausal) {  // last visible global key of the tile: q0 + 127
          const int last = s.q0[q] + kBM - 1 - p.k_off;
          n = min(n, last >= 0 ? last / kBN + 1 : 0);
        }
      }
    }
    s.nkv[q] = n;
  }
  s.T = s.sparse ? p.tc : max(s.nkv[0], s.nkv[1]);
  return s;
}


template <int D, bool BF16, bool OUT_F32, int NQ, bool DROP>
__global__ void __launch_bounds__(fwd_threads<NQ>(), NQ == 2 ? 1 : 2)
    tatn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                    const FwdParams p) {
  using Cfg = FwdCfg<D, NQ>;
  constexpr int kProducerWarp = 4 * NQ, kMmaWarp = 4 * NQ + 1;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));

  const uint32_t sQ = smem_base + Cfg::kOffQ;
  const uint32_t sK = smem_base + Cfg::kOffK;
  const uint32_t sV = smem_base + Cfg::kOffV;
  const uint32_t bar0 = smem_base + Cfg::kOffBar;
  // barrier slots (8 bytes each)
  auto BAR = [&](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };
  const int kBarQ = 0;
  const int kBarKFull = 1;                       // + stage
  const int kBarKEmpty = kBarKFull + Cfg::kStages;
  const int kBarVFull = kBarKEmpty + Cfg::kStages;
  const int kBarVEmpty = kBarVFull + Cfg::kStages;
  const int kBarSFull = kBarVEmpty + Cfg::kStages;  // + q
  const int kBarPFull = kBarSFull + 2;
  const int kBarOFinal = kBarPFull + 2;
  // NQ = 1 only: S consumed into registers (QK(t+1) may overwrite it) / PV(t) complete (P free)
  const int kBarSFree = kBarOFinal + 2;
  const int kBarPVDone = kBarSFree + 1;
  const int kNumBars = kBarPVDone + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_gen + Cfg::kOffBar + 8 * 30);

  const int warp = static_cast<int>(warp_id());
  const int lane = static_cast<int>(lane_id());
  // 1-D grid in head groups: the CTAs of `group` heads are dispatched together
  // (their K/V stay L2-resident), heaviest causal tiles first within the group
  // (longest-processing-time order, so the tail is made of light tiles).
  int bh, slot;
  {
    const int per_group = p.group * p.n_pairs;
    const int grp = static_cast<int>(blockIdx.x) / per_group;
    const int r = static_cast<int>(blockIdx.x) - grp * per_group;
    const int gsz = min(p.group, p.B * p.H - grp * p.group);
    slot = r / gsz;
    bh = grp * p.group + (r - slot * gsz);
  }
  const int b = bh / p.H;
  const int h = bh - b * p.H;
  const int pair = (p.mask_kind == kMaskCausal && p.grid == nullptr) ? (p.n_pairs - 1 - slot) : slot;
  uint32_t* mask_smem = reinterpret_cast<uint32_t*>(smem_gen + Cfg::kOffMask);
  if (threadIdx.x == 0) TATN_TRACE_AT(0);
  TATN_EV_INIT();

  if (threadIdx.x == 0) {
    mbar_init(BAR(kBarQ), 1);
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(BAR(kBarKFull + s), 1);
      mbar_init(BAR(kBarKEmpty + s), 1);
      mbar_init(BAR(kBarVFull + s), 1);
      mbar_init(BAR(kBarVEmpty + s), 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(BAR(kBarSFull + q), 1);
      mbar_init(BAR(kBarPFull + q), 128);
      mbar_init(BAR(kBarOFinal + q), 1);
    }
    mbar_init(BAR(kBarSFree), 128);
    mbar_init(BAR(kBarPVDone), 1);
    (void)kNumBars;
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    tmem_alloc(smem_u32(tmem_slot), Cfg::kTmemCols);
    tmem_relinquish();
  }
  FwdSched sc = make_fwd_sched<NQ>(p, b, pair);
  sc.mask[0] = mask_smem;
  sc.mask[1] = mask_smem + kMaxSparseTiles / 32;
  if (sc.sparse && warp == kProducerWarp) {
    // block-sparse: read the two grid rows once (coalesced) into shared-memory bitmasks
    for (int q = 0; q < 2; ++q)
      for (int base = 0; base < p.tc; base += 32) {
        const int t = base + lane;
        const bool v = sc.row[q] != nullptr && t < p.tc && sc.row[q][t] != 0;
        const uint32_t bits = __ballot_sync(0xffffffffu, v);
        if (lane == 0) mask_smem[q * (kMaxSparseTiles / 32) + (base >> 5)] = bits;
      }
  }
  griddep_wait();  // the previous kernel's outputs are visible from here on
  griddep_launch();  // one item per CTA: dependents may fill slots of finished CTAs
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  int n_steps_dbg = 0;
  (void)n_steps_dbg;
  if (warp >= kProducerWarp) {
  if constexpr (NQ == 2) setmaxnreg_dec<80>();  // the whole third warpgroup, before it splits by role
  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ TMA producer
    // whole warp runs the loop (waits), one elected lane issues
    if (elect_one_sync()) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmO);
      mbar_expect_tx(BAR(kBarQ), NQ * Cfg::kTileBytes);
      for (int q = 0; q < NQ; ++q)
        for (int s = 0; s < Cfg::kSubs; ++s)
          tma_load_4d(sQ + q * Cfg::kTileBytes + s * Cfg::kSubBytes, &tmQ, BAR(kBarQ), s * 64, sc.q0[q], h, b);
    }
    __syncwarp();
    int stage = 0;
    uint32_t ph = 0;
    for (int t = sc.next(0); t < sc.T; t = sc.next(t + 1)) {
      mbar_wait(BAR(kBarKEmpty + stage), ph ^ 1);
      if (elect_one_sync()) {
        mbar_expect_tx(BAR(kBarKFull + stage), Cfg::kTileBytes);
        for (int s = 0; s < Cfg::kSubs; ++s)
          tma_load_4d(sK + stage * Cfg::kTileBytes + s * Cfg::kSubBytes, &tmK, BAR(kBarKFull + stage), s * 64,
                      t * kBN, h, b);
      }
      __syncwarp();
      mbar_wait(BAR(kBarVEmpty + stage), ph ^ 1);
      if (elect_one_sync()) {
        mbar_expect_tx(BAR(kBarVFull + stage), Cfg::kTileBytes);
        for (int s = 0; s < Cfg::kSubs; ++s)
          tma_load_4d(sV + stage * Cfg::kTileBytes + s * Cfg::kSubBytes, &tmV, BAR(kBarVFull + stage), s * 64,
                      t * kBN, h, b);
      }
      __syncwarp();
      if (++stage == Cfg::kStages) {
        stage = 0;
        ph ^= 1;
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // whole warp runs the schedule (waits); one elected lane issues tcgen05.mma/commit.
    constexpr uint32_t ab = BF16 ? 1u : 0u;
    constexpr uint32_t idesc_qk = make_idesc_f16(ab, 128, kBN, 0, 0);
    constexpr uint32_t idesc_pv = make_idesc_f16(ab, 128, D, 0, 1);
    // base descriptors; per-MMA operands add (byte offset >> 4) to the start-address field
    const uint64_t qdesc0 = make_sdesc_sw128(sQ, 16, 1024);
    const uint64_t kdesc0 = make_sdesc_sw128(sK, 16, 1024);
    const uint64_t vdesc0 = make_sdesc_sw128(sV, Cfg::kSubBytes, 1024);
    mbar_wait(BAR(kBarQ), 0);
    tc_fence_after();
    TATN_TRACE_AT(7);
    uint32_t acc[2] = {0, 0};
    uint32_t pph[2] = {0, 0};
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
          const long long bit = static_cast<long long>(pair * NQ + q) * p.tc + t;
          atomicOr(p.visited + (bit >> 5), 1u << (bit & 31));
        }
      }
      __syncwarp();
    };
    if constexpr (NQ == 1) {
      // One Q tile: the softmax holds S(t) in registers, so QK(t+1) is issued as soon as
      // S(t) has been read out (SFree) and runs under softmax(t); PV(t) follows P(t).
      int t = sc.next(0);
      int stage = 0;
      uint32_t ph = 0, fph = 0, pph1 = 0;
      int mt = 0;  // tiles issued (trace index)
      if (t < sc.T) {
        mbar_wait(BAR(kBarKFull + 0), 0);
        tc_fence_after();
        issue_qk(0, t, 0);
        if (elect_one_sync()) mma_commit(BAR(kBarKEmpty + 0));
        __syncwarp();
      }
      while (t < sc.T) {
        const int tn = sc.next(t + 1);
        const int sn = (stage + 1 == Cfg::kStages) ? 0 : stage + 1;
        const uint32_t phn = (sn == 0) ? (ph ^ 1) : ph;
        if (tn < sc.T) {
          mbar_wait(BAR(kBarSFree), fph);
          fph ^= 1;
          mbar_wait(BAR(kBarKFull + sn), phn);
          tc_fence_after();
          issue_qk(0, tn, sn);
          if (elect_one_sync()) mma_commit(BAR(kBarKEmpty + sn));
          __syncwarp();
          if (lane == 0) TATN_EV(mt + 1, 4);
        }
        mbar_wait(BAR(kBarPFull + 0), pph1);
        pph1 ^= 1;
        if (lane == 0) TATN_EV(mt, 3);
        mbar_wait(BAR(kBarVFull + stage), ph);
        tc_fence_after();
        if (lane == 0) TATN_EV(mt, 5);
        if (elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk)
            mma_ts(tmem_base + Cfg::kTmemO, tmem_base + Cfg::kTmemP + kk * 8,
                   vdesc0 + ((stage * Cfg::kTileBytes + kk * 2048) >> 4), idesc_pv, (acc[0] | (kk > 0 ? 1u : 0u)));
          mma_commit(BAR(kBarPVDone));
          mma_commit(BAR(kBarVEmpty + stage));
        }
        __syncwarp();
        acc[0] = 1;
        t = tn;
        stage = sn;
        ph = phn;
        ++mt;
      }
      if (elect_one_sync()) mma_commit(BAR(kBarOFinal + 0));
      __syncwarp();
    } else {
    // Schedule per K/V tile t (union order over the CTA's two Q tiles):
    //   PV_A(t), QK_A(t+1), PV_B(t), QK_B(t+1)
    // so softmax A(t+1) starts while softmax B(t) still runs (ping-pong). The
    // look-ahead QK goes only one tile ahead, which keeps the ring deadlock-free
    // when the two tiles visit different block-sparse columns.
    int t = sc.next(0);
    int stage = 0;
    uint32_t ph = 0;
    bool ofinal_done[2] = {false, false};
#ifdef TATN_TRACE
    int dbg_pv = 0;
#endif
    if (t < sc.T) {
      mbar_wait(BAR(kBarKFull + 0), 0);
      tc_fence_after();
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (sc.member(q, t)) issue_qk(q, t, 0);
      if (elect_one_sync()) mma_commit(BAR(kBarKEmpty + 0));
      __syncwarp();
    }
    while (t < sc.T) {
      const int tn = sc.next(t + 1);
      const int sn = (stage + 1 == Cfg::kStages) ? 0 : stage + 1;
      const uint32_t phn = (sn == 0) ? (ph ^ 1) : ph;
      bool k_ready = false;
      bool qk_done[2] = {false, false};
      mbar_wait(BAR(kBarVFull + stage), ph);
      tc_fence_after();
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if (!sc.member(q, t)) continue;
        mbar_wait(BAR(kBarPFull + q), pph[q]);
        pph[q] ^= 1;
        tc_fence_after();
#ifdef TATN_TRACE
        if (q == 0 && ++dbg_pv == 3) TATN_TRACE_AT(11);
#endif
        if (elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < kBN / 16; ++kk) {
            // V tile is MN-major for this product: 16 keys = 2 x 1024B swizzle atoms.
            mma_ts(tmem_base + Cfg::kTmemO + q * D,
                   tmem_base + Cfg::kTmemP + q * (Cfg::kSeparateP ? 64 : 128) + kk * 8,
                   vdesc0 + ((stage * Cfg::kTileBytes + kk * 2048) >> 4), idesc_pv, (acc[q] | (kk > 0 ? 1u : 0u)));
          }
        }
        __syncwarp();
        acc[q] = 1;
        if (!sc.has_after(q, t)) {  // last PV of tile q: its epilogue may start under the other tile's work
          if (elect_one_sync()) mma_commit(BAR(kBarOFinal + q));
          __syncwarp();
          ofinal_done[q] = true;
        }
        if (tn < sc.T && sc.member(q, tn)) {
          if (!k_ready) {
            mbar_wait(BAR(kBarKFull + sn), phn);
            tc_fence_after();
            k_ready = true;
          }
          issue_qk(q, tn, sn);
          qk_done[q] = true;
#ifdef TATN_TRACE
          if (q == 0 && dbg_pv == 3) TATN_TRACE_AT(12);
#endif
        }
      }
      if (elect_one_sync()) mma_commit(BAR(kBarVEmpty + stage));
      __syncwarp();
      if (tn < sc.T) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
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
      stage = sn;
      ph = phn;
    }
    if (elect_one_sync())
      for (int q = 0; q < NQ; ++q)
        if (!ofinal_done[q]) mma_commit(BAR(kBarOFinal + q));
    __syncwarp();
    }  // NQ == 2
  }
  } else {
    if constexpr (NQ == 2) setmaxnreg_inc<208>();  // 2*128*(208-168) <= 128*(168-80)
    // ------------------------------------------------------------ softmax warpgroups
    const int q = warp >> 2;               // Q tile of this warpgroup
    // this warpgroup's schedule as scalars (no dynamically indexed struct -> no local memory)
    const int my_q0 = (q == 0) ? sc.q0[0] : sc.q0[1];
    const int my_nkv = (q == 0) ? sc.nkv[0] : sc.nkv[1];
    const uint32_t* my_mask = (q == 0) ? sc.mask[0] : sc.mask[1];
    auto is_member = [&](int t) -> bool {
      return sc.sparse ? (((my_mask[t >> 5] >> (t & 31)) & 1u) != 0u) : (t < my_nkv);
    };
    const int wq = warp & 3;               // TMEM lane quadrant
    const int row = wq * 32 + lane;        // row within the tile == TMEM lane
    const int grow = my_q0 + row;       // global query row
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t tS = tmem_base + lane_off + Cfg::kTmemS + q * 128;
    const uint32_t tO = tmem_base + lane_off + Cfg::kTmemO + q * D;
    const uint32_t tP = tmem_base + lane_off + Cfg::kTmemP + q * (Cfg::kSeparateP ? 64 : 128);
    // dropout: per-row hash of the reference's positional generator (slice seed = seed + b*H + h)
    uint64_t drow = 0;
    if constexpr (DROP) drow = drop_row_hash(p.drop_seed + static_cast<uint64_t>(bh), grow);
    const float sl2 = p.scale_log2;
    const bool causal = p.mask_kind == kMaskCausal;
    const uint64_t sl2x2 = f2_pack(sl2, sl2);
    const int my_q0c = my_q0 - p.k_off, growc = grow - p.k_off;  // query rows in local key coordinates
    // Custom mask (MaskKind::Custom): this row's keep bits, 4 words per 128-key tile. The row
    // pointer is recomputed from the kernel parameters at each use (no live registers on the
    // unmasked path).
    const bool custom_on = p.custom != nullptr;
    auto load_cw = [&](int t, uint32_t (&cw)[4]) {
      if (p.custom != nullptr && grow < p.Nq) {
        const uint4 w = *reinterpret_cast<const uint4*>(p.custom + static_cast<size_t>(b) * p.custom_bstride +
                                                        static_cast<size_t>(grow) * p.custom_words + p.k_off / 32 +
                                                        4 * t);
        cw[0] = w.x;
        cw[1] = w.y;
        cw[2] = w.z;
        cw[3] = w.w;
      } else {
        cw[0] = cw[1] = cw[2] = cw[3] = (p.custom != nullptr) ? 0u : ~0u;  // rows past Nq are never stored
      }
    };

    float m_run = -INFINITY;  // running max of tau*s*log2(e), possibly stale by <= threshold
    float l_run = 0.f;        // running denominator relative to m_run
    int n_done = 0;
    uint32_t sph = 0;

    if constexpr (NQ == 1) {
      // One Q tile per CTA (d = 64, two CTAs per SM). S(t) is pulled into registers at
      // once and released (SFree) so QK(t+1) runs under this tile's exponentials; P(t)
      // goes to its own TMEM columns once PV(t-1) has drained them (PVDone).
      uint32_t pvph = 0;
      auto wait_pv = [&]() {
        mbar_wait(BAR(kBarPVDone), pvph);
        pvph ^= 1;
        tc_fence_after();
      };
      for (int t = sc.next(0); t < sc.T; t = sc.next(t + 1)) {
        mbar_wait(BAR(kBarSFull + 0), sph);
        sph ^= 1;
        tc_fence_after();
        if (threadIdx.x == 0) TATN_EV(n_done, 0);
        if (threadIdx.x == 0 && n_done == 0) TATN_TRACE_AT(1);
        if (threadIdx.x == 0 && n_done == 2) TATN_TRACE_AT(8);
        if (threadIdx.x == 0 && n_done == 3) TATN_TRACE_AT(13);
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
        if (threadIdx.x == 0) TATN_EV(n_done, 1);
        const int k0 = t * kBN;
        const bool need_mask = (k0 + kBN > sc.kv_limit) || (causal && k0 + kBN - 1 > my_q0c) || custom_on;
        const int lim = min(sc.kv_limit, causal ? growc + 1 : sc.kv_limit) - k0;  // columns >= lim are masked
        auto step = [&](auto masked_t) {
          constexpr bool kMasked = decltype(masked_t)::value;
          if constexpr (kMasked) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int i = 0; i < 32; ++i)
                sv[c][i] = (c * 32 + i >= lim) ? __float_as_uint(-INFINITY) : sv[c][i];
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
          bool pv_ready = n_done == 0;
          if (__any_sync(0xffffffffu, jump)) {  // warp-uniform: TMEM ld/st below are .sync.aligned
            float alpha = 1.f;
            if (jump) {
              alpha = ex2_approx(m_run - m_tile);  // 0 when m_run == -inf
              m_run = m_tile;
              l_run *= alpha;
            }
            if (!pv_ready) {
              wait_pv();  // O is final up to tile t-1
              pv_ready = true;
#pragma unroll 1
              for (int c = 0; c < D / 16; ++c) {  // 16 columns at a time: S(t) is still live
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
              // the polynomial needs finite x: full tiles only (m_run <= true max + threshold)
              if (!kMasked && !DROP && kEmuPairs > 0 && (i & 7) < kEmuPairs) {
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
            if (c == 0 && !pv_ready) wait_pv();  // PV(t-1) has read P(t-1)
            tmem_st16(tP + c * 16, pk);
          }
          float rs0, rs1, rs2, rs3;
          f2_unpack(rsum0, rs0, rs1);
          f2_unpack(rsum1, rs2, rs3);
          l_run += (rs0 + rs1) + (rs2 + rs3);
        };
        if (custom_on) {  // Custom mask: -inf where the keep bit is 0 (then the usual masked step)
          uint32_t cw[4];
          load_cw(t, cw);
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i)
              sv[c][i] = ((cw[c] >> i) & 1u) ? sv[c][i] : __float_as_uint(-INFINITY);
        }
        if (need_mask) step(std::true_type{});
        else step(std::false_type{});
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(BAR(kBarPFull + 0));
        if (threadIdx.x == 0) TATN_EV(n_done, 2);
        if (threadIdx.x == 0) TATN_TRACE_AT(2);
        if (threadIdx.x == 0 && n_done == 2) TATN_TRACE_AT(10);
        ++n_done;
      }
    } else {
    for (int t = sc.next(0); t < sc.T; t = sc.next(t + 1)) {
      if (!is_member(t)) continue;
      mbar_wait(BAR(kBarSFull + q), sph);
      if (threadIdx.x == 0 && n_done == 0) TATN_TRACE_AT(1);
      if (threadIdx.x == 0 && n_done == 2) TATN_TRACE_AT(8);
      if (threadIdx.x == 0 && n_done == 3) TATN_TRACE_AT(13);
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
      // One streaming pass over S: p = 2^(s*scale_log2 - m_use) per 32-column chunk
      // (FFMA2 scale, MUFU ex2 or the FMA-pipe polynomial for (i & 7) < kEmuPairs on
      // full tiles), P (16-bit) to TMEM at tP, row sum in FP32x2; optionally tracks
      // the raw row max. With aliased P (tP == tS) chunk c lands on S columns
      // [16c, 16c+16), which the pass has already consumed.
      auto exp_pass = [&](float m_use, float& raw_max) -> float {
        const uint64_t negm = f2_pack(-m_use, -m_use);
        uint64_t rsum0 = f2_pack(0.f, 0.f), rsum1 = rsum0;
        float mx0 = -INFINITY, mx1 = -INFINITY;
        uint32_t ra[32], rb[32];
        tmem_ld32_async(tS, ra);
        tmem_ld_wait32(ra);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t (&r)[32] = (c & 1) ? rb : ra;
          uint32_t (&nxt)[32] = (c & 1) ? ra : rb;
          if (c + 1 < 4) tmem_ld32_async(tS + (c + 1) * 32, nxt);
          apply_mask(r, c);
          if (Cfg::kSeparateP) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              mx0 = fmax3(mx0, __uint_as_float(r[i]), __uint_as_float(r[i + 1]));
              mx1 = fmax3(mx1, __uint_as_float(r[i + 2]), __uint_as_float(r[i + 3]));
            }
          }
          uint32_t pk[16];
          // straight-line bodies: the polynomial pairs interleave with the MUFU pairs
          auto exp_chunk = [&](auto emu_on) {
            constexpr bool kEmu = decltype(emu_on)::value;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const int i = c * 16 + k;
              const uint64_t x =
                  f2_fma(f2_pack(__uint_as_float(r[2 * k]), __uint_as_float(r[2 * k + 1])), sl2x2, negm);
              uint64_t pv;
              if constexpr (TATN_EX2_16 && !OUT_F32 && !DROP) {
                float x0, x1;
                f2_unpack(x, x0, x1);
                pk[k] = ex2_pair16<BF16>(x0, x1);
                pv = widen_pair16<BF16>(pk[k]);  // l sums exactly the P the MMA consumes
              } else {
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
              }
              if (k & 1) rsum1 = f2_add(rsum1, pv);
              else rsum0 = f2_add(rsum0, pv);
            }
          };
          // the polynomial needs finite x: full tiles with m_use <= the true max + threshold
          if (kEmuPairsD<D> > 0 && !need_mask && !DROP) exp_chunk(std::true_type{});
          else exp_chunk(std::false_type{});
          tmem_st16(tP + c * 16, pk);
          if (c + 1 < 4) tmem_ld_wait32(nxt);
        }
        raw_max = fmaxf(mx0, mx1);
        float rs0, rs1, rs2, rs3;
        f2_unpack(rsum0, rs0, rs1);
        f2_unpack(rsum1, rs2, rs3);
        return (rs0 + rs1) + (rs2 + rs3);
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
      bool settled = false;
      if (Cfg::kSeparateP && n_done > 0 && __all_sync(0xffffffffu, m_run != -INFINITY)) {
        // optimistic single pass against the running max; redo only if the max jumped
        // past the lazy-rescale threshold (the polynomial clamps overflowing inputs, and
        // such a pass is discarded)
        float raw_max;
        row_sum = exp_pass(m_run, raw_max);
        const float m_tile = raw_max * sl2;
        const bool jumped = m_tile - m_run > kRescaleThreshold;
        settled = !__any_sync(0xffffffffu, jumped);
        if (!settled) {  // warp-uniform branch: TMEM ld/st below are .sync.aligned
          float alpha = 1.f;
          if (jumped) {
            alpha = ex2_approx(m_run - m_tile);
            m_run = m_tile;
            l_run *= alpha;
          }
          rescale_o(alpha, jumped);
        }
      }
      if (!settled) {
        float m_tile;
        if (Cfg::kSeparateP && n_done > 0 && __all_sync(0xffffffffu, m_run != -INFINITY)) {
          m_tile = m_run;  // already advanced above
        } else {
          // pass 1: row max, streaming S from TMEM in 32-column chunks (3-input max)
          float mx0 = -INFINITY, mx1 = -INFINITY;
          uint32_t ra[32], rb[32];
          tmem_ld32_async(tS, ra);
          tmem_ld_wait32(ra);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t (&cur)[32] = (c & 1) ? rb : ra;
            uint32_t (&nxt)[32] = (c & 1) ? ra : rb;
            if (c + 1 < 4) tmem_ld32_async(tS + (c + 1) * 32, nxt);
            apply_mask(cur, c);
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              mx0 = fmax3(mx0, __uint_as_float(cur[i]), __uint_as_float(cur[i + 1]));
              mx1 = fmax3(mx1, __uint_as_float(cur[i + 2]), __uint_as_float(cur[i + 3]));
            }
            if (c + 1 < 4) tmem_ld_wait32(nxt);
          }
          m_tile = fmaxf(mx0, mx1) * sl2;
          float alpha = 1.f;
          if (m_tile - m_run > kRescaleThreshold) {  // false for NaN (both -inf)
            alpha = ex2_approx(m_run - m_tile);      // 0 when m_run == -inf
            m_run = m_tile;
          }
          l_run *= alpha;
          rescale_o(alpha, (n_done > 0) && (alpha != 1.f));
        }
        if (threadIdx.x == 0 && n_done == 2) TATN_TRACE_AT(9);
        float unused;
        row_sum = exp_pass((m_run == -INFINITY) ? 0.f : m_run, unused);
      }
      l_run += row_sum;
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(BAR(kBarPFull + q));
      if (threadIdx.x == 0) TATN_TRACE_AT(2);
      if (threadIdx.x == 0 && n_done == 2) TATN_TRACE_AT(10);
      ++n_done;
    }
    }  // NQ == 2

    n_steps_dbg = n_done;
    // ------------------------------------------------------------ epilogue
    if (my_q0 < p.Nq) {
      mbar_wait(BAR(kBarQ), 0);  // Q_q smem is reused as the O staging buffer
      const float inv_l = (l_run > 0.f) ? 1.f / l_run : 0.f;
      const uint32_t sO = sQ + q * Cfg::kTileBytes;
      if (n_done > 0) {
        mbar_wait(BAR(kBarOFinal + q), 0);
        tc_fence_after();
      }
      if (threadIdx.x == 0) TATN_TRACE_AT(3);
      float* orow = nullptr;
      if constexpr (OUT_F32)
        orow = p.o_f32 + static_cast<size_t>(b) * p.o_sb + static_cast<size_t>(h) * p.o_sh +
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
          const int sub = (c * 32) / 64;
          const int chunk0 = ((c * 32) % 64) / 8;
          const uint32_t rbase = sO + sub * Cfg::kSubBytes + row * 128;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t addr = rbase + (((chunk0 + j) ^ (row & 7)) << 4);
            st_shared_v4(addr, pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          }
        }
      }
      if (grow < p.Nq) {
        const float lse = (l_run > 0.f) ? (m_run + __log2f(l_run)) * 0.69314718055994530942f : -INFINITY;
        p.lse[static_cast<size_t>(bh) * p.Nq + grow] = lse;
      }
      if constexpr (!OUT_F32) {
        fence_proxy_async_smem();
        named_bar_sync(1 + q, 128);
        if (row == 0) {
          for (int s = 0; s < Cfg::kSubs; ++s) tma_store_4d(&tmO, sO + s * Cfg::kSubBytes, s * 64, my_q0, h, b);
          bulk_commit();
          bulk_wait_read_all();
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    TATN_TRACE_AT(4);
#ifdef TATN_TRACE
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    if (g_tatn_trace) g_tatn_trace[static_cast<size_t>(blockIdx.x) * 16 + 5] = smid;
    if (g_tatn_trace) g_tatn_trace[static_cast<size_t>(blockIdx.x) * 16 + 6] = static_cast<unsigned long long>(n_steps_dbg);
#endif
  }
  if (warp == kMmaWarp) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

}  // namespace tatn_dev

namespace tatn_dev {
// ---------------------------------------------------------------- partial-result merge
// merge_stats (softmax.cpp:62-83) in log form over R key shards; one thread per 8 elements
// of a row. HBM-bound: reads R * (d * 4 + 4) bytes and writes d * es + 4 bytes per row.
__global__ void __launch_bounds__(256) tatn_merge_kernel(int R, long long rows, int d, int H, int Nq,
                                                         const float* __restrict__ o_parts,
                                                         const float* __restrict__ lse_parts, void* __restrict__ o,
                                                         int o_dtype, int64_t ob, int64_t oh, int64_t on,
                                                         float* __restrict__ lse) {
  griddep_wait();  // programmatic dependent launch: inputs of the previous kernel visible
  griddep_launch();
  // grid (row blocks, H, B): no per-thread 64-bit index divisions
  const int chunks = d / 8;
  const int c = static_cast<int>(threadIdx.x) % chunks;
  const int n = static_cast<int>(blockIdx.x) * (256 / chunks) + static_cast<int>(threadIdx.x) / chunks;
  const int h = static_cast<int>(blockIdx.y), b = static_cast<int>(blockIdx.z);
  if (n >= Nq) return;
  const long long row = (static_cast<long long>(b) * H + h) * Nq + n;
  float m = -INFINITY;
  for (int r = 0; r < R; ++r) m = fmaxf(m, lse_parts[static_cast<size_t>(r) * rows + row]);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float wsum = 0.f;
  if (m != -INFINITY) {
    for (int r = 0; r < R; ++r) {
      const float lr = lse_parts[static_cast<size_t>(r) * rows + row];
      const float w = (lr == -INFINITY) ? 0.f : expf(lr - m);
      if (w == 0.f) continue;
      wsum += w;
      const float4* src = reinterpret_cast<const float4*>(o_parts + (static_cast<size_t>(r) * rows + row) * d + c * 8);
      const float4 a = src[0], b = src[1];
      acc[0] = fmaf(w, a.x, acc[0]); acc[1] = fmaf(w, a.y, acc[1]); acc[2] = fmaf(w, a.z, acc[2]);
      acc[3] = fmaf(w, a.w, acc[3]); acc[4] = fmaf(w, b.x, acc[4]); acc[5] = fmaf(w, b.y, acc[5]);
      acc[6] = fmaf(w, b.z, acc[6]); acc[7] = fmaf(w, b.w, acc[7]);
    }
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  const size_t off = static_cast<size_t>(b) * ob + static_cast<size_t>(h) * oh + static_cast<size_t>(n) * on + c * 8;
  if (o_dtype == 2) {
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(o) + off);
    dst[0] = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
    dst[1] = make_float4(acc[4] * inv, acc[5] * inv, acc[6] * inv, acc[7] * inv);
  } else {
    uint4 out;
    if (o_dtype == 0) {
      out = make_uint4(pack2<true>(acc[0] * inv, acc[1] * inv), pack2<true>(acc[2] * inv, acc[3] * inv),
                       pack2<true>(acc[4] * inv, acc[5] * inv), pack2<true>(acc[6] * inv, acc[7] * inv));
    } else {
      out = make_uint4(pack2<false>(acc[0] * inv, acc[1] * inv), pack2<false>(acc[2] * inv, acc[3] * inv),
                       pack2<false>(acc[4] * inv, acc[5] * inv), pack2<false>(acc[6] * inv, acc[7] * inv));
    }
    *reinterpret_cast<uint4*>(static_cast<uint16_t*>(o) + off) = out;
  }
  if (c == 0) lse[row] = wsum > 0.f ? m + logf(wsum) : -INFINITY;
}
}  // namespace tatn_dev
