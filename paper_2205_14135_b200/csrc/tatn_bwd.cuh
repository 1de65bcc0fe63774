// tatn_bwd.cuh — FlashAttention backward for sm_100a (kernels K2, K3, K4).
//
// Replaces the body of tatn::flash_backward / tatn::blocksparse_backward
// (reference flash.hpp:53-73), i.e. Algorithm 4 without
// dropout: P is recomputed per tile from the saved logsumexp, D_i =
// rowsum(dO_i * O_i) (reference.cpp:287-290), dS = P * (dP - D),
// dV = P^T dO, dK = tau dS^T Q, dQ = tau dS K. As in Alg 4 the K/V block is
// the outer loop (one CTA per 128-key tile) and dQ is a read-modify-write
// accumulation — here an fp32 bulk reduce-add into an L2-resident workspace.
//
//   K2 tatn_bwd_pre   : -D_i, -lse2_i = -LSE_i*log2(e) (-inf for empty/padded rows), zero dQacc
//   K3 tatn_bwd_kernel: per (b, h, key tile) loop over 64-row Q tiles
//   K4 tatn_bwd_post  : dQ = bf16/fp16(dQacc)
//
// K3 CTA layout (d = 64: 480 threads, d = 128: 448):
//   warps 0-3 "softmax 0": thread = key row (TMEM lane). Recompute P^T, dS^T for even Q tiles.
//   warps 4-7 "softmax 1": the same for odd Q tiles (ping-pong: two tiles in softmax at once).
//   warps 8-11 "dQ":       thread = head-dim row of dQ^T (TMEM lane); stage + bulk reduce.
//   warp 12   TMA producer (K, V once; Q_i, dO_i, lse2_i, D_i ring)
//   warp 13   TMEM allocator + tcgen05.mma issuer (d = 64: the fronts)
//   warp 14   d = 64 only: tcgen05.mma issuer of the backs (dV, dK, dQ^T)
// Per Q tile i the MMA computes (M = 128 keys unless noted)
//   front: S^T = K Q_i^T, dP^T = V dO_i^T                      (N = 64 queries)
//   back : dV += P^T dO_i, dK += dS^T Q_i  (A from TMEM)       (N = d)
//          dQ_i^T = K^T dS^T  (M = d rows used, A/B from SMEM) (N = 64 queries)
// with two TMEM buffers X0/X1 holding {S^T | dP^T}, one per softmax warpgroup.
// dS is kept unscaled (tau is applied to dK in the epilogue and to dQ in the dQ
// warpgroup), so the softmax step is P = 2^(S*tau*log2e - lse2), dS = P*(dP - D).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <type_traits>

#include "../../include/tatn_b200.h"
#include "sm100_ptx.cuh"
#include "tatn_params.h"
#include "tatn_launch.h"

#ifndef TATN_BWD_SEP_STAGE
#define TATN_BWD_SEP_STAGE 1  // d = 64: dK / dV staging in its own shared-memory region
#endif
#ifndef TATN_BWD_STAGES_D64
#define TATN_BWD_STAGES_D64 5  // d = 64 Q / dO ring depth (the early front (g + 2) reads stage (g + 2) % S)
#endif
#ifndef TATN_BWD_DS_BUFS
#define TATN_BWD_DS_BUFS 2  // d = 64 dS^T buffers (3 measured no faster: the softmax is not waiting on them)
#endif
#ifndef TATN_DQ_RED
#define TATN_DQ_RED 1  // dQ partials: red.global.add from registers (1) or smem staging + bulk reduce (0)
#endif

namespace tatn_dev {

constexpr int kBwdQT = 64;    // query rows per Q tile
constexpr int kBwdKT = 128;   // keys per CTA

template <int D, bool DROP = false>
struct BwdCfg {
  static constexpr int kSubs = D / 64;
  static constexpr int kKVTile = kSubs * 128 * 128;   // 128 rows x D x 2B
  static constexpr int kQSub = 64 * 128;              // 64 rows x 128B
  static constexpr int kQTile = kSubs * kQSub;        // 64 rows x D x 2B
  // d = 128 with dropout drops to 2 stages to make room for the per-warpgroup row hashes
  static constexpr int kStages = (D == 128) ? (DROP ? 2 : 3) : TATN_BWD_STAGES_D64;
  static constexpr int kDSBytes = 128 * 128;          // 128 keys x 64 q x 2B
  // dS^T shared-memory buffers (tile g uses g % kDSBufs): with 3 at d = 64 the softmax of tile
  // g waits for the dQ^T MMA of tile g - 3, not g - 2 (issued after the front of tile g)
  static constexpr int kDSBufs = (D == 64) ? TATN_BWD_DS_BUFS : 2;
  static_assert(kDSBufs >= 2, "the ping-pong needs two dS^T buffers");
  // fp32 dQ staging (d = 64 issues its dQ reductions from registers: no staging)
  static constexpr int kDQBytes = (TATN_DQ_RED && D == 64) ? 0 : kBwdQT * D * 4;
  static constexpr int kVecBytes = 2 * kBwdQT * 4;    // lse2 + D
  // K/V buffers: double-buffered at d = 64 (the next item's K/V lands while this one runs)
  static constexpr int kKVBufs = (D == 64) ? 2 : 1;
  static constexpr int kOffKV = 0;
  static constexpr int kOffQ = kOffKV + kKVBufs * 2 * kKVTile;
  static constexpr int kOffDO = kOffQ + kStages * kQTile;
  static constexpr int kOffDS = kOffDO + kStages * kQTile;
  static constexpr int kOffDQ = kOffDS + kDSBufs * kDSBytes;
  static constexpr int kOffVec = kOffDQ + kDQBytes;
  static constexpr int kOffBar = kOffVec + kStages * kVecBytes;
  static constexpr int kOffRing = kOffBar + 384;       // item ring (kItemRing ints)
  static constexpr int kOffMask = kOffRing + 64;       // block-sparse q-tile bitmasks, 128 words each
  // d = 64: one bitmask per item-ring slot (block-sparse launches run persistent too);
  // d = 128 has no shared memory left for them: block-sparse runs one item per CTA
  static constexpr int kMaskSlots = (D == 64) ? 4 : 1;
  static constexpr int kOffDrop = kOffMask + 512 * kMaskSlots;  // dropout: 64 query-row hashes per softmax warpgroup
  // d = 64: the dK / dV output staging has its own region (d = 128 has no room: it aliases the
  // dS^T + dQ staging and the next item's first dS^T store waits for the store to read it)
  static constexpr bool kSepStage = D == 64 && TATN_BWD_SEP_STAGE;
  static constexpr int kOffStage = ((kOffDrop + (DROP ? 1024 : 0)) + 1023) / 1024 * 1024;
  static constexpr int kSmemBytes =
      kSepStage ? kOffStage + 2 * 128 * D * 2 : kOffDrop + (DROP ? 1024 : 0);  // declared __align__(1024)
  static_assert(kSmemBytes <= 232448, "K3 shared memory exceeds the 227 KB opt-in limit");
  static_assert(2 * 128 * D * 2 <= kOffVec - kOffDS, "dK/dV staging must fit the dS^T + dQ staging region");
  static constexpr uint32_t kTmemX = 0;    // X_x = x*128: S^T [0,64) dP^T [64,128)
  // d = 64: P^T / dS^T (16-bit) go to their own columns PdS_x = [256 + 64x, 320 + 64x) (P^T
  // [0,32), dS^T [32,64)) instead of over S^T / dP^T, so the softmax releases X_x as soon as it
  // holds S^T / dP^T in registers and the front of Q tile g + 2 runs under the rest of its work
  // (with X_x aliased the front had to wait for back(g)); dQ^T(g) then lands in PdS_x once
  // back(g) has read P^T / dS^T. d = 128 has no free columns: P^T / dS^T alias X_x.
  static constexpr bool kEarlyX = (D == 64);
  // warps 0-7 softmax, 8-11 dQ, 12 TMA producer, 13 MMA (d = 64: fronts), 14 (d = 64) MMA backs
  static constexpr int kThreads = kEarlyX ? 480 : 448;
  static constexpr uint32_t kTmemPdS = 256;
  static constexpr uint32_t kTmemDV = kEarlyX ? 384 : 256;
  static constexpr uint32_t kTmemDK = kTmemDV + D;
  // dQ partials by red.global.add from registers (d = 64: frees the shared-memory port of
  // the staging write + bulk-reduce read); d = 128 keeps smem staging + one bulk reduce,
  // which measured faster there (r01 sweep)
  static constexpr bool kDQRed = TATN_DQ_RED && D == 64;
  // d = 64: dQ^T by an M = 64 MMA. Its rows live in TMEM lanes 0-15 of each 32-lane
  // quadrant (row = 16 * quadrant + lane).
  static constexpr bool kDQ64 = D == 64;
};

struct BwdSched {
  int k0;        // first key of the tile
  int kv_limit;  // keys >= kv_limit are masked
  int i_begin;   // first candidate Q tile (64 rows)
  int i_end;     // one past the last candidate Q tile
  const uint8_t* gcol;  // block-sparse grid column base (grid + j), stride tc; nullptr = dense
  int tc;
  const uint32_t* mask; // block-sparse: shared-memory bitmask over 64-row Q tiles

  // first visited Q tile >= i (i_end when none)
  __device__ __forceinline__ int next(int i) const {
    if (gcol == nullptr) return i;
    while (i < i_end) {
      const int w = i >> 5;
      const uint32_t m = mask[w] >> (i & 31);
      if (m) return i + __ffs(m) - 1;
      i = (w + 1) << 5;
    }
    return i_end;
  }
};

// duplicate each of the 16 low bits: b0 b1 ... -> b0 b0 b1 b1 ...
__device__ __forceinline__ uint32_t spread_bits16(uint32_t x) {
  x &= 0xffffu;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x | (x << 1);
}

__device__ __forceinline__ BwdSched make_bwd_sched(const BwdParams& p, int b, int j) {
  BwdSched s;
  s.k0 = j * kBwdKT;
  int kv_limit = p.Nk;
  // key j of this call is global key k_off + j (sequence-parallel shards); valid_len is global
  if (p.mask_kind == kMaskKeyPadding && p.valid_len != nullptr) kv_limit = min(kv_limit, max(p.valid_len[b] - p.k_off, 0));
  s.kv_limit = kv_limit;
  s.tc = p.tc;
  const int n_qt = (p.Nq + kBwdQT - 1) / kBwdQT;
  if (p.grid != nullptr) {
    s.gcol = p.grid + j;
    s.i_begin = 0;
    s.i_end = n_qt;
  } else {
    s.gcol = nullptr;
    s.i_begin = (p.mask_kind == kMaskCausal) ? ((s.k0 + p.k_off) / kBwdQT) : 0;
    s.i_end = (s.k0 < kv_limit) ? n_qt : 0;
  }
  if (s.i_begin > s.i_end) s.i_begin = s.i_end;
  return s;
}

// ---------------------------------------------------------------- K2
// One 8-element chunk per thread; grid (row blocks, H, B) so no thread divides 64-bit indices
// (the divisions cost as much issue time as the bytes these HBM-bound kernels move). Rows are
// padded to a multiple of 128.
// DO_F32: dO (and O) are fp32 — the fp32-input check mode (tatn_tf32.cuh)
template <int D, bool BF16, bool O_F32, bool DO_F32 = false>
__global__ void __launch_bounds__(256) tatn_bwd_pre(const void* __restrict__ o_, const void* __restrict__ dO_,
                                                    const float* __restrict__ lse, int64_t ob, int64_t oh, int64_t on,
                                                    int B, int H, int Nq, int Nq_pad, float* __restrict__ lse2,
                                                    float* __restrict__ delta, float* __restrict__ dq_acc,
                                                    int* __restrict__ item_counter) {
  griddep_wait();  // programmatic dependent launch: inputs of the previous kernel visible
  griddep_launch();
  constexpr int kChunks = D / 8;
  constexpr int kRowsPerBlock = 256 / kChunks;
  const int c = static_cast<int>(threadIdx.x) % kChunks;
  const int qi = static_cast<int>(blockIdx.x) * kRowsPerBlock + static_cast<int>(threadIdx.x) / kChunks;
  const int h = static_cast<int>(blockIdx.y), b = static_cast<int>(blockIdx.z);
  const long long bh = static_cast<long long>(b) * H + h;
  const long long row = bh * Nq_pad + qi;  // over B*H*Nq_pad
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0)
    *item_counter = 0;  // K3's persistent scheduler starts from item 0
  float part = 0.f;
  if (qi < Nq_pad) {
    if (qi < Nq) {
      const size_t off = static_cast<size_t>(b) * ob + static_cast<size_t>(h) * oh + static_cast<size_t>(qi) * on + c * 8;
      float of[8], df[8];
      if constexpr (DO_F32) {
        // tf32 check mode: dP = dO V^T is formed from dO rounded to tf32, so D = rowsum(dO o O)
        // uses the same rounded dO — then sum_j P_ij (dP_ij - D_i) = 0 holds as in exact arithmetic
        // (the gradient is exact for the rounded dO instead of carrying its rounding in dS)
        const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(dO_) + off);
        const float4 a0 = src[0], a1 = src[1];
        df[0] = round_tf32(a0.x); df[1] = round_tf32(a0.y); df[2] = round_tf32(a0.z); df[3] = round_tf32(a0.w);
        df[4] = round_tf32(a1.x); df[5] = round_tf32(a1.y); df[6] = round_tf32(a1.z); df[7] = round_tf32(a1.w);
      } else {
        const uint4 dv = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dO_) + off);
        const uint32_t* dw = reinterpret_cast<const uint32_t*>(&dv);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float2 bb;
          if constexpr (BF16) bb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&dw[k]));
          else bb = __half22float2(*reinterpret_cast<const __half2*>(&dw[k]));
          df[2 * k] = bb.x;
          df[2 * k + 1] = bb.y;
        }
      }
      if constexpr (O_F32) {
        const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(o_) + off);
        const float4 a0 = src[0], a1 = src[1];
        of[0] = a0.x; of[1] = a0.y; of[2] = a0.z; of[3] = a0.w;
        of[4] = a1.x; of[5] = a1.y; of[6] = a1.z; of[7] = a1.w;
      } else {
        const uint4 ov = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(o_) + off);
        const uint32_t* ow = reinterpret_cast<const uint32_t*>(&ov);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float2 a;
          if constexpr (BF16) a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ow[k]));
          else a = __half22float2(*reinterpret_cast<const __half2*>(&ow[k]));
          of[2 * k] = a.x;
          of[2 * k + 1] = a.y;
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) part = fmaf(of[k], df[k], part);
    }
    float4* dst = reinterpret_cast<float4*>(dq_acc + row * D + c * 8);
    dst[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    dst[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // reduce over the kChunks lanes of this row (kChunks in {8, 16}, aligned within a warp)
#pragma unroll
  for (int off = kChunks / 2; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
  if (qi < Nq_pad && c == 0) {
    delta[row] = -part;    // stored negated: the softmax step adds it
    float nl2 = -INFINITY;  // P = 0 for padded or fully-masked rows
    if (qi < Nq) {
      const float l = lse[bh * Nq + qi];
      if (l != -INFINITY) nl2 = -l * 1.4426950408889634f;
    }
    lse2[row] = nl2;
  }
}

// ---------------------------------------------------------------- K4
template <int D, bool BF16, bool OUT_F32>
__global__ void __launch_bounds__(256) tatn_bwd_post(const float* __restrict__ dq_acc, void* __restrict__ dq,
                                                     int64_t qb, int64_t qh, int64_t qn, int B, int H, int Nq,
                                                     int Nq_pad) {
  griddep_wait();  // programmatic dependent launch: inputs of the previous kernel visible
  griddep_launch();
  constexpr int kChunks = D / 8;
  constexpr int kRowsPerBlock = 256 / kChunks;
  const int c = static_cast<int>(threadIdx.x) % kChunks;
  const int qi = static_cast<int>(blockIdx.x) * kRowsPerBlock + static_cast<int>(threadIdx.x) / kChunks;
  const int h = static_cast<int>(blockIdx.y), b = static_cast<int>(blockIdx.z);
  const long long bh = static_cast<long long>(b) * H + h;
  if (qi >= Nq) return;
  const float4* src = reinterpret_cast<const float4*>(dq_acc + (bh * Nq_pad + qi) * D + c * 8);
  const float4 a = src[0], bb = src[1];
  const size_t off = static_cast<size_t>(b) * qb + static_cast<size_t>(h) * qh + static_cast<size_t>(qi) * qn + c * 8;
  if constexpr (OUT_F32) {
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(dq) + off);
    dst[0] = a;
    dst[1] = bb;
  } else {
    uint4 out;
    out.x = pack2<BF16>(a.x, a.y);
    out.y = pack2<BF16>(a.z, a.w);
    out.z = pack2<BF16>(bb.x, bb.y);
    out.w = pack2<BF16>(bb.z, bb.w);
    *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dq) + off) = out;
  }
}

// ---------------------------------------------------------------- K4, deterministic dQ
// dQ = sum over the key tiles j that visited the row's Q tile, in ascending j, of the partials K3
// stored in slot j (plain stores, no atomics): bit-reproducible, and the same for a dense call and
// an all-true block grid. Which (j, Q tile) pairs K3 visited is recomputed from K3's schedule
// (make_bwd_sched; qt = K3's Q-tile height: 64, or the tf32 kernel's): causal ->
// qt-tile index >= (128 j + k_off) / qt; key padding -> 128 j < valid_len[b] - k_off; block grid
// -> grid[row / 128][j].
template <int D, bool BF16, bool OUT_F32>
__global__ void __launch_bounds__(256) tatn_bwd_post_det(const float* __restrict__ dq_part, void* __restrict__ dq,
                                                         int64_t qb, int64_t qh, int64_t qn, int B, int H, int Nq,
                                                         int Nq_pad, int tc, int qt, int causal, int k_off,
                                                         const int32_t* __restrict__ valid_len,
                                                         const uint8_t* __restrict__ grid) {
  griddep_wait();  // programmatic dependent launch: inputs of the previous kernel visible
  griddep_launch();
  constexpr int kChunks = D / 8;
  constexpr int kRowsPerBlock = 256 / kChunks;
  const int c = static_cast<int>(threadIdx.x) % kChunks;
  const int qi = static_cast<int>(blockIdx.x) * kRowsPerBlock + static_cast<int>(threadIdx.x) / kChunks;
  const int h = static_cast<int>(blockIdx.y), b = static_cast<int>(blockIdx.z);
  if (qi >= Nq) return;
  const long long bh = static_cast<long long>(b) * H + h;
  const long long slot = static_cast<long long>(B) * H * Nq_pad * D;
  int kv_limit = 1 << 30;
  if (valid_len != nullptr) kv_limit = valid_len[b] - k_off;
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int j = 0; j < tc; ++j) {
    bool visited;
    if (grid != nullptr) visited = grid[static_cast<size_t>(qi / 128) * tc + j] != 0;
    else visited = (!causal || qi / qt >= (128 * j + k_off) / qt) && 128 * j < kv_limit;
    if (!visited) continue;
    const float4* src = reinterpret_cast<const float4*>(dq_part + j * slot + (bh * Nq_pad + qi) * D + c * 8);
    const float4 x = src[0], y = src[1];
    a[0] += x.x; a[1] += x.y; a[2] += x.z; a[3] += x.w;
    a[4] += y.x; a[5] += y.y; a[6] += y.z; a[7] += y.w;
  }
  const size_t off = static_cast<size_t>(b) * qb + static_cast<size_t>(h) * qh + static_cast<size_t>(qi) * qn + c * 8;
  if constexpr (OUT_F32) {
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(dq) + off);
    dst[0] = make_float4(a[0], a[1], a[2], a[3]);
    dst[1] = make_float4(a[4], a[5], a[6], a[7]);
  } else {
    uint4 out;
    out.x = pack2<BF16>(a[0], a[1]);
    out.y = pack2<BF16>(a[2], a[3]);
    out.z = pack2<BF16>(a[4], a[5]);
    out.w = pack2<BF16>(a[6], a[7]);
    *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dq) + off) = out;
  }
}

// ---------------------------------------------------------------- K2b (Custom masks only)
// Transpose the keep bits [nb][Nq][words] (query rows) into [nb][Nk][Nq_pad/32] (key rows), so
// K3's softmax thread (one key row) reads its 64 query bits of a Q tile with one 8-byte load.
// One warp per 32 x 32 bit block: lane l loads row q0+l's word, 32 ballots transpose it.
__global__ void __launch_bounds__(256) tatn_custom_transpose(const uint32_t* __restrict__ in, int words, int64_t bstride,
                                                             int nb, int Nq, int Nk, int tw, uint32_t* __restrict__ out,
                                                             int kw_off) {
  griddep_wait();  // programmatic dependent launch: inputs of the previous kernel visible
  griddep_launch();
  const long long wid = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = static_cast<int>(threadIdx.x & 31);
  const int kwords = (Nk + 31) / 32;
  const long long total = static_cast<long long>(nb) * tw * kwords;
  if (wid >= total) return;  // warp-uniform
  const int kw = static_cast<int>(wid % kwords);
  const long long r = wid / kwords;
  const int qw = static_cast<int>(r % tw);
  const int bsel = static_cast<int>(r / tw);
  const int q = qw * 32 + lane;
  const uint32_t w =
      (q < Nq) ? in[static_cast<size_t>(bsel) * bstride + static_cast<size_t>(q) * words + kw_off + kw] : 0u;
  uint32_t mine = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const uint32_t col = __ballot_sync(0xffffffffu, (w >> j) & 1u);  // bit l = keep(q0 + l, 32 kw + j)
    if (lane == j) mine = col;
  }
  const int kj = kw * 32 + lane;
  if (kj < Nk) out[(static_cast<size_t>(bsel) * Nk + kj) * tw + qw] = mine;
}

// ---------------------------------------------------------------- K3
// Item w (one 128-key tile of one head) -> (bh, j). Items are laid out in head groups:
// the key tiles of `group` heads are adjacent, so their Q / dO tiles and fp32 dQ
// accumulators stay L2-resident; within a group the heaviest tiles (j = 0 under a
// causal mask) come first.
__device__ __forceinline__ void bwd_item(const BwdParams& p, int w, int& bh, int& j) {
  const int per_group = p.group * p.n_ktiles;
  const int grp = w / per_group;
  const int r = w - grp * per_group;
  const int gsz = min(p.group, p.B * p.H - grp * p.group);
  j = r / gsz;
  bh = grp * p.group + (r - j * gsz);
}
constexpr int kItemRing = 4;  // items published by the producer warp to the other roles

template <int D, bool BF16, bool OUT_F32, bool DROP>
__global__ void __launch_bounds__(BwdCfg<D, DROP>::kThreads, 1)
    tatn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                    const __grid_constant__ CUtensorMap tmDK, const __grid_constant__ CUtensorMap tmDV,
                    const BwdParams p, const float* __restrict__ lse2, int Nq_pad) {
  using Cfg = BwdCfg<D, DROP>;
  constexpr int S = Cfg::kStages;
  constexpr int NKV = Cfg::kKVBufs;
  constexpr int kProducerWarp = 12, kMmaWarp = 13, kBackWarp = 14;
  constexpr int kConsumerWarps = Cfg::kThreads / 32 - 1;  // every warp but the producer reads the item ring
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if ((smem_u32(smem_raw) & 1023u) != 0u) __trap();  // 128B-swizzle atoms need 1024B alignment
  const uint32_t smem_base = smem_u32(smem_raw);
  uint8_t* smem_gen = smem_raw + (smem_base - smem_u32(smem_raw));

  const uint32_t sKV = smem_base + Cfg::kOffKV;  // buffer b: K at b*2*kKVTile, V at +kKVTile
  const uint32_t sQ = smem_base + Cfg::kOffQ;
  const uint32_t sDO = smem_base + Cfg::kOffDO;
  const uint32_t sDS = smem_base + Cfg::kOffDS;
  const uint32_t sDQ = smem_base + Cfg::kOffDQ;
  // dK / dV output staging: its own region at d = 64, else the dS^T + dQ staging region
  const uint32_t sStage = Cfg::kSepStage ? smem_base + Cfg::kOffStage : sDS;
  const uint32_t sVec = smem_base + Cfg::kOffVec;
  const float* vec_gen = reinterpret_cast<const float*>(smem_gen + Cfg::kOffVec);
  const uint32_t bar0 = smem_base + Cfg::kOffBar;
  auto BAR = [&](int i) { return bar0 + 8u * static_cast<uint32_t>(i); };
  const int kBarQFull = 0;
  const int kBarQEmpty = kBarQFull + S;
  const int kBarSFull = kBarQEmpty + S;     // [2]
  const int kBarPFull = kBarSFull + 2;      // [2]
  const int kBarDQFull = kBarPFull + 2;     // [2]
  const int kBarDQEmpty = kBarDQFull + 2;   // [2]
  const int kBarXFree = kBarDQEmpty + 2;    // [2] d = 64: S^T / dP^T of X_x in registers (count 128)
  const int kBarDSEmpty = kBarXFree + 2;    // [kDSBufs]
  const int kBarKVFull = kBarDSEmpty + Cfg::kDSBufs;  // [NKV]
  const int kBarKVFree = kBarKVFull + NKV;  // [NKV] MMAs of the buffer's item done
  const int kBarFinal = kBarKVFree + NKV;   // item's MMAs done (dK, dV final in TMEM)
  const int kBarAccFree = kBarFinal + 1;    // dK / dV drained from TMEM (count 128)
  // slot kBarStageFree is not an mbarrier but a counter: items whose output staging the TMA
  // store has read (a softmax warpgroup may skip items, so it waits on a count, not a parity)
  const int kBarStageFree = kBarAccFree + 1;
  const int kBarItem = kBarStageFree + 1;   // [kItemRing] item id published
  const int kBarItemFree = kBarItem + kItemRing;  // [kItemRing] slot read by every consumer warp
  const int kNumBars = kBarItemFree + kItemRing;
  static_assert(8 * (2 * S + 10 + Cfg::kDSBufs + 2 * NKV + 3 + 2 * kItemRing) <= 8 * 46, "barrier region");
  volatile int* ring = reinterpret_cast<volatile int*>(smem_gen + Cfg::kOffRing);
  // Dense launches are persistent (one CTA per SM): the producer claims items from a
  // global counter (zeroed by K2) and publishes them; block-sparse launches run exactly
  // one item per CTA (item = blockIdx.x).
  auto take_item = [&](int n) -> int {  // called by whole warps
    mbar_wait(BAR(kBarItem + n % kItemRing), static_cast<uint32_t>((n / kItemRing) & 1));
    const int w = ring[n % kItemRing];
    __syncwarp();
    if (lane_id() == 0) mbar_arrive(BAR(kBarItemFree + n % kItemRing));
    return w;
  };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_gen + Cfg::kOffBar + 8 * 46);

  const int warp = static_cast<int>(warp_id());
  const int lane = static_cast<int>(lane_id());
  uint32_t* mask_smem = reinterpret_cast<uint32_t*>(smem_gen + Cfg::kOffMask);
  if (threadIdx.x == 0) TATN_TRACE_AT(0);
  TATN_EV_INIT();

  if (threadIdx.x == 0) {
    // (the counter slot is never an mbarrier: an mbarrier init is a SYNCS-unit write that is
    // not ordered with a plain store to the same word)
    for (int i = 0; i < kNumBars; ++i)
      if (i != kBarStageFree) mbar_init(BAR(i), 1);
    *reinterpret_cast<volatile uint64_t*>(smem_gen + Cfg::kOffBar + 8 * kBarStageFree) = 0;
    for (int x = 0; x < 2; ++x) {
      mbar_init(BAR(kBarPFull + x), 128);
      mbar_init(BAR(kBarDQEmpty + x), 128);
      mbar_init(BAR(kBarXFree + x), 128);
    }
    mbar_init(BAR(kBarAccFree), 128);
    for (int k = 0; k < kItemRing; ++k) mbar_init(BAR(kBarItemFree + k), kConsumerWarps);
    if (Cfg::kEarlyX)
      for (int k = 0; k < NKV; ++k) mbar_init(BAR(kBarKVFree + k), 2);  // front and back issuers
    fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    tmem_alloc(smem_u32(tmem_slot), 512);
    tmem_relinquish();
  }
  // block-sparse grid column of item w (key tile j) -> bitmask over 64-row Q tiles, read once
  auto build_col_mask = [&](int w, uint32_t* dst) {  // whole producer warp
    int bh0, j0;
    bwd_item(p, w, bh0, j0);
    // strided column of the grid: 128-row blocks -> bits over 64-row Q tiles (each bit doubled)
    warp_nonzero_bits(p.grid + j0, p.tr, p.tc, lane_id(), [&](int wd, uint32_t bits) {
      dst[2 * wd] = spread_bits16(bits);
      dst[2 * wd + 1] = spread_bits16(bits >> 16);
    });
    __syncwarp();
  };
  constexpr bool kSparsePersistent = Cfg::kMaskSlots == kItemRing;
  griddep_wait();  // K2's outputs (workspace, item counter) are visible from here on
  // d = 128 block-sparse launches run one item per CTA (grid = items)
  if (!kSparsePersistent && p.grid != nullptr && warp == kProducerWarp) build_col_mask(static_cast<int>(blockIdx.x), mask_smem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // per-item schedule, identical in every role
  struct Item {
    int bh, b, h, j, cnt;
    BwdSched sc;
  };
  auto item = [&](int w, int n) {
    Item it;
    bwd_item(p, w, it.bh, it.j);
    it.b = it.bh / p.H;
    it.h = it.bh - it.b * p.H;
    it.sc = make_bwd_sched(p, it.b, it.j);
    it.sc.mask = mask_smem + (kSparsePersistent ? (n % kItemRing) * 128 : 0);
    it.cnt = 0;
    if (it.sc.gcol == nullptr) it.cnt = it.sc.i_end - it.sc.i_begin;
    else
      for (int i = it.sc.next(it.sc.i_begin); i < it.sc.i_end; i = it.sc.next(i + 1)) ++it.cnt;
    return it;
  };

  if (warp == kProducerWarp) {
    // ------------------------------------------------------------ TMA producer
    // whole warp runs the loop (waits), one elected lane issues
    if (elect_one_sync()) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmDO);
    }
    __syncwarp();
    int g = 0;  // Q tiles loaded so far (ring position)
    for (int n = 0;; ++n) {
      // claim item n of this CTA and publish it in ring slot n % kItemRing
      if (n >= kItemRing)
        mbar_wait(BAR(kBarItemFree + n % kItemRing), static_cast<uint32_t>((n / kItemRing - 1) & 1));
      int w = -1;
      if (p.grid != nullptr && !kSparsePersistent) {
        w = (n == 0) ? static_cast<int>(blockIdx.x) : -1;
      } else if (lane == 0) {
        w = atomicAdd(p.item_counter, 1);
      }
      w = __shfl_sync(0xffffffffu, w, 0);
      if (w >= p.n_items) w = -1;
      if (w < 0 && TATN_PDL_EARLY) griddep_launch();  // no more items: K4 may take freed SM slots
      if (kSparsePersistent && p.grid != nullptr && w >= 0) build_col_mask(w, mask_smem + (n % kItemRing) * 128);
      if (lane == 0) {
        ring[n % kItemRing] = w;
        mbar_arrive(BAR(kBarItem + n % kItemRing));
      }
      __syncwarp();
      if (w < 0) break;
      if (lane == 0) TATN_EVI(n, 0);  // claimed and published
      const Item it = item(w, n);
      const int kb = n % NKV;
      if (n >= NKV) mbar_wait(BAR(kBarKVFree + kb), static_cast<uint32_t>((n / NKV - 1) & 1));
      if (lane == 0) TATN_EVI(n, 1);  // K / V buffer free: load issued next
      if (elect_one_sync()) {
        const uint32_t sK = sKV + kb * 2 * Cfg::kKVTile, sV = sK + Cfg::kKVTile;
        mbar_expect_tx(BAR(kBarKVFull + kb), 2 * Cfg::kKVTile);
        for (int s = 0; s < Cfg::kSubs; ++s) {
          tma_load_4d(sK + s * 128 * 128, &tmK, BAR(kBarKVFull + kb), s * 64, it.sc.k0, it.h, it.b);
          tma_load_4d(sV + s * 128 * 128, &tmV, BAR(kBarKVFull + kb), s * 64, it.sc.k0, it.h, it.b);
        }
      }
      __syncwarp();
      for (int i = it.sc.next(it.sc.i_begin); i < it.sc.i_end; i = it.sc.next(i + 1), ++g) {
        const int stage = g % S;
        mbar_wait(BAR(kBarQEmpty + stage), static_cast<uint32_t>(((g / S) & 1) ^ 1));
        if (elect_one_sync()) {
          const uint32_t fb = BAR(kBarQFull + stage);
          mbar_expect_tx(fb, 2 * Cfg::kQTile + Cfg::kVecBytes);
          for (int s = 0; s < Cfg::kSubs; ++s) {
            tma_load_4d(sQ + stage * Cfg::kQTile + s * Cfg::kQSub, &tmQ, fb, s * 64, i * kBwdQT, it.h, it.b);
            tma_load_4d(sDO + stage * Cfg::kQTile + s * Cfg::kQSub, &tmDO, fb, s * 64, i * kBwdQT, it.h, it.b);
          }
          const float* src = lse2 + static_cast<size_t>(it.bh) * Nq_pad + i * kBwdQT;
          const uint32_t vdst = sVec + stage * Cfg::kVecBytes;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           vdst),
                       "l"(src), "r"(kBwdQT * 4), "r"(fb)
                       : "memory");
          const float* srcd = p.delta + static_cast<size_t>(it.bh) * Nq_pad + i * kBwdQT;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           vdst + kBwdQT * 4),
                       "l"(srcd), "r"(kBwdQT * 4), "r"(fb)
                       : "memory");
        }
        __syncwarp();
      }
    }
  } else if (!Cfg::kEarlyX && warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer, d = 128
    // whole warp runs the schedule (waits); one elected lane issues tcgen05.mma/commit (d = 64
    // runs the single-lane two-issuer schedule below)
    constexpr uint32_t ab = BF16 ? 1u : 0u;
    constexpr uint32_t idesc_s = make_idesc_f16(ab, 128, kBwdQT, 0, 0);   // S^T, dP^T
    constexpr uint32_t idesc_acc = make_idesc_f16(ab, 128, D, 0, 1);      // dV, dK (B MN-major)
    // dQ^T (A, B MN-major): M = d; at d = 64 an M = 64 MMA (half the A bytes of M = 128)
    constexpr uint32_t idesc_dq = make_idesc_f16(ab, Cfg::kDQ64 ? 64 : 128, kBwdQT, 1, 1);
    // base descriptors; per-MMA operands add (byte offset >> 4) to the start-address field
    const uint64_t dKV0 = make_sdesc_sw128(sKV, 16, 1024);               // K / V as K-major A
    const uint64_t dQk0 = make_sdesc_sw128(sQ, 16, 1024);                // Q as K-major B
    const uint64_t dDOk0 = make_sdesc_sw128(sDO, 16, 1024);              // dO as K-major B
    const uint64_t dQmn0 = make_sdesc_sw128(sQ, Cfg::kQSub, 1024);       // Q as MN-major B
    const uint64_t dDOmn0 = make_sdesc_sw128(sDO, Cfg::kQSub, 1024);     // dO as MN-major B
    const uint64_t dKmn0 = make_sdesc_sw128(sKV, 128 * 128, 1024);       // K^T as MN-major A
    const uint64_t dDS0 = make_sdesc_sw128(sDS, 128 * 128, 1024);        // dS^T as MN-major B
    int g0 = 0;  // Q tiles issued before the current item
    int w_next = take_item(0);
    for (int n = 0; w_next >= 0; ++n) {
      const int w = w_next;
      const int cnt = item(w, n).cnt;
      const int kb = n % NKV;
      const uint32_t koff = static_cast<uint32_t>(kb * 2 * Cfg::kKVTile);  // K of buffer kb
      const uint32_t voff = koff + Cfg::kKVTile;
      if (lane == 0) TATN_EVI(n, 2);  // MMA warp starts the item (item taken)
      mbar_wait(BAR(kBarKVFull + kb), static_cast<uint32_t>((n / NKV) & 1));
      if (lane == 0) TATN_EVI(n, 3);  // K / V landed
      tc_fence_after();
      if (lane == 0 && n == 0) TATN_TRACE_AT(1);
#ifdef TATN_TRACE
      if (lane == 0 && n == 0 && g_tatn_trace) g_tatn_trace[static_cast<size_t>(blockIdx.x) * 16 + 6] = cnt;
#endif
      auto front_dp = [&](int g, uint32_t voff) {  // dP^T = V dO^T  -> X cols [64,128)
        const int s = g % S;
        const int x = g & 1;
        mbar_wait(BAR(kBarQFull + s), static_cast<uint32_t>((g / S) & 1));
        tc_fence_after();
        if (elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t offa = voff + (kk >> 2) * (128 * 128) + (kk & 3) * 32;
            const uint32_t offb = (kk >> 2) * Cfg::kQSub + (kk & 3) * 32;
            mma_ss(tmem_base + Cfg::kTmemX + x * 128 + 64, dKV0 + (offa >> 4),
                   dDOk0 + ((s * Cfg::kQTile + offb) >> 4), idesc_s, kk > 0 ? 1u : 0u);
          }
        }
        __syncwarp();
      };
      auto front_s = [&](int g, uint32_t koff) {  // S^T = K Q^T  -> X cols [0,64)
        const int s = g % S;
        const int x = g & 1;
        if (elect_one_sync()) {
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t offa = koff + (kk >> 2) * (128 * 128) + (kk & 3) * 32;
            const uint32_t offb = (kk >> 2) * Cfg::kQSub + (kk & 3) * 32;
            mma_ss(tmem_base + Cfg::kTmemX + x * 128, dKV0 + (offa >> 4), dQk0 + ((s * Cfg::kQTile + offb) >> 4),
                   idesc_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(BAR(kBarSFull + x));
        }
        __syncwarp();
        if (lane == 0) TATN_EV(g, 3);
      };
      auto wait_dq_drained = [&](int g) {  // dQ^T of Q tile g read out of its TMEM buffer
        mbar_wait(BAR(kBarDQEmpty + (g & 1)), static_cast<uint32_t>((g >> 1) & 1));
        tc_fence_after();
      };
      for (int i = 0; i < cnt && i < 2; ++i) {
        const int g = g0 + i;
        front_dp(g, voff);
        if (g >= 2) wait_dq_drained(g - 2);  // X_x still holds dQ^T(g - 2)
        front_s(g, koff);
      }
      if (n > 0) {  // previous dK / dV drained (every item, empty ones included: see the d = 64 issuer)
        mbar_wait(BAR(kBarAccFree), static_cast<uint32_t>((n - 1) & 1));
        tc_fence_after();
      }
      for (int i = 0; i < cnt; ++i) {
        const int g = g0 + i;
        const int x = g & 1;
        const int s = g % S;
        mbar_wait(BAR(kBarPFull + x), static_cast<uint32_t>((g >> 1) & 1));
        tc_fence_after();
        if (lane == 0) TATN_EV(g, 2);
        if (lane == 0 && i == 2 && n == 0) TATN_TRACE_AT(11);
        const uint32_t accf = i > 0 ? 1u : 0u;
        if (elect_one_sync()) {
          // dV += P^T dO   (P^T 16-bit in X_x cols [0,32); dO MN-major, 16 queries per step)
#pragma unroll
          for (int kk = 0; kk < kBwdQT / 16; ++kk)
            mma_ts(tmem_base + Cfg::kTmemDV, tmem_base + Cfg::kTmemX + x * 128 + kk * 8,
                   dDOmn0 + ((s * Cfg::kQTile + kk * 2048) >> 4), idesc_acc, accf | (kk > 0 ? 1u : 0u));
          // dK += dS^T Q   (dS^T 16-bit in X_x cols [64,96))
#pragma unroll
          for (int kk = 0; kk < kBwdQT / 16; ++kk)
            mma_ts(tmem_base + Cfg::kTmemDK, tmem_base + Cfg::kTmemX + x * 128 + 64 + kk * 8,
                   dQmn0 + ((s * Cfg::kQTile + kk * 2048) >> 4), idesc_acc, accf | (kk > 0 ? 1u : 0u));
        }
        __syncwarp();
        auto issue_dq = [&]() {
          // dQ^T = K^T dS^T  (K MN-major as A; dS^T MN-major as B; 16 keys per step)
          const uint32_t tDQ = tmem_base + Cfg::kTmemX + x * 128;
          if (elect_one_sync()) {
#pragma unroll
            for (int kk = 0; kk < kBwdKT / 16; ++kk)
              mma_ss(tDQ, dKmn0 + ((koff + kk * 2048) >> 4), dDS0 + (((g % Cfg::kDSBufs) * Cfg::kDSBytes + kk * 2048) >> 4), idesc_dq,
                     kk > 0 ? 1u : 0u);
            mma_commit(BAR(kBarDQFull + x));
            mma_commit(BAR(kBarQEmpty + s));
            mma_commit(BAR(kBarDSEmpty + g % Cfg::kDSBufs));
          }
          __syncwarp();
          if (lane == 0) TATN_EV(g, 4);
        };
        issue_dq();  // dQ^T lands in X_x cols [0,64): the next front waits for the dQ warpgroup
        if (i + 2 < cnt) {
          front_dp(g + 2, voff);
          wait_dq_drained(g);
          front_s(g + 2, koff);
        }
      }
      if (elect_one_sync()) {
        mma_commit(BAR(kBarFinal));
        mma_commit(BAR(kBarKVFree + kb));
      }
      __syncwarp();
      w_next = take_item(n + 1);
      g0 += cnt;
    }
  } else if (Cfg::kEarlyX && (warp == kMmaWarp || warp == kBackWarp)) {
    // ------------------------------------------------------------ MMA issuers
    // One elected lane runs a whole schedule (waits, tcgen05.mma, commits). Inside a single
    // elect region ptxas knows one lane is active and issues each MMA group straight from
    // uniform registers; with the warp running the loop and electing a lane per group it
    // wrapped every tcgen05.mma in an elect / vote loop (scripts/micro/mma_issue.cu: the d = 64
    // Q-tile stream 1600-1800 -> 1050 cycles). At d = 64 the fronts (S^T, dP^T into X_x) and the
    // backs (dV, dK, dQ^T: PdS_x, accumulators) touch disjoint TMEM, so two warps issue them:
    // warp 13 the fronts, warp 14 the backs, and neither waits behind the other's barrier waits
    // and descriptor set-up (the issuing lane, not the tensor pipe, set the pace with one warp).
    // Each warp's tcgen05.commit tracks its own MMAs; the K/V buffer is free once both have
    // committed (kBarKVFree counts 2).
    constexpr uint32_t ab = BF16 ? 1u : 0u;
    constexpr uint32_t idesc_s = make_idesc_f16(ab, 128, kBwdQT, 0, 0);   // S^T, dP^T
    constexpr uint32_t idesc_acc = make_idesc_f16(ab, 128, D, 0, 1);      // dV, dK (B MN-major)
    // dQ^T (A, B MN-major): M = d; at d = 64 an M = 64 MMA (half the A bytes of M = 128)
    constexpr uint32_t idesc_dq = make_idesc_f16(ab, Cfg::kDQ64 ? 64 : 128, kBwdQT, 1, 1);
    // base descriptors; per-MMA operands add (byte offset >> 4) to the start-address field
    const uint64_t dKV0 = make_sdesc_sw128(sKV, 16, 1024);               // K / V as K-major A
    const uint64_t dQk0 = make_sdesc_sw128(sQ, 16, 1024);                // Q as K-major B
    const uint64_t dDOk0 = make_sdesc_sw128(sDO, 16, 1024);              // dO as K-major B
    const uint64_t dQmn0 = make_sdesc_sw128(sQ, Cfg::kQSub, 1024);       // Q as MN-major B
    const uint64_t dDOmn0 = make_sdesc_sw128(sDO, Cfg::kQSub, 1024);     // dO as MN-major B
    const uint64_t dKmn0 = make_sdesc_sw128(sKV, 128 * 128, 1024);       // K^T as MN-major A
    const uint64_t dDS0 = make_sdesc_sw128(sDS, 128 * 128, 1024);        // dS^T as MN-major B
    const bool fronts = warp == kMmaWarp;                                // else the backs
    if (elect_one_sync()) {
      // take_item for a single lane: the ring slot's consumer arrival is this warp's one arrival
      auto take_item_1 = [&](int n) -> int {
        mbar_wait(BAR(kBarItem + n % kItemRing), static_cast<uint32_t>((n / kItemRing) & 1));
        const int w = ring[n % kItemRing];
        mbar_arrive(BAR(kBarItemFree + n % kItemRing));
        return w;
      };
      auto front_dp = [&](int g, uint32_t voff) {  // dP^T = V dO^T  -> X cols [64,128)
        const int s = g % S;
        const int x = g & 1;
        mbar_wait(BAR(kBarQFull + s), static_cast<uint32_t>((g / S) & 1));
        tc_fence_after();
        TATN_EV2(g, 2);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t offa = voff + (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          const uint32_t offb = (kk >> 2) * Cfg::kQSub + (kk & 3) * 32;
          mma_ss(tmem_base + Cfg::kTmemX + x * 128 + 64, dKV0 + (offa >> 4), dDOk0 + ((s * Cfg::kQTile + offb) >> 4),
                 idesc_s, kk > 0 ? 1u : 0u);
        }
      };
      auto front_s = [&](int g, uint32_t koff) {  // S^T = K Q^T  -> X cols [0,64)
        const int s = g % S;
        const int x = g & 1;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t offa = koff + (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          const uint32_t offb = (kk >> 2) * Cfg::kQSub + (kk & 3) * 32;
          mma_ss(tmem_base + Cfg::kTmemX + x * 128, dKV0 + (offa >> 4), dQk0 + ((s * Cfg::kQTile + offb) >> 4), idesc_s,
                 kk > 0 ? 1u : 0u);
        }
        mma_commit(BAR(kBarSFull + x));
        TATN_EV(g, 3);
      };
      // back(g): dV += P^T dO, dK += dS^T Q (A from TMEM), then dQ^T = K^T dS^T
      // The previous item's dK / dV drained out of TMEM (once per item, empty items included: each
      // AccFree phase is waited on in turn, so the Final commits below can never run two phases
      // ahead of the dQ warpgroup that waits on them — with the issuers racing through empty
      // items that aliased a parity and left the last epilogue waiting forever)
      auto wait_acc_free = [&](int n) {
        if (n > 0) {
          mbar_wait(BAR(kBarAccFree), static_cast<uint32_t>((n - 1) & 1));
          tc_fence_after();
        }
      };
      auto back = [&](int g, int i, int n, uint32_t koff) {
        const int x = g & 1;
        const int s = g % S;
        mbar_wait(BAR(kBarPFull + x), static_cast<uint32_t>((g >> 1) & 1));
        tc_fence_after();
        TATN_EV(g, 2);
        if (i == 2 && n == 0) TATN_TRACE_AT(11);
        const uint32_t accf = i > 0 ? 1u : 0u;
        // P^T, dS^T (16-bit): PdS_x cols [0,32) / [32,64)
        const uint32_t tP = tmem_base + Cfg::kTmemPdS + x * 64;
        const uint32_t tDS = tP + 32;
#pragma unroll
        for (int kk = 0; kk < kBwdQT / 16; ++kk)  // dV += P^T dO   (dO MN-major, 16 queries per step)
          mma_ts(tmem_base + Cfg::kTmemDV, tP + kk * 8, dDOmn0 + ((s * Cfg::kQTile + kk * 2048) >> 4), idesc_acc,
                 accf | (kk > 0 ? 1u : 0u));
#pragma unroll
        for (int kk = 0; kk < kBwdQT / 16; ++kk)  // dK += dS^T Q
          mma_ts(tmem_base + Cfg::kTmemDK, tDS + kk * 8, dQmn0 + ((s * Cfg::kQTile + kk * 2048) >> 4), idesc_acc,
                 accf | (kk > 0 ? 1u : 0u));
        // Q_i / dO_i are done with (front(g) completed before S^T reached the softmax; the tile's
        // lse2 / D were read by the softmax before PFull)
        mma_commit(BAR(kBarQEmpty + s));
        TATN_EV2(g, 5);
        // dQ^T into PdS_x (after dV / dK have read it: in-order pipe)
#pragma unroll
        for (int kk = 0; kk < kBwdKT / 16; ++kk)
          mma_ss(tP, dKmn0 + ((koff + kk * 2048) >> 4), dDS0 + (((g % Cfg::kDSBufs) * Cfg::kDSBytes + kk * 2048) >> 4), idesc_dq,
                 kk > 0 ? 1u : 0u);
        mma_commit(BAR(kBarDQFull + x));
        mma_commit(BAR(kBarDSEmpty + g % Cfg::kDSBufs));
        TATN_EV(g, 4);
      };
      int g0 = 0;  // Q tiles issued before the current item
      int w_next = take_item_1(0);
      for (int n = 0; w_next >= 0; ++n) {
        const int w = w_next;
        const int cnt = item(w, n).cnt;
        const int kb = n % NKV;
        const uint32_t koff = static_cast<uint32_t>(kb * 2 * Cfg::kKVTile);  // K of buffer kb
        const uint32_t voff = koff + Cfg::kKVTile;
        if (fronts) TATN_EVI(n, 2);  // MMA warp starts the item (item taken)
        mbar_wait(BAR(kBarKVFull + kb), static_cast<uint32_t>((n / NKV) & 1));
        if (fronts) TATN_EVI(n, 3);  // K / V landed
        tc_fence_after();
        if (fronts && n == 0) TATN_TRACE_AT(1);
#ifdef TATN_TRACE
        if (fronts && n == 0 && g_tatn_trace) g_tatn_trace[static_cast<size_t>(blockIdx.x) * 16 + 6] = cnt;
#endif
        if (fronts) {
          // front(g) as soon as the softmax holds S^T / dP^T of tile g - 2 (same X buffer) in registers
          for (int i = 0; i < cnt; ++i) {
            const int g = g0 + i;
            TATN_EV2(g, 0);
            if (g >= 2) {
              mbar_wait(BAR(kBarXFree + (g & 1)), static_cast<uint32_t>(((g >> 1) & 1) ^ 1));
              tc_fence_after();
            }
            TATN_EV2(g, 1);
            front_dp(g, voff);
            front_s(g, koff);
          }
        } else {
          wait_acc_free(n);
          for (int i = 0; i < cnt; ++i) back(g0 + i, i, n, koff);
          mma_commit(BAR(kBarFinal));
        }
        mma_commit(BAR(kBarKVFree + kb));  // one of two arrivals
        w_next = take_item_1(n + 1);
        g0 += cnt;
      }
    }
    __syncwarp();
  } else if (warp < 8) {
    // ------------------------------------------------------------ softmax warpgroups
    // warpgroup sg takes the Q tiles of parity sg (ping-pong over the two X buffers)
    const int sg = warp >> 2;
    const int r = (warp & 3) * 32 + lane;   // key row within tile == TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2_pack(sl2, sl2);
    const bool causal = p.mask_kind == kMaskCausal;
    uint64_t* drop_rows = reinterpret_cast<uint64_t*>(smem_gen + Cfg::kOffDrop + sg * 512);
    int g0 = 0;
    for (int n = 0;; ++n) {
      const int w = take_item(n);
      if (w < 0) break;
      const Item it = item(w, n);
      const BwdSched& sc = it.sc;
      const int kj = sc.k0 + r;
      bool first = true;  // first dS^T store of this warpgroup in this item
      int g = g0;
      for (int i = sc.next(sc.i_begin); i < sc.i_end; i = sc.next(i + 1), ++g) {
        if ((g & 1) != sg) continue;
        const int s = g % S;
        const int x = g & 1;  // X buffer (== sg)
        const uint32_t tX = tmem_base + lane_off + Cfg::kTmemX + x * 128;
        // P^T, dS^T (16-bit): PdS_x cols [0,32) / [32,64) at d = 64, else over S^T / dP^T in X_x
        const uint32_t tP = Cfg::kEarlyX ? tmem_base + lane_off + Cfg::kTmemPdS + x * 64 : tX;
        const uint32_t tDS = tP + (Cfg::kEarlyX ? 32 : 64);
        if (p.visited != nullptr && r == 0) {
          const long long bit = static_cast<long long>(i >> 1) * p.tc + it.j;
          atomicOr(p.visited + (bit >> 5), 1u << (bit & 31));
        }
        mbar_wait(BAR(kBarQFull + s), static_cast<uint32_t>((g / S) & 1));  // lse2 / D vectors landed
        if (r == 0) TATN_EV(g, 7);
        mbar_wait(BAR(kBarSFull + x), static_cast<uint32_t>((g >> 1) & 1));
        tc_fence_after();
        if (r == 0) TATN_EV(g, 0);
        if (r == 0 && g == 0) TATN_TRACE_AT(2);
        if (r == 0 && g == 2) TATN_TRACE_AT(9);
        const uint64_t* nl2 = reinterpret_cast<const uint64_t*>(vec_gen + s * (Cfg::kVecBytes / 4));  // -lse2 pairs
        const uint64_t* nD = nl2 + kBwdQT / 2;                                                          // -D pairs
        const int i0 = i * kBwdQT;
        if constexpr (DROP) {
          // the tile's 64 query-row hashes (thread r < 64 computes row i0 + r)
          named_bar_sync(3 + sg, 128);  // previous tile's hashes fully consumed
          if (r < kBwdQT) drop_rows[r] = drop_row_hash(p.drop_seed + static_cast<uint64_t>(it.bh), i0 + r);
          named_bar_sync(3 + sg, 128);
        }
        const bool custom_on = p.custom_t != nullptr;
        const bool need_mask =
            (sc.k0 + kBwdKT > sc.kv_limit) || (causal && p.k_off + sc.k0 + kBwdKT - 1 > i0) || custom_on;
        // masked keys: kj >= kv_limit for every query; causal: k_off + kj > i0 + c  <=>  c < k_off + kj - i0
        const int c_lo = (kj >= sc.kv_limit) ? kBwdQT : (causal ? p.k_off + kj - i0 : 0);  // first visible query
        // Custom mask: keep bits of this key row for the tile's 64 queries (K2b's transpose)
        uint2 cbits = make_uint2(~0u, ~0u);
        if (custom_on) {
          cbits = make_uint2(0u, 0u);
          if (kj < p.Nk)
            cbits = *reinterpret_cast<const uint2*>(
                p.custom_t + (static_cast<size_t>(p.custom_t_b ? it.b : 0) * p.Nk + kj) * p.custom_t_words + i * 2);
        }
        uint32_t sr[32], dp[32];
        tmem_ld32_async(tX, sr);
        tmem_ld32_async(tX + 64, dp);
        tmem_ld_wait32(sr);
        tmem_ld_wait32(dp);
        if (D == 64 && r == 0) TATN_EV(g, 6);
        const int xs = g % Cfg::kDSBufs;  // dS^T buffer
        const uint32_t drow = sDS + xs * Cfg::kDSBytes + r * 128;
        auto body = [&](auto masked_t) {
          constexpr bool kMasked = decltype(masked_t)::value;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            // queries [32*half, 32*half + 32); half 1 is loaded while half 0's results are stored
            uint32_t pk[16], dk[16];
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2) {
              const int c4 = half * 32 + 4 * k2;  // four query columns c4 .. c4 + 3
              const ulonglong2 l4 = *reinterpret_cast<const ulonglong2*>(nl2 + (c4 >> 1));
              const ulonglong2 d4 = *reinterpret_cast<const ulonglong2*>(nD + (c4 >> 1));
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int k = 2 * k2 + e;
                const int c = c4 + 2 * e;
                const uint64_t xv = f2_fma(f2_pack(__uint_as_float(sr[2 * k]), __uint_as_float(sr[2 * k + 1])), sl2x2,
                                           e ? l4.y : l4.x);
                float p0, p1;
                f2_unpack(xv, p0, p1);
                p0 = ex2_approx(p0);
                p1 = ex2_approx(p1);
                if constexpr (kMasked) {
                  const uint32_t cwv = (c < 32) ? cbits.x : cbits.y;
                  p0 = (c < c_lo || ((cwv >> (c & 31)) & 1u) == 0u) ? 0.f : p0;
                  p1 = (c + 1 < c_lo || ((cwv >> ((c + 1) & 31)) & 1u) == 0u) ? 0.f : p1;
                }
                const uint64_t nd = e ? d4.y : d4.x;
                if constexpr (DROP) {  // dP through the mask, dV from P * Z / (1 - p) (reference.cpp:118-141)
                  float d0, d1;
                  f2_unpack(nd, d0, d1);
                  const float z0 = drop_keep(drop_rows[c], p.k_off + kj, p.drop_thresh) ? p.drop_scale : 0.f;
                  const float z1 = drop_keep(drop_rows[c + 1], p.k_off + kj, p.drop_thresh) ? p.drop_scale : 0.f;
                  dk[k] = pack2<BF16>(p0 * fmaf(__uint_as_float(dp[2 * k]), z0, d0),
                                      p1 * fmaf(__uint_as_float(dp[2 * k + 1]), z1, d1));
                  pk[k] = pack2<BF16>(p0 * z0, p1 * z1);
                } else {
                  const uint64_t ds = f2_mul(
                      f2_pack(p0, p1), f2_add(f2_pack(__uint_as_float(dp[2 * k]), __uint_as_float(dp[2 * k + 1])), nd));
                  float d0, d1;
                  f2_unpack(ds, d0, d1);
                  pk[k] = pack2<BF16>(p0, p1);
                  dk[k] = pack2<BF16>(d0, d1);
                }
              }
            }
            if (r == 0) TATN_EV2(g, half == 0 ? 3 : 6);  // half computed
            if (half == 0) {
              tmem_ld32_async(tX + 32, sr);
              tmem_ld32_async(tX + 96, dp);
              if constexpr (Cfg::kEarlyX) {
                // all of S^T / dP^T in registers: X_x may take the front of tile g + 2
                tmem_ld_wait32(sr);
                tmem_ld_wait32(dp);
                tc_fence_before();
                mbar_arrive(BAR(kBarXFree + x));
                if (r == 0) TATN_EV2(g, 7);
                // PdS_x: dQ^T(g - 2) read out by the dQ warpgroup
                mbar_wait(BAR(kBarDQEmpty + x), static_cast<uint32_t>(((g >> 1) & 1) ^ 1));
                tc_fence_after();
                if (r == 0) TATN_EV2(g, 4);
              }
            }
            tmem_st16(tP + half * 16, pk);   // P^T
            tmem_st16(tDS + half * 16, dk);  // dS^T
            if (half == 0) {
              // the dQ^T MMA of tile g - 2 must have released the dS^T buffer, and in a new
              // item the previous item's dK / dV staging must have been stored
              mbar_wait(BAR(kBarDSEmpty + xs), static_cast<uint32_t>(((g / Cfg::kDSBufs) & 1) ^ 1));
              if (!Cfg::kSepStage && first) wait_counter_ge(BAR(kBarStageFree), static_cast<uint32_t>(n));
              first = false;
            }
            // dS^T -> smem [key][64 queries], 128B swizzle (B operand of dQ^T, MN-major)
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              const int chunk = half * 4 + cc;
              st_shared_v4(drow + ((chunk ^ (r & 7)) << 4), dk[4 * cc], dk[4 * cc + 1], dk[4 * cc + 2], dk[4 * cc + 3]);
            }
            if (!Cfg::kEarlyX && half == 0) {
              tmem_ld_wait32(sr);
              tmem_ld_wait32(dp);
            }
          }
        };
        if (need_mask) body(std::true_type{});
        else body(std::false_type{});
        fence_proxy_async_smem();
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(BAR(kBarPFull + x));
        if (r == 0) TATN_EV(g, 1);
        if (r == 0 && g == 2) TATN_TRACE_AT(10);
      }
      g0 += it.cnt;
    }
    if (r == 0 && sg == 0) TATN_TRACE_AT(3);
  } else {
    // ------------------------------------------------------------ dQ warpgroup (warps 8-11)
    // per Q tile: dQ^T out of TMEM -> fp32 staging -> bulk reduce-add into the workspace;
    // per item: dK / dV out of TMEM -> 16-bit staging -> TMA store (the softmax warpgroups
    // meanwhile start the next item)
    const int wq = warp & 3;
    const int row = wq * 32 + lane;  // TMEM lane: key row of dK / dV
    // head-dim index of dQ^T held by this thread's TMEM lane
    const int dd = Cfg::kDQ64 ? wq * 16 + lane : row;
    const bool active = Cfg::kDQ64 ? lane < 16 : row < D;
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
    const float tau = p.tau;
    const bool leader = warp == 8 && lane == 0;
    int g = 0;
    for (int n = 0;; ++n) {
      const int w = take_item(n);
      if (w < 0) break;
      const Item it = item(w, n);
      for (int i = it.sc.next(it.sc.i_begin); i < it.sc.i_end; i = it.sc.next(i + 1), ++g) {
        const int x = g & 1;
        mbar_wait(BAR(kBarDQFull + x), static_cast<uint32_t>((g >> 1) & 1));
        tc_fence_after();
        if (row == 0) TATN_EV(g, 5);
        if (row == 0 && g == 2) TATN_TRACE_AT(12);
        uint32_t v[64];
        if (Cfg::kDQ64 || active) {  // warp-uniform: tcgen05.ld is .sync.aligned
          const uint32_t tX = tmem_base + lane_off + (Cfg::kEarlyX ? Cfg::kTmemPdS + x * 64 : Cfg::kTmemX + x * 128);
          tmem_ld32(tX, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
          tmem_ld32(tX + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        }
        tc_fence_before();
        mbar_arrive(BAR(kBarDQEmpty + x));
        // staging buffer free once the previous bulk reduce has read it
        if constexpr (Cfg::kDQRed) {
        // fire-and-forget fp32 reductions straight from registers into the L2-resident
        // accumulator: lanes hold consecutive head-dim columns, so each instruction is one
        // coalesced 64-byte reduction, and no shared-memory bandwidth is spent on dQ
        if (active) {
          if (p.dq_part != nullptr) {  // deterministic: this key tile's own slot, plain stores (K4 sums in j order)
            float* dst = p.dq_part + ((static_cast<size_t>(it.j) * p.B * p.H + it.bh) * Nq_pad +
                                      static_cast<size_t>(i) * kBwdQT) * D + dd;
#pragma unroll
            for (int c = 0; c < 64; ++c) dst[c * D] = __uint_as_float(v[c]) * tau;
          } else {
            float* dst = p.dq_acc + (static_cast<size_t>(it.bh) * Nq_pad + static_cast<size_t>(i) * kBwdQT) * D + dd;
#pragma unroll
            for (int c = 0; c < 64; ++c) atomicAdd(dst + c * D, __uint_as_float(v[c]) * tau);
          }
        }
        continue;
        }
        if (leader) bulk_wait_read_all();
        named_bar_sync(2, 128);
        if (active) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(sDQ + (c * D + dd) * 4), "f"(__uint_as_float(v[c]) * tau)
                         : "memory");
        }
        fence_proxy_async_smem();
        named_bar_sync(2, 128);
        if (leader) {
          if (p.dq_part != nullptr) {  // deterministic: bulk store into this key tile's own slot
            float* dst = p.dq_part + ((static_cast<size_t>(it.j) * p.B * p.H + it.bh) * Nq_pad +
                                      static_cast<size_t>(i) * kBwdQT) * D;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sDQ),
                         "r"(Cfg::kDQBytes)
                         : "memory");
          } else {
            float* dst = p.dq_acc + (static_cast<size_t>(it.bh) * Nq_pad + static_cast<size_t>(i) * kBwdQT) * D;
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                         "r"(sDQ), "r"(Cfg::kDQBytes)
                         : "memory");
          }
          bulk_commit();
          TATN_EV(g, 6);
          if (g == 2) TATN_TRACE_AT(13);
        }
      }
      // ---------------- item epilogue: dK = tau * acc_K, dV = acc_V
      mbar_wait(BAR(kBarFinal), static_cast<uint32_t>(n & 1));
      tc_fence_after();
      if (row == 0 && n == 0) TATN_TRACE_AT(4);
      const int kj = it.sc.k0 + row;
      if (leader) bulk_wait_read_all();  // the last dQ reduce has read the staging region
      named_bar_sync(2, 128);
#pragma unroll 1
      for (int which = 0; which < 2; ++which) {
        const uint32_t tacc = tmem_base + lane_off + (which == 0 ? Cfg::kTmemDK : Cfg::kTmemDV);
        const float oscale = which == 0 ? tau : 1.f;
        const uint32_t stg = sStage + which * (128 * D * 2);
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t v[32];
          if (it.cnt > 0) {
            tmem_ld32(tacc + c * 32, v);
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = 0u;
          }
          if constexpr (OUT_F32) {
            float* gp = which == 0 ? p.dk_f32 + static_cast<size_t>(it.b) * p.k_sb + static_cast<size_t>(it.h) * p.k_sh +
                                         static_cast<size_t>(kj) * p.k_sn
                                   : p.dv_f32 + static_cast<size_t>(it.b) * p.v_sb + static_cast<size_t>(it.h) * p.v_sh +
                                         static_cast<size_t>(kj) * p.v_sn;
            if (kj < p.Nk) {
#pragma unroll
              for (int e = 0; e < 8; ++e)
                reinterpret_cast<float4*>(gp + c * 32)[e] =
                    make_float4(__uint_as_float(v[4 * e]) * oscale, __uint_as_float(v[4 * e + 1]) * oscale,
                                __uint_as_float(v[4 * e + 2]) * oscale, __uint_as_float(v[4 * e + 3]) * oscale);
            }
          } else {
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              pk[e] = pack2<BF16>(__uint_as_float(v[2 * e]) * oscale, __uint_as_float(v[2 * e + 1]) * oscale);
            const int sub = (c * 32) / 64;
            const int chunk0 = ((c * 32) % 64) / 8;
            const uint32_t rb = stg + sub * 128 * 128 + row * 128;
#pragma unroll
            for (int e = 0; e < 4; ++e)
              st_shared_v4(rb + (((chunk0 + e) ^ (row & 7)) << 4), pk[4 * e], pk[4 * e + 1], pk[4 * e + 2],
                           pk[4 * e + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(BAR(kBarAccFree));  // TMEM accumulators may be overwritten by the next item
      if constexpr (!OUT_F32) {
        fence_proxy_async_smem();
        named_bar_sync(2, 128);
        if (leader) {
          for (int s = 0; s < Cfg::kSubs; ++s) {
            tma_store_4d(&tmDK, sStage + s * 128 * 128, s * 64, it.sc.k0, it.h, it.b);
            tma_store_4d(&tmDV, sStage + 128 * D * 2 + s * 128 * 128, s * 64, it.sc.k0, it.h, it.b);
          }
          bulk_commit();
          bulk_wait_read_all();
        }
      }
      if (leader) st_release_u32(BAR(kBarStageFree), static_cast<uint32_t>(n + 1));
    }
    if (leader) bulk_wait_all();
    if (leader) TATN_TRACE_AT(8);
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
  }
  if (warp == kMmaWarp) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace tatn_dev

// ---------------------------------------------------------------- host launcher
namespace tatn_host {
// dropout threshold of the reference's test u >= p with u = (h >> 11) * 2^-53:
// keep iff h >= ceil(p * 2^53) << 11 (exact: p * 2^53 is exact in binary64)
inline void set_dropout(const tatn_attn_desc& d, uint64_t* seed, uint64_t* thresh, float* scale) {
  *seed = d.seed;
  const double t = std::ceil(d.p_drop * 9007199254740992.0);  // 2^53
  *thresh = static_cast<uint64_t>(t) << 11;
  *scale = d.p_drop > 0.0 ? static_cast<float>(1.0 / (1.0 - d.p_drop)) : 1.f;
}
cudaEvent_t profile_begin(int which, cudaStream_t s);
int schedule_group(int heads, int tiles_per_head, double l2_bytes_per_head, int ctas_per_sm);
constexpr int kMaxDevices = 64;
int sm_count();
cudaError_t ensure_smem_attr(const void* kern, int bytes);
bool make_map_4d_ext(CUtensorMap* map, int dtype, const void* base, int d, int n, int H, int B, const int64_t str[3],
                     int box_rows, bool mn_major = false);
// deterministic dQ: the per-key-tile partial slots, the last region of the backward workspace
inline float* dq_part_ptr(const tatn_attn_desc& d, void* ws) {
  const size_t rows = static_cast<size_t>(d.B) * d.H * ((d.Nq + 127) / 128 * 128);
  size_t off = rows * d.d * sizeof(float) + 2 * rows * sizeof(float) + 16;
  if (d.mask_kind == TATN_MASK_CUSTOM) {
    const size_t nb = d.custom_bstride != 0 ? static_cast<size_t>(d.B) : 1;
    off += nb * static_cast<size_t>(d.Nk) * ((d.Nq + 127) / 128 * 4) * sizeof(uint32_t);
  }
  return reinterpret_cast<float*>(static_cast<char*>(ws) + off);
}
template <int D, bool BF16, bool OUT_F32>
cudaError_t launch_post_det(const tatn_attn_desc& d, const float* dq_part, void* dq, int Nq_pad, int qt,
                            cudaStream_t stream) {
  const dim3 blocks(static_cast<unsigned>((d.Nq + 256 / (D / 8) - 1) / (256 / (D / 8))), d.H, d.B);
  return launch(tatn_dev::tatn_bwd_post_det<D, BF16, OUT_F32>, blocks, dim3(256), 0, stream, dq_part, dq, d.q_str[0],
                d.q_str[1], d.q_str[2], d.B, d.H, d.Nq, Nq_pad, (d.Nk + 127) / 128, qt,
                d.mask_kind == TATN_MASK_CAUSAL ? 1 : 0, d.k_offset,
                d.mask_kind == TATN_MASK_KEY_PADDING ? d.valid_len : nullptr, d.block_grid);
}
}

template <int D, bool BF16, bool OUT_F32, bool DROP>
static cudaError_t tatn_bwd_launch_t(const tatn_attn_desc& d, const void* q, const void* k, const void* v,
                                     const void* o, const void* dO, const float* lse, void* dq, void* dk, void* dv,
                                     void* ws, cudaStream_t stream, int* launches) {
  using Cfg = tatn_dev::BwdCfg<D, DROP>;
  const int Nq_pad = (d.Nq + 127) / 128 * 128;
  const size_t rows = static_cast<size_t>(d.B) * d.H * Nq_pad;
  float* dq_acc = static_cast<float*>(ws);
  float* lse2 = dq_acc + rows * D;
  float* delta = lse2 + rows;
  int* item_counter = reinterpret_cast<int*>(delta + rows);
  uint32_t* custom_t = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(item_counter) + 16);
  const int custom_t_words = Nq_pad / 32;
  const bool custom = d.mask_kind == TATN_MASK_CUSTOM;
  float* dq_part = d.deterministic ? tatn_host::dq_part_ptr(d, ws) : nullptr;
  if (custom) {
    const int nb = d.custom_bstride != 0 ? d.B : 1;
    const long long warps = static_cast<long long>(nb) * custom_t_words * ((d.Nk + 31) / 32);
    const int blocks = static_cast<int>((warps * 32 + 255) / 256);
    cudaError_t e = tatn_host::launch(tatn_dev::tatn_custom_transpose, dim3(blocks), dim3(256), 0, stream, d.custom_mask,
                                      d.custom_words, d.custom_bstride, nb, d.Nq, d.Nk, custom_t_words, custom_t,
                                      d.k_offset / 32);
    if (e != cudaSuccess) return e;
  }
  {
    const dim3 blocks(static_cast<unsigned>((Nq_pad + 256 / (D / 8) - 1) / (256 / (D / 8))), d.H, d.B);
    cudaError_t e = tatn_host::launch(tatn_dev::tatn_bwd_pre<D, BF16, OUT_F32>, blocks, dim3(256), 0, stream, o,
                                      dO, lse, d.o_str[0], d.o_str[1], d.o_str[2], d.B,
                                      d.H, d.Nq, Nq_pad, lse2, delta, dq_acc, item_counter);
    if (e != cudaSuccess) return e;
  }
  CUtensorMap mq, mk, mv, mdo, mdk, mdv;
  if (!tatn_host::make_map_4d_ext(&mq, d.dtype, q, D, d.Nq, d.H, d.B, d.q_str, 64) ||
      !tatn_host::make_map_4d_ext(&mk, d.dtype, k, D, d.Nk, d.H, d.B, d.k_str, 128) ||
      !tatn_host::make_map_4d_ext(&mv, d.dtype, v, D, d.Nk, d.H, d.B, d.v_str, 128) ||
      !tatn_host::make_map_4d_ext(&mdo, d.dtype, dO, D, d.Nq, d.H, d.B, d.o_str, 64) ||
      !tatn_host::make_map_4d_ext(&mdk, d.dtype, OUT_F32 ? k : dk, D, d.Nk, d.H, d.B, d.k_str, 128) ||
      !tatn_host::make_map_4d_ext(&mdv, d.dtype, OUT_F32 ? v : dv, D, d.Nk, d.H, d.B, d.v_str, 128))
    return cudaErrorInvalidValue;
  tatn_dev::BwdParams p{};
  p.B = d.B;
  p.H = d.H;
  p.Nq = d.Nq;
  p.Nk = d.Nk;
  p.scale_log2 = d.tau * 1.4426950408889634f;
  p.tau = d.tau;
  p.mask_kind = d.mask_kind;
  p.valid_len = d.valid_len;
  p.grid = d.block_grid;
  p.tr = (d.Nq + 127) / 128;
  p.tc = (d.Nk + 127) / 128;
  p.visited = d.visited_bitmap;
  p.lse = lse;
  p.delta = delta;
  p.dq_acc = dq_acc;
  p.n_ktiles = p.tc;
  p.n_items = d.B * d.H * p.n_ktiles;
  p.item_counter = item_counter;
  p.custom_t = custom ? custom_t : nullptr;
  p.dq_part = dq_part;
  p.custom_t_words = custom_t_words;
  p.custom_t_b = (custom && d.custom_bstride != 0) ? 1 : 0;
  p.k_off = d.k_offset;
  // persistent + dynamic claims: one head group (global longest-first order) unless the heads'
  // Q / dO / dQ accumulators would not stay L2-resident (block-sparse d = 128: one CTA per item)
  p.group = tatn_host::schedule_group(d.B * d.H, (d.block_grid != nullptr && D == 128) ? p.n_ktiles : 1,
                                      static_cast<double>(d.Nq) * D * 8.0, 1);
  p.dk_f32 = OUT_F32 ? static_cast<float*>(dk) : nullptr;
  p.dv_f32 = OUT_F32 ? static_cast<float*>(dv) : nullptr;
  p.k_sb = d.k_str[0];
  p.k_sh = d.k_str[1];
  p.k_sn = d.k_str[2];
  p.v_sb = d.v_str[0];
  p.v_sh = d.v_str[1];
  p.v_sn = d.v_str[2];
  tatn_host::set_dropout(d, &p.drop_seed, &p.drop_thresh, &p.drop_scale);
  auto kern = tatn_dev::tatn_bwd_kernel<D, BF16, OUT_F32, DROP>;
  {
    cudaError_t e = tatn_host::ensure_smem_attr(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
  }
  // persistent, one CTA per SM looping over items (d = 128 block-sparse: one CTA per item, the grid
  // column read once into a shared-memory bitmask)
  const int n_sm = tatn_host::sm_count();
  dim3 grid(static_cast<unsigned>((d.block_grid != nullptr && !(Cfg::kMaskSlots == tatn_dev::kItemRing))
                                       ? p.n_items
                                       : std::min(p.n_items, n_sm)));
  cudaEvent_t prof_stop = tatn_host::profile_begin(1, stream);
  cudaError_t e = tatn_host::launch(kern, grid, dim3(Cfg::kThreads), Cfg::kSmemBytes, stream, mq, mk, mv, mdo,
                                    mdk, mdv, p, static_cast<const float*>(lse2), Nq_pad);
  if (prof_stop) cudaEventRecord(prof_stop, stream);
  if (e != cudaSuccess) return e;
  {
    const dim3 blocks(static_cast<unsigned>((d.Nq + 256 / (D / 8) - 1) / (256 / (D / 8))), d.H, d.B);
    if (dq_part != nullptr)
      e = tatn_host::launch_post_det<D, BF16, OUT_F32>(d, dq_part, dq, Nq_pad, tatn_dev::kBwdQT, stream);
    else
      e = tatn_host::launch(tatn_dev::tatn_bwd_post<D, BF16, OUT_F32>, blocks, dim3(256), 0, stream,
                            static_cast<const float*>(dq_acc), dq, d.q_str[0], d.q_str[1], d.q_str[2], d.B, d.H, d.Nq,
                            Nq_pad);
    if (e != cudaSuccess) return e;
  }
  *launches = custom ? 4 : 3;
  return cudaSuccess;
}

static inline int tatn_bwd_launch(const tatn_attn_desc& d, const void* q, const void* k, const void* v, const void* o,
                                  const void* dO, const float* lse, void* dq, void* dk, void* dv, void* ws,
                                  cudaStream_t stream, int* launches) {
  const int sel = (d.d == 128 ? 8 : 0) + (d.dtype == TATN_DTYPE_BF16 ? 4 : 0) + (d.out_dtype == TATN_OUT_FP32 ? 2 : 0) +
                  (d.p_drop > 0.0 ? 1 : 0);
  cudaError_t e = cudaErrorInvalidValue;
#define TATN_BWD_CASE(i, DD, B16, F32, DR) \
  case i: e = tatn_bwd_launch_t<DD, B16, F32, DR>(d, q, k, v, o, dO, lse, dq, dk, dv, ws, stream, launches); break;
  switch (sel) {
    TATN_BWD_CASE(0, 64, false, false, false)
    TATN_BWD_CASE(1, 64, false, false, true)
    TATN_BWD_CASE(2, 64, false, true, false)
    TATN_BWD_CASE(3, 64, false, true, true)
    TATN_BWD_CASE(4, 64, true, false, false)
    TATN_BWD_CASE(5, 64, true, false, true)
    TATN_BWD_CASE(6, 64, true, true, false)
    TATN_BWD_CASE(7, 64, true, true, true)
    TATN_BWD_CASE(8, 128, false, false, false)
    TATN_BWD_CASE(9, 128, false, false, true)
    TATN_BWD_CASE(10, 128, false, true, false)
    TATN_BWD_CASE(11, 128, false, true, true)
    TATN_BWD_CASE(12, 128, true, false, false)
    TATN_BWD_CASE(13, 128, true, false, true)
    TATN_BWD_CASE(14, 128, true, true, false)
    TATN_BWD_CASE(15, 128, true, true, true)
  }
#undef TATN_BWD_CASE
  return e == cudaSuccess ? TATN_OK : TATN_E_CUDA;
}
