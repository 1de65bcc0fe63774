// tatn_fwd.cuh — constants shared by the forward kernels (K1) and the partial-result merge.
//
// The forward itself (tatn::flash_forward / tatn::blocksparse_forward, reference
// proj/core/include/tatn/flash.hpp:43-67; Algorithm 2) lives in
//   tatn_fwd1.cuh  d = 64, persistent, one 128-row Q tile per item, two CTAs per SM;
//   tatn_fwd2.cuh  d = 128, persistent, Q-tile pairs, one CTA per SM;
//   tatn_tf32.cuh  fp32 inputs (check mode, kind::tf32).
// The reference's loop order is K/V-block outer, Q-block inner with O/l/m read-modify-written
// to HBM each outer pass; outputs are schedule-invariant (flash.hpp:37-40), so here
// each CTA owns its Q tiles and streams K/V tiles through shared memory: O, l, m never leave the
// SM until the final write.
#pragma once

#include <type_traits>

#include "sm100_ptx.cuh"
#include "tatn_params.h"

namespace tatn_dev {

constexpr int kBM = 128;  // query rows per Q tile
constexpr int kBN = 128;  // keys per K/V tile
constexpr float kRescaleThreshold = 8.0f;  // lazy O rescale (log2 units)
// exp2 pairs per group of 8 computed by the polynomial on the FMA pipe instead of MUFU
// (MUFU.EX2 retires 16/clk/SM). Swept on B200 (r01): 1 of 8 is best (+3-5%); 2 or 3 of 8
// lose to the extra FMA-pipe issue. Full tiles only (masked tiles hold -inf).
#ifndef TATN_EMU_PAIRS
#define TATN_EMU_PAIRS 1
#endif
constexpr int kEmuPairs = TATN_EMU_PAIRS;
#ifndef TATN_EMU_PAIRS_D128
#define TATN_EMU_PAIRS_D128 0  // d = 128 forward: exp2 pairs (of 8) on the FMA pipe
#endif
// d = 128 keeps every exp2 on MUFU: there the MMA and MUFU are balanced and the FMA-pipe
// polynomial measured slower (N = 8K causal fwd 889 -> 912 TFLOP/s without it)
template <int D>
constexpr int kEmuPairsD = D == 128 ? TATN_EMU_PAIRS_D128 : kEmuPairs;

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
