// Microbenchmark: the d = 64 backward's MMA-issuer loop on its own (no softmax / dQ / producer
// work: every mbarrier it waits on is already complete), in the issue styles under test.
//   style 0: K3's structure — whole warp runs the loop, four mbarrier waits per Q tile, one
//            elect_one_sync() block per MMA group, operands from shared-memory values
//   style 1: one lane runs the loop (no elect / syncwarp per group)
//   style 2: style 1 + descriptors advanced per k-step from one base per group
// cycles per Q tile (24 tcgen05.mma); mma_insitu.cu: 892 for back-to-back issue.
#include <cstdio>
#include <cstdint>
#include "../../paper_2205_14135_b200/csrc/sm100_ptx.cuh"
using namespace tatn_dev;

constexpr int S = 4;  // Q / dO stages
constexpr int kQTile = 64 * 128, kQSub = 64 * 128, kKV = 128 * 128, kDS = 128 * 128;

__global__ void __launch_bounds__(384, 1) kissue(unsigned long long* out, int R, int style, int noise = 0) {
  __shared__ volatile int stop;
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = smem_u32(sm);
  __shared__ uint64_t bar[8];
  __shared__ uint32_t slot;
  __shared__ volatile int ring[4];
  for (int i = threadIdx.x; i < 196608 / 16; i += blockDim.x) st_shared_v4(base + 16 * i, 0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int b = 0; b < 8; ++b) mbar_init(smem_u32(&bar[b]), 1);
    fence_mbar_init();
    ring[0] = 0; ring[1] = 1;
    stop = 0;
  }
  if (threadIdx.x < 32) { tmem_alloc(smem_u32(&slot), 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = slot;
  if (threadIdx.x >= 128) {  // noise warps (2 per SM sub-partition, like K3's softmax warpgroups)
    const int w = threadIdx.x >> 5;
    uint32_t acc = 0, r[32];
    float f0 = threadIdx.x * 1e-3f, f1 = 0.5f;
    const uint32_t vbase = base + 196608 - 1024;  // a small broadcast vector region
    while (noise && !stop) {
      if (noise == 1) {  // LDS.128 broadcasts (the softmax's lse2 / D vector reads)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint32_t a0, a1, a2, a3;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(vbase + u * 16));
          acc += a0 ^ a3;
        }
      } else if (noise == 2) {  // mbarrier polling
        acc += mbar_try_wait(smem_u32(&bar[7]), 0) ? 1u : 0u;
      } else if (noise == 3) {  // tcgen05.ld
        tmem_ld32(tmem_base + (((w & 3) * 32u) << 16) + ((w & 4) ? 64 : 0), r);
        acc += r[0] ^ r[31];
      } else if (noise == 4) {
#pragma unroll
        for (int u = 0; u < 16; ++u) { f0 = ex2_approx(f0 * 0.999f); f1 = fmaf(f1, 0.999f, f0); }
      } else if (noise == 5) {  // st.shared.v4 (dS^T stores)
        const uint32_t a = base + 150000 + (threadIdx.x - 128) * 16;
#pragma unroll
        for (int u = 0; u < 4; ++u) st_shared_v4(a + (u & 1) * 4096, acc, u, 0, 0);
        ++acc;
      }
    }
    if (acc == 0x12345678u || f1 == 123.f) out[0] = acc;
  }
  const uint32_t sKV = base, sQ = base + 65536, sDO = sQ + S * kQTile, sDS = sDO + S * kQTile;
  auto BAR = [&](int i) { return smem_u32(&bar[i]); };
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    constexpr uint32_t idesc_s = make_idesc_f16(1, 128, 64, 0, 0);
    constexpr uint32_t idesc_acc = make_idesc_f16(1, 128, 64, 0, 1);
    constexpr uint32_t idesc_dq = make_idesc_f16(1, 64, 64, 1, 1);
    const uint64_t dKV0 = make_sdesc_sw128(sKV, 16, 1024);
    const uint64_t dQk0 = make_sdesc_sw128(sQ, 16, 1024);
    const uint64_t dDOk0 = make_sdesc_sw128(sDO, 16, 1024);
    const uint64_t dQmn0 = make_sdesc_sw128(sQ, kQSub, 1024);
    const uint64_t dDOmn0 = make_sdesc_sw128(sDO, kQSub, 1024);
    const uint64_t dKmn0 = make_sdesc_sw128(sKV, 128 * 128, 1024);
    const uint64_t dDS0 = make_sdesc_sw128(sDS, 128 * 128, 1024);
    const int cnt = ring[1] * R;  // not provably uniform, like K3's item count
    const uint32_t koff = static_cast<uint32_t>(ring[0]) * 2 * kKV, voff = koff + kKV;
    const bool solo = style == 1 || style == 2;
    const bool do_wait = style < 4 || style == 10 || style >= 12, do_fence = style < 3 || style == 10 || style >= 12;
    const bool one_elect = style >= 6 && style <= 9;
    const bool in_elect = style >= 10;
    // 12: dQ^T(g) written over the TS A operand of back(g) (TMEM write-after-read in the pipe);
    // 13: front(g + 2) written over it instead (K3's pre-round-2 order)
    const int war = style - 11;
    const int nst = style == 8 ? 1 : (style == 9 ? 2 : S);  // 8: one Q / dO stage, 9: two
    const uint32_t voff_dp = style == 7 ? koff : voff;  // 7: dP^T front reads K (operand reuse test)
    auto WAIT = [&](int b) {
      if (do_wait) mbar_wait(BAR(b), 1);
      if (do_fence) tc_fence_after();
    };
    unsigned long long t0 = clock64();
    if (in_elect) {
      if (elect_one_sync()) {
        for (int g = 0; g < cnt; ++g) {
          const int x = g & 1, s = g % S;
          WAIT(0);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ts(tmem_base + 256, tmem_base + x * 128 + kk * 8, dDOmn0 + ((s * kQTile + kk * 2048) >> 4), idesc_acc, 1u);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ts(tmem_base + 320, tmem_base + x * 128 + 64 + kk * 8, dQmn0 + ((s * kQTile + kk * 2048) >> 4), idesc_acc, 1u);
          const int s2 = (g + 2) % S;
          WAIT(1);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ss(tmem_base + x * 128 + 64, dKV0 + ((voff + kk * 32) >> 4), dDOk0 + ((s2 * kQTile + kk * 32) >> 4), idesc_s, kk > 0 ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ss(tmem_base + x * 128, dKV0 + ((koff + kk * 32) >> 4), dQk0 + ((s2 * kQTile + kk * 32) >> 4), idesc_s, kk > 0 ? 1u : 0u);
          mma_commit(BAR(2 + x));
          WAIT(4);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ss(tmem_base + (war == 1 ? x * 128 : 384 + x * 64), dKmn0 + ((koff + kk * 2048) >> 4),
                   dDS0 + (((g % 2) * kDS + kk * 2048) >> 4), idesc_dq, kk > 0 ? 1u : 0u);
          mma_commit(BAR(5));
          mma_commit(BAR(6));
          mma_commit(BAR(7));
        }
        mma_commit(BAR(0));
      }
    } else if (!solo || lane == 0) {
      auto issue = [&](auto&& fn) {
        if (solo || one_elect) fn();
        else {
          if (elect_one_sync()) fn();
          __syncwarp();
        }
      };
      const bool el = one_elect ? elect_one_sync() : true;
      for (int g = 0; g < cnt && el; ++g) {
        const int x = g & 1, s = g % nst;
        WAIT(0);  // PFull (complete)
        issue([&] {
          if (style == 2) {
            const uint64_t bdo = dDOmn0 + ((s * kQTile) >> 4), bq = dQmn0 + ((s * kQTile) >> 4);
            const uint32_t tx = tmem_base + x * 128;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma_ts(tmem_base + 256, tx + kk * 8, bdo + kk * 128, idesc_acc, 1u);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) mma_ts(tmem_base + 320, tx + 64 + kk * 8, bq + kk * 128, idesc_acc, 1u);
          } else {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ts(tmem_base + 256, tmem_base + x * 128 + kk * 8, dDOmn0 + ((s * kQTile + kk * 2048) >> 4), idesc_acc, 1u);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ts(tmem_base + 320, tmem_base + x * 128 + 64 + kk * 8, dQmn0 + ((s * kQTile + kk * 2048) >> 4), idesc_acc, 1u);
          }
        });
        const int g2 = g + 2, s2 = g2 % nst;
        WAIT(1);  // QFull(g + 2) (complete)
        issue([&] {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t offa = voff_dp + kk * 32, offb = kk * 32;
            mma_ss(tmem_base + x * 128 + 64, dKV0 + (offa >> 4), (style == 7 ? dQk0 : dDOk0) + ((s2 * kQTile + offb) >> 4), idesc_s,
                   kk > 0 ? 1u : 0u);
          }
        });
        issue([&] {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t offa = koff + kk * 32, offb = kk * 32;
            mma_ss(tmem_base + x * 128, dKV0 + (offa >> 4), dQk0 + ((s2 * kQTile + offb) >> 4), idesc_s, kk > 0 ? 1u : 0u);
          }
          mma_commit(BAR(2 + x));
        });
        WAIT(4);  // DQEmpty (complete)
        issue([&] {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ss(tmem_base + 384 + x * 64, dKmn0 + ((koff + kk * 2048) >> 4), dDS0 + (((g % 2) * kDS + kk * 2048) >> 4), idesc_dq,
                   kk > 0 ? 1u : 0u);
          mma_commit(BAR(5));
          mma_commit(BAR(6));
          mma_commit(BAR(7));
        });
      }
      if (one_elect) { if (el) mma_commit(BAR(0)); }
      else issue([&] { mma_commit(BAR(0)); });  // final: BAR(0) phase 0 completes after every MMA
    }
    __syncwarp();
    mbar_wait(BAR(0), 0);
    unsigned long long t1 = clock64();
    if (lane == 0) { out[blockIdx.x] = t1 - t0; stop = 1; }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem_base, 512); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(kissue, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 1024);
  const int R = 512;
  const char* names[14] = {"K3 structure (warp + elect per group)", "one lane runs the loop", "one lane + per-group bases",
                          "K3 without tcgen05.fence::after", "K3 without mbarrier waits", "K3 without waits and fences",
                          "one elect per tile, no waits / fences", "6 + dP front reads K, Q (reuse)",
                          "6 with one Q / dO stage", "6 with two Q / dO stages",
                          "loop inside one elect region, waits", "loop inside one elect region, no waits",
                          "10 + dQ over back's A operand (WAR)", "10 (same)"};
  for (int style = 0; style < 14; ++style) {
    kissue<<<148, 384, 196608 + 1024>>>(d, 16, style);
    cudaDeviceSynchronize();
    kissue<<<148, 384, 196608 + 1024>>>(d, R, style);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
    printf("%-40s: %7.1f cycles per Q tile (24 MMAs) %s\n", names[style], s / 148 / R, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  const char* nn[6] = {"none", "LDS.128 broadcast", "mbarrier try_wait", "tcgen05.ld x32", "ex2 + ffma", "st.shared.v4"};
  for (int noise = 0; noise < 6; ++noise) {
    kissue<<<148, 384, 196608 + 1024>>>(d, 16, 10, noise);
    cudaDeviceSynchronize();
    kissue<<<148, 384, 196608 + 1024>>>(d, R, 10, noise);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double sum = 0; for (int i = 0; i < 148; ++i) sum += h[i];
    printf("style 10 + 8 warps of %-20s: %7.1f cycles per Q tile %s\n", nn[noise], sum / 148 / R, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  cudaFree(d);
  return 0;
}
