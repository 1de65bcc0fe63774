// Microbenchmark: cycles per tcgen05.mma (kind::f16, M=128, K=16) on one SM for N in
// {32, 64, 128, 256}, A from shared memory (SS) or TMEM (TS). One CTA per SM, one thread
// issues R MMAs back to back on fixed operands, then commit + wait; clock64 around it.
#include <cstdio>
#include <cstdint>
#include "../../paper_2205_14135_b200/csrc/sm100_ptx.cuh"
using namespace tatn_dev;

template <int N, bool TS, int M = 128, int AMN = 0>
__global__ void __launch_bounds__(128, 1) k(unsigned long long* out, int R) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = smem_u32(sm);
  // zero 64 KB of operands
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) st_shared_v4(base + 16 * i, 0, 0, 0, 0);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  if (threadIdx.x < 32) { tmem_alloc(smem_u32(&slot), 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x < 32) {
    const uint64_t da = make_sdesc_sw128(base, 16, 1024);
    const uint64_t db = make_sdesc_sw128(base + 32768, 16, 1024);
    constexpr uint32_t idesc = make_idesc_f16(1, M, N, AMN, 0);
    unsigned long long t0 = clock64();
    if (elect_one_sync()) {
      for (int r = 0; r < R; ++r) {
        if (TS) mma_ts(tm + 256, tm + (r & 3) * 8, db + ((r & 3) * 32 >> 4), idesc, r > 0 ? 1u : 0u);
        else mma_ss(tm + 256, da + ((r & 3) * 32 >> 4), db + ((r & 3) * 32 >> 4), idesc, r > 0 ? 1u : 0u);
      }
      mma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

template <int N, bool TS, int M = 128, int AMN = 0>
void run(int R) {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  auto f = k<N, TS, M, AMN>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  f<<<148, 128, 65536 + 1024>>>(d, 64);
  cudaDeviceSynchronize();
  f<<<148, 128, 65536 + 1024>>>(d, R);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
  printf("M=%d AMN=%d %s N=%3d: %7.1f cycles/MMA  (floor 128*N/256 = %d)  %s\n", M, AMN, TS ? "TS" : "SS", N, s / 148 / R, 128 * N / 256,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

// The backward's per-Q-tile MMA stream at d = 64 (dV, dK TS N=64; S^T, dP^T SS N=64; dQ^T SS M=64),
// R times back to back: cycles per tile-equivalent (24 MMAs; ideal 1024 at 128 B/clk smem).
__global__ void __launch_bounds__(128, 1) kmix(unsigned long long* out, int R, int variant, int noise = 0) {
  __shared__ volatile int stop;
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = smem_u32(sm);
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) st_shared_v4(base + 16 * i, 0, 0, 0, 0);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); stop = 0; }
  if (threadIdx.x < 32) { tmem_alloc(smem_u32(&slot), 512); tmem_relinquish(); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x >= 32 && noise == 2) {  // other warps: TMEM -> register loads (their lane quarter)
    const uint32_t w = tm + (((threadIdx.x >> 5) & 3) * 32u << 16);
    uint32_t acc = 0, r[32];
    while (!stop) {
      tmem_ld32(w + 0, r);
      acc += r[0] ^ r[31];
    }
    if (acc == 0x12345678u) out[0] = acc;
  }
  if (threadIdx.x >= 32 && noise == 1) {  // other warps: 16-byte st.shared into a separate 16 KB region
    const uint32_t w = base + 49152 + (threadIdx.x - 32) * 16;
    uint32_t i = 0;
    while (!stop) {
      for (int u = 0; u < 8; ++u) st_shared_v4(w + ((i + u) & 7) * 1536, i, u, 0, 0);
      i += 8;
    }
  }
  if (threadIdx.x < 32) {
    const uint64_t dA = make_sdesc_sw128(base, 16, 1024);            // K-major A (K or V)
    const uint64_t dB = make_sdesc_sw128(base + 32768, 16, 1024);    // K-major B (Q or dO)
    const uint64_t dBmn = make_sdesc_sw128(base + 32768, 8192, 1024);
    const uint64_t dAmn = make_sdesc_sw128(base, 16384, 1024);
    constexpr uint32_t id_s = make_idesc_f16(1, 128, 64, 0, 0);
    constexpr uint32_t id_acc = make_idesc_f16(1, 128, 64, 0, 1);
    constexpr uint32_t id_dq = make_idesc_f16(1, 64, 64, 1, 1);
    unsigned long long t0 = clock64();
    if (elect_one_sync()) {
      for (int r = 0; r < R; ++r) {
        const uint32_t x = (r & 1) * 128;
        if (variant == 0 || variant == 1) {
          for (int kk = 0; kk < 4; ++kk) mma_ts(tm + 256, tm + x + kk * 8, dBmn + ((kk * 2048) >> 4), id_acc, 1u);  // dV
          for (int kk = 0; kk < 4; ++kk) mma_ts(tm + 320, tm + x + 64 + kk * 8, dBmn + ((kk * 2048) >> 4), id_acc, 1u);  // dK
        }
        if (variant == 0 || variant == 2) {
          for (int kk = 0; kk < 4; ++kk) mma_ss(tm + x + 64, dA + ((kk * 32) >> 4), dB + ((kk * 32) >> 4), id_s, kk > 0);  // dP^T
          for (int kk = 0; kk < 4; ++kk) mma_ss(tm + x, dA + ((kk * 32) >> 4), dB + ((kk * 32) >> 4), id_s, kk > 0);  // S^T
        }
        if (variant == 0 || variant == 3)
          for (int kk = 0; kk < 8; ++kk) mma_ss(tm + 384 + (r & 1) * 64, dAmn + ((kk * 2048) >> 4), dBmn + ((kk * 2048) >> 4), id_dq, kk > 0);  // dQ^T
        if (variant == 4) {  // 128 query rows per step: fronts N = 128, dV / dK K = 128, dQ M = 128
          constexpr uint32_t id_s128 = make_idesc_f16(1, 128, 128, 0, 0);
          constexpr uint32_t id_dq128 = make_idesc_f16(1, 128, 64, 0, 1);
          for (int kk = 0; kk < 8; ++kk) mma_ts(tm + 384, tm + kk * 8, dBmn + ((kk * 2048) >> 4), id_acc, 1u);  // dV
          for (int kk = 0; kk < 8; ++kk) mma_ts(tm + 448, tm + 64 + kk * 8, dBmn + ((kk * 2048) >> 4), id_acc, 1u);  // dK
          for (int kk = 0; kk < 4; ++kk) mma_ss(tm + 128, dA + ((kk * 32) >> 4), dB + ((kk * 32) >> 4), id_s128, kk > 0);  // dP^T
          for (int kk = 0; kk < 4; ++kk) mma_ss(tm, dA + ((kk * 32) >> 4), dB + ((kk * 32) >> 4), id_s128, kk > 0);  // S^T
          for (int kk = 0; kk < 8; ++kk) mma_ss(tm + 256, dA + ((kk * 32) >> 4), dBmn + ((kk * 2048) >> 4), id_dq128, kk > 0);  // dQ
        }
        if (variant == 5)  // dQ as M = 128 over two 64-row Q tiles (half a tile's worth per rep)
          for (int kk = 0; kk < 4; ++kk) mma_ss(tm + 384, dA + ((kk * 32) >> 4), dBmn + ((kk * 2048) >> 4), make_idesc_f16(1, 128, 64, 0, 1), kk > 0);
      }
      mma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; stop = 1; }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 512); }
}
void runmix(int R) {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(kmix, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  const char* names[6] = {"full tile (24 MMAs)", "dV+dK TS (8)", "S^T+dP^T SS (8)", "dQ^T M=64 SS (8)",
                          "128-row tile (32 MMAs)", "dQ M=128 half (4)"};
  const int cnt[6] = {24, 8, 8, 8, 32, 4};
  for (int vv = 0; vv < 18; ++vv) {
    const int v = vv % 6, noise = vv / 6;
    if (noise == 1 && v == 0) printf("-- with 3 warps streaming st.shared.v4 --\n");
    if (noise == 2 && v == 0) printf("-- with 3 warps streaming tcgen05.ld 32x32b.x32 --\n");
    kmix<<<148, 128, 65536 + 1024>>>(d, 16, v, noise);
    cudaDeviceSynchronize();
    kmix<<<148, 128, 65536 + 1024>>>(d, R, v, noise);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
    printf("bwd stream %-22s: %7.1f cycles per tile, %5.1f per MMA %s\n", names[v], s / 148 / R, s / 148 / R / cnt[v],
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  cudaFree(d);
}

int main() {
  const int R = 4096;
  run<32, false>(R); run<64, false>(R); run<128, false>(R); run<256, false>(R);
  run<32, true>(R); run<64, true>(R); run<128, true>(R); run<256, true>(R);
  runmix(512);
  run<64, false, 64, 0>(R); run<64, false, 64, 1>(R); run<64, false, 128, 1>(R); run<128, false, 64, 1>(R);
  return 0;
}
