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
int main() {
  const int R = 4096;
  run<32, false>(R); run<64, false>(R); run<128, false>(R); run<256, false>(R);
  run<32, true>(R); run<64, true>(R); run<128, true>(R); run<256, true>(R);
  run<64, false, 64, 0>(R); run<64, false, 64, 1>(R); run<64, false, 128, 1>(R); run<128, false, 64, 1>(R);
  return 0;
}
