// Microbenchmark: TMEM -> register read throughput (tcgen05.ld.32x32b.x32) per SM on this GPU.
// One CTA per SM (grid 148), W warps; every warp reads its 32 TMEM lanes x 32 columns (4 KB) per
// load, NL loads in flight before tcgen05.wait::ld. Prints bytes / clk / SM.
#include <cstdint>
#include <cstdio>
#include "../../paper_2205_14135_b200/csrc/sm100_ptx.cuh"
using namespace tatn_dev;

template <int NL>
__global__ void __launch_bounds__(512, 1) k(unsigned* out, int iters, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) { tmem_alloc(smem_u32(&slot), 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t base = slot + ((static_cast<uint32_t>(warp & 3) * 32) << 16) + (warp >> 2) * 64;
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[NL][32];
#pragma unroll
    for (int l = 0; l < NL; ++l) tmem_ld32_async(base + (l & 1) * 32, r[l]);
#pragma unroll
    for (int l = 0; l < NL; ++l) tmem_ld_wait32(r[l]);
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
      for (int i = 0; i < 32; ++i) acc ^= r[l][i];
  }
  const long long t1 = clock64();
  if (acc == 0x12345678u) out[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(slot, 512); }
}

template <int NL>
void run(int warps) {
  unsigned* o; long long* c;
  cudaMalloc(&o, 4); cudaMalloc(&c, 148 * 8);
  const int iters = 2000;
  k<NL><<<148, warps * 32>>>(o, 10, c); cudaDeviceSynchronize();
  k<NL><<<148, warps * 32>>>(o, iters, c); cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  double mean = 0; for (int i = 0; i < 148; ++i) mean += h[i]; mean /= 148;
  const double bytes = double(warps) * iters * NL * 4096;
  printf("warps %2d loads-in-flight %d: %.1f B/clk/SM (%s)\n", warps, NL, bytes / mean, cudaGetErrorString(e));
}
int main() {
  for (int w : {4, 8, 16}) { run<1>(w); run<2>(w); run<4>(w); }
  return 0;
}
