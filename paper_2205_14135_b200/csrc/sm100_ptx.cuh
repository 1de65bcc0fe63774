// sm100_ptx.cuh — thin inline-PTX wrappers for the sm_100a features the
// attention kernels use: mbarriers, TMA (cp.async.bulk.tensor), tcgen05
// (alloc / mma / commit / ld / st / fences) and UMMA descriptors.
//
// Everything here is hand-written PTX; no CUTLASS/CuTe code is included.
// Bit layouts of the shared-memory matrix descriptor and the instruction
// descriptor follow the PTX ISA "tcgen05 matrix descriptors" section.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace tatn_dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }

// One lane of a converged warp (elect.sync): lets ptxas issue TMA / tcgen05 ops from
// the uniform datapath without a per-thread serialisation loop.
__device__ __forceinline__ bool elect_one_sync() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// Programmatic dependent launch (kernels launched with the PDL attribute, tatn_launch.h): every
// kernel runs griddep_wait() before its first global-memory access, so its prologue (barrier
// init, TMEM allocation, descriptor prefetch) overlaps the previous kernel's tail; it signals
// griddep_launch() once it needs no more SM slots (no items left to claim).
#ifndef TATN_PDL_EARLY
#define TATN_PDL_EARLY 0  // 1: persistent kernels signal dependents once no items are left (measured slower:
                          // the waiting dependent CTAs share SMs with the tail)
#endif
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// monotonic shared-memory progress counters (for waits a lagging consumer may be >= 2 phases
// behind or ahead of, which an mbarrier parity wait cannot express)
__device__ __forceinline__ void st_release_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void wait_counter_ge(uint32_t addr, uint32_t target) {
  while (ld_acquire_u32(addr) < target) __nanosleep(32);
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Watchdog: a wait that has not completed after ~2^35 SM cycles (~17 s at 1.965 GHz)
// is a deadlock; trap so the launch fails loudly instead of hanging the device.
constexpr long long kWatchdogCycles = 1ll << 35;
#ifdef TATN_WAIT_DEBUG
// debug builds: a wait stuck for ~1 s records (block, thread, barrier, parity) in g_tatn_wait_dbg
// (host-mapped, so it survives the watchdog trap) and keeps waiting
__device__ unsigned long long* g_tatn_wait_dbg = nullptr;
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(bar, parity)) {
#ifdef TATN_WAIT_DEBUG
    if (clock64() - t0 > (1ll << 31) && g_tatn_wait_dbg) {  // record once, keep waiting (host-mapped buffer)
      const unsigned long long i = atomicAdd(g_tatn_wait_dbg, 1ull);
      if (i < 1000)
        g_tatn_wait_dbg[1 + i] = (static_cast<unsigned long long>(blockIdx.x) << 40) |
                                 (static_cast<unsigned long long>(threadIdx.x) << 28) |
                                 (static_cast<unsigned long long>(bar & 0xffffu) << 4) | parity;
      __threadfence_system();
      while (!mbar_try_wait(bar, parity)) {
        if (clock64() - t0 > kWatchdogCycles) __trap();
      }
      return;
    }
#endif
    if (clock64() - t0 > kWatchdogCycles) __trap();
  }
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
// 4-D tiled load, completion signalled on `bar` (complete_tx bytes).
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const void* tmap, uint32_t bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// 4-D tiled store from shared memory (bulk-group completion).
__device__ __forceinline__ void tma_store_4d(const void* tmap, uint32_t src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// 4-D tiled reduce-add (fp32) from shared memory into global.
__device__ __forceinline__ void tma_reduce_add_4d(const void* tmap, uint32_t src, int c0, int c1,
                                                  int c2, int c3) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group"
      " [%0, {%2, %3, %4, %5}], [%1];" ::"l"(reinterpret_cast<uint64_t>(tmap)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// Make generic-proxy shared-memory writes visible to the async proxy (TMA).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Warpgroup register re-balancing (all 128 threads of a warpgroup execute it).
// .inc only draws on registers the same CTA released with .dec: with R0 registers
// per thread at launch, sum(inc - R0) over the growing warpgroups must not exceed
// sum(R0 - dec) over the shrinking ones, or the .inc blocks forever.
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T  (kind::f16: bf16/fp16 in, fp32 accumulate)
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// kind::tf32 (fp32 operands read as tf32, fp32 accumulate): the fp32-input check mode
__device__ __forceinline__ void mma_ss_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_ts_tf32(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// fp32 -> tf32, round to nearest (ties away): the value the tf32 MMA then reads exactly
__device__ __forceinline__ float round_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// Arrive on `bar` once every tcgen05 op previously issued by this thread completes.
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}

// Shared-memory matrix descriptor, 128-byte swizzle (layout type 2), version 1.
//   start address >> 4 : bits [0,14)
//   leading byte offset >> 4 : bits [16,30)
//   stride byte offset >> 4  : bits [32,46)
//   version = 1 : bits [46,48); base offset = 0; lbo mode = 0
//   layout type : bits [61,64)
__device__ __forceinline__ uint64_t make_sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// Instruction descriptor for kind::f16 / kind::tf32 with fp32 accumulation.
//   c_format (bits 4-5) = 1 (F32); a_format (7-9), b_format (10-12): 0 F16, 1 BF16, 2 TF32
//   a_major (15), b_major (16): 0 K-major, 1 MN-major; N>>3 at 17-22; M>>4 at 24-28
__host__ __device__ constexpr uint32_t make_idesc_f16(uint32_t ab_fmt, uint32_t m, uint32_t n,
                                                      uint32_t a_mn_major, uint32_t b_mn_major) {
  return (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) | (a_mn_major << 15) | (b_mn_major << 16) |
         ((n >> 3) << 17) | ((m >> 4) << 24);
}

// 32 lanes x 32 bits, N columns: thread i of the warp gets TMEM lane
// (warp%4)*32 + i, registers r[c] = column (taddr.col + c). Load and
// wait::ld are fused in one asm statement so no register is read early.
#define TATN_TMEM_LD_FUSED_32(taddr, r)                                                          \
  asm volatile(                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                                  \
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                                  \
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"             \
      "tcgen05.wait::ld.sync.aligned;"                                                           \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])             \
      : "r"(taddr)                                                                               \
      : "memory")

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  TATN_TMEM_LD_FUSED_32(taddr, r);
}

// Asynchronous variant: issue only. The registers must not be read before
// tmem_ld_wait32(r) — which ties them to the wait so no use can be hoisted above it.
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait32(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                 "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
                 "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]),
                 "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]),
                 "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------- block-grid bitmasks
// Bitmask of the nonzero entries of a u8 vector (entry i at base[i * stride], i < n) into
// dst[0 .. ceil(n / 32)), by one whole warp. The loads of 16 ballot rounds are issued before the
// ballots, so the (L2-latency-bound, possibly strided) reads of a long grid row / column overlap
// instead of costing one round trip per 32 entries (N = 64K: 16 rounds per item).
#ifndef TATN_MASK_ROUNDS
#define TATN_MASK_ROUNDS 4  // A/B (butterfly N = 64K bwd): 1 -> 493, 4 -> 542, 8 -> 545, 16 -> 514 TFLOP/s; 16K equal
#endif
template <typename Store>
__device__ __forceinline__ void warp_nonzero_bits(const uint8_t* base, int n, int64_t stride, uint32_t lane,
                                                  Store store) {
  constexpr int R = TATN_MASK_ROUNDS;  // ballot rounds whose loads are in flight together
  for (int b0 = 0; b0 < n; b0 += 32 * R) {
    uint32_t v[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int i = b0 + 32 * u + static_cast<int>(lane);
      v[u] = (base != nullptr && i < n) ? __ldg(base + static_cast<int64_t>(i) * stride) : 0u;
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const uint32_t bits = __ballot_sync(0xffffffffu, v[u] != 0u);
      if (lane == 0 && b0 + 32 * u < n) store((b0 >> 5) + u, bits);
    }
  }
}

// ---------------------------------------------------------------- dropout
// splitmix64 finaliser of the reference's positional generator (dropout.cpp:7-12).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// per query row: mix64(mix64(seed) ^ (i + 1))   (dropout.cpp:14-17)
__device__ __forceinline__ uint64_t drop_row_hash(uint64_t seed, int i) {
  return mix64(mix64(seed) ^ (static_cast<uint64_t>(i) + 1));
}
// keep (i, j) iff u = (h >> 11) * 2^-53 >= p  <=>  h >= ceil(p * 2^53) << 11   (dropout.cpp:18-27)
__device__ __forceinline__ bool drop_keep(uint64_t row_hash, int j, uint64_t thresh) {
  return mix64(row_hash ^ ((static_cast<uint64_t>(j) + 1) << 1)) >= thresh;
}

// ---------------------------------------------------------------- math
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---- packed fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2 on sm_100a) and 3-input max (FMNMX3)
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_add_rm(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rm.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// 2^x for a pair of finite x <= 64 on the FMA/ALU pipes instead of MUFU:
// Cody-Waite split x = j + f (j = floor(x) via a round-toward-minus-infinity add
// of 1.5*2^23), 2^f by a degree-3 polynomial (max rel. error 8.6e-5 on [0, 1)),
// and 2^j added straight into the exponent field. x is clamped at -127.
__device__ __forceinline__ uint64_t exp2_poly_f2(uint64_t x) {
  float x0, x1;
  f2_unpack(x, x0, x1);
  x = f2_pack(fmaxf(x0, -127.f), fmaxf(x1, -127.f));
  const uint64_t magic = f2_pack(12582912.f, 12582912.f);
  const uint64_t y = f2_add_rm(x, magic);        // bits: 0x4B400000 + floor(x)
  const uint64_t fr = f2_sub(x, f2_sub(y, magic));  // x - floor(x) in [0, 1)
  uint64_t pp = f2_fma(f2_pack(0.07706515491008759f, 0.07706515491008759f), fr,
                       f2_pack(0.22764705121517181f, 0.22764705121517181f));
  pp = f2_fma(pp, fr, f2_pack(0.6951163411140442f, 0.6951163411140442f));
  pp = f2_fma(pp, fr, f2_pack(1.f, 1.f));
  const uint32_t ylo = static_cast<uint32_t>(y), yhi = static_cast<uint32_t>(y >> 32);
  const uint32_t plo = static_cast<uint32_t>(pp), phi = static_cast<uint32_t>(pp >> 32);
  return (static_cast<uint64_t>(phi + (yhi << 23)) << 32) | static_cast<uint64_t>(plo + (ylo << 23));
}

// 2^x on a packed pair of 16-bit values (one MUFU op for two results). The
// fp32 pair is rounded to the 16-bit type first; the result is already the
// packed P operand of the P.V MMA.
template <bool BF16>
__device__ __forceinline__ uint32_t ex2_pair16(float x0, float x1) {
  uint32_t in, out;
  if constexpr (BF16) {
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(in) : "f"(x1), "f"(x0));
    asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(out) : "r"(in));
  } else {
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(in) : "f"(x1), "f"(x0));
    asm("ex2.approx.f16x2 %0, %1;" : "=r"(out) : "r"(in));
  }
  return out;
}
// widen a packed 16-bit pair to a packed fp32 pair
template <bool BF16>
__device__ __forceinline__ uint64_t widen_pair16(uint32_t v) {
  float lo, hi;
  if constexpr (BF16) {
    lo = __uint_as_float(v << 16);
    hi = __uint_as_float(v & 0xffff0000u);
  } else {
    const __half2 h = *reinterpret_cast<const __half2*>(&v);
    lo = __low2float(h);
    hi = __high2float(h);
  }
  return f2_pack(lo, hi);
}

template <bool BF16>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  if constexpr (BF16) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
  } else {
    __half2 v = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
  }
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

// ---- per-CTA globaltimer trace (debug builds only: -DTATN_TRACE)
#ifdef TATN_TRACE
__device__ unsigned long long* g_tatn_trace = nullptr;  // [grid][8] globaltimer stamps (debug builds only)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TATN_TRACE_AT(slot)                                                                     \
  do {                                                                                          \
    if (g_tatn_trace) g_tatn_trace[static_cast<size_t>(blockIdx.x) * 16 + (slot)] = gtimer();   \
  } while (0)
#else
#define TATN_TRACE_AT(slot) \
  do {                      \
  } while (0)
#endif
// per-event SM clock trace of CTA 0 (debug builds only): slot `ev` of Q tile g
#ifdef TATN_TRACE
// TATN_EV_INIT caches the trace pointer in a register (a global load per event would
// perturb the timeline it measures)
#define TATN_EV_INIT() unsigned long long* const tatn_ev_buf = (blockIdx.x == 0) ? g_tatn_trace : nullptr
// per-item events of CTA 0 (item n < 256, slot ev < 4) after the per-tile region
#define TATN_EVI(n, ev)                                                                                  \
  do {                                                                                                   \
    if (tatn_ev_buf && (n) < 256)                                                                        \
      tatn_ev_buf[200000ull * 16 + 8192 + static_cast<unsigned long long>(n) * 4 + (ev)] = clock64();    \
  } while (0)
#define TATN_EV(g, ev)                                                                                   \
  do {                                                                                                   \
    if (tatn_ev_buf && (g) < 1024)                                                                       \
      tatn_ev_buf[200000ull * 16 + static_cast<unsigned long long>(g) * 8 + (ev)] = clock64();           \
  } while (0)
// a second bank of 8 per-tile events (after the per-item region)
#define TATN_EV2(g, ev)                                                                                  \
  do {                                                                                                   \
    if (tatn_ev_buf && (g) < 1024)                                                                       \
      tatn_ev_buf[200000ull * 16 + 9216 + static_cast<unsigned long long>(g) * 8 + (ev)] = clock64();    \
  } while (0)
#else
#define TATN_EV_INIT() \
  do {                 \
  } while (0)
#define TATN_EV(g, ev) \
  do {                 \
  } while (0)
#define TATN_EV2(g, ev) \
  do {                  \
  } while (0)
#define TATN_EVI(n, ev) \
  do {                  \
  } while (0)
#endif

}  // namespace tatn_dev
